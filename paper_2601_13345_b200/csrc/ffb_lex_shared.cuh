// Shared pieces of the two lexer kernels (exact walk in ffb_lex.cu, fast path in ffb_lexfast.cu):
// byte classes, the packed-token classifier, operand descriptors, declaration parsers and the
// statement emitter.  Everything sits in an anonymous namespace of the including file.
#pragma once
#include "ffb_records.cuh"

// Byte-serial helpers are real calls: inlined at every use they made each lexer kernel 15-25 K
// instructions long, far beyond the instruction cache (ncu r1l: 80% of the issue slots of the
// record-mode lexer were "no instruction" stalls).  walk_line stays inline: it owns the hot
// per-lane state of the exact kernel.
#define FFB_COLD __device__ __noinline__
#define FFB_COLD_INLINE __device__ __forceinline__

namespace {

constexpr int kWarps = 8;
constexpr int kTile = 4096;                 // bytes staged per warp
constexpr int kPad = 64;                    // readable slack after the tile (look-ahead)
constexpr int kLaneBytes = kTile / 32;
constexpr int kMaxLines = 1024;
constexpr int kWarpSmem = kTile + kPad + kMaxLines * 2;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint8_t kNlInBlock = 0x8A;        // newline that sits inside a /* */ comment (T1 -> T2)

enum Phase { PH_SEARCH = 0, PH_HEADER, PH_BODY, PH_DONE };

// byte classes of the per-line feature scan
enum { CC_WS = 1, CC_SEMI = 2, CC_LBRACE = 4, CC_RBRACE = 8, CC_COLON = 16, CC_LABEL = 32, CC_OPEN = 64, CC_CLOSE = 128 };
FFB_HD uint8_t char_class(unsigned c) {
  return (uint8_t)((ffb_is_ws(c) ? CC_WS : 0) | (c == ';' ? CC_SEMI : 0) | (c == '{' ? CC_LBRACE : 0) |
                   (c == '}' ? CC_RBRACE : 0) | (c == ':' ? CC_COLON : 0) | (ffb_is_label_char(c) ? CC_LABEL : 0) |
                   ((c == '[' || c == '{' || c == '(') ? CC_OPEN : 0) | ((c == ']' || c == '}' || c == ')') ? CC_CLOSE : 0));
}
// what the feature scan makes of a line (anything it cannot prove simple is LK_COMPLEX and
// takes the general statement walk)
enum { LK_BLANK = 0, LK_STMT, LK_LABEL, LK_SKIP, LK_COMPLEX };

// comment automaton states
enum { S_CODE = 0, S_SLASH, S_SLASH2, S_LINE, S_LINE_SLASH, S_BLK, S_BLK_STAR, S_LBLK, S_LBLK_STAR };

struct LexArgs {
  const uint8_t* text;
  int64_t n_bytes;            // readable bytes (multiple of 16)
  const int64_t* seg_off;     // [K+1]
  int64_t n_segs;
  const int32_t* order;       // optional processing order
  const uint8_t* want_name;   // optional kernel name filter (device)
  int want_len;
  unsigned long long* work;   // work counter
  uint32_t* hist;             // [K, 9]
  FfbSegInfo* info;           // [K]
  // record mode
  const int64_t* ins_base;
  const int64_t* lab_base;
  const int64_t* ins_cap;     // optional per-segment record capacities (single-pass mode)
  const int64_t* lab_cap;
  FfbInsRec* ins;
  FfbLabelRec* labels;
  uint32_t* meta;             // optional compact copy of the meta words
  FfbSpanRec* spans;          // optional, parallel to ins
  FfbDeclRec* decls;          // optional, [K, FFB_MAX_DECLS]
  // fast path -> exact kernel hand-over (ffb_lexfast.cuh)
  int32_t* fb_list;           // segments the fast path declined
  unsigned long long* fb_count;
  const unsigned long long* n_work;   // exact kernel: number of entries of `order` to process (device), or NULL = n_segs
};

// ---- small warp helpers -------------------------------------------------------------------
FFB_D int warp_excl_sum(int v, int* total) {
  const int lane = threadIdx.x & 31;
  int x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int o = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += o;
  }
  *total = __shfl_sync(kFull, x, 31);
  return x - v;
}
FFB_D int warp_min(int v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { int o = __shfl_xor_sync(kFull, v, d); v = o < v ? o : v; }
  return v;
}
FFB_D unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}

FFB_D int next_bit(const uint32_t m[4], int from);

// ---- T1: comment automaton ------------------------------------------------------------------
// allow_block = false: "/*" no longer opens a comment (the reference's regex only matches a
// "/*" that has a closing "*/" somewhere behind it, ptx.py:140)
FFB_D int cm_step(int st, unsigned c, bool allow_block) {
  const bool sl = c == '/', star = c == '*' && allow_block, nl = c == '\n';
  switch (st) {
    case S_CODE: return sl ? S_SLASH : S_CODE;
    case S_SLASH: return star ? S_BLK : (sl ? S_SLASH2 : S_CODE);
    case S_SLASH2: return star ? S_BLK : (sl ? S_LINE_SLASH : (nl ? S_CODE : S_LINE));
    case S_LINE: return sl ? S_LINE_SLASH : (nl ? S_CODE : S_LINE);
    case S_LINE_SLASH: return star ? S_LBLK : (sl ? S_LINE_SLASH : (nl ? S_CODE : S_LINE));
    case S_BLK: return star ? S_BLK_STAR : S_BLK;
    case S_BLK_STAR: return sl ? S_CODE : (star ? S_BLK_STAR : S_BLK);
    case S_LBLK: return star ? S_LBLK_STAR : (nl ? S_BLK : S_LBLK);
    default: /* S_LBLK_STAR */ return sl ? S_LINE : (star ? S_LBLK_STAR : (nl ? S_BLK : S_LBLK));
  }
}

// Runs the automaton over s[c0,c1) from state `st`; when `blank` is set rewrites comment
// bytes to ' ' (newlines inside block comments become kNlInBlock).  Returns the exit state.
// noblk_from: first position whose "/*" must NOT open a comment; last_open: position of the
// last "/*" that did open one (for the unterminated-comment fix-up).
FFB_D int cm_run(uint8_t* s, int c0, int c1, int st, bool blank, const uint32_t slash[4], int chunk_base,
                 int noblk_from, int* last_open) {
  for (int i = c0; i < c1; ++i) {
    if (st == S_CODE) {                       // nothing happens in code until the next '/'
      i = chunk_base + next_bit(slash, i - chunk_base);
      if (i >= c1) break;
    }
    const unsigned c = s[i];
    const int nx = cm_step(st, c, i - 1 < noblk_from);
    if (nx >= S_BLK && st < S_BLK) *last_open = i - 1;
    if (blank) {
      const bool in_blk = st >= S_BLK;
      if (in_blk) {
        s[i] = (c == '\n') ? kNlInBlock : ' ';
      } else if (st == S_LINE || st == S_LINE_SLASH) {
        if (c != '\n') s[i] = ' ';
      } else if (st == S_SLASH) {
        if (nx == S_BLK) { s[i - 1] = ' '; s[i] = ' '; }
      } else if (st == S_SLASH2) {
        if (nx == S_BLK) { s[i - 1] = ' '; s[i] = ' '; }          // "//*": first '/' stays code
        else { s[i - 2] = ' '; s[i - 1] = ' '; if (c != '\n') s[i] = ' '; }
      }
    }
    st = nx;
  }
  return st;
}

// 4-bit mask (bit i <-> byte i) of the bytes of w equal to the replicated pattern
FFB_D uint32_t eq_nibble(uint32_t w, uint32_t pattern) {
  const uint32_t m = __vcmpeq4(w, pattern) & 0x08040201u;
  return (m * 0x01010101u) >> 24;
}
// 128-bit position masks of a lane's aligned 128-byte chunk: bytes equal to pat_a or pat_b
// (mask_ab) and bytes equal to pat_b alone (mask_b).  Bits outside [lo_bit, hi_bit) are cleared.
FFB_D void chunk_masks(const uint8_t* chunk, uint32_t pat_a, uint32_t pat_b, int lo_bit, int hi_bit,
                       uint32_t mask_ab[4], uint32_t mask_b[4]) {
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const uint4 q = *reinterpret_cast<const uint4*>(chunk + v * 16);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t ab = 0, b = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t nb = eq_nibble(w[j], pat_b);
      ab |= (eq_nibble(w[j], pat_a) | nb) << (4 * j);
      b |= nb << (4 * j);
    }
    // v covers bytes [16v, 16v+16): halves of the 32-bit mask words
    if (v & 1) { mask_ab[v >> 1] |= ab << 16; mask_b[v >> 1] |= b << 16; }
    else { mask_ab[v >> 1] = ab; mask_b[v >> 1] = b; }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int lo = lo_bit - 32 * k, hi = hi_bit - 32 * k;
    uint32_t keep = 0xffffffffu;
    if (lo > 0) keep &= lo >= 32 ? 0u : (0xffffffffu << lo);
    if (hi < 32) keep &= hi <= 0 ? 0u : (0xffffffffu >> (32 - hi));
    mask_ab[k] &= keep; mask_b[k] &= keep;
  }
}
FFB_D int next_bit(const uint32_t m[4], int from) {       // first set bit at position >= from, or 128
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (from >= 32 * (k + 1)) continue;
    const int sh = from > 32 * k ? from - 32 * k : 0;
    const uint32_t x = m[k] & (0xffffffffu << sh);
    if (x) return 32 * k + __ffs((int)x) - 1;
  }
  return 128;
}

// ---- opcode classification (ptx.py:99-136, :64-76) ---------------------------------------------
// Dot-separated tokens of at most 8 bytes are packed into one u64 and looked up in a 256-slot
// perfect-hash table held in shared memory (multiplier found offline: no two of the 61 tokens
// the classifier knows share a slot).
struct OpcodeInfo {
  uint32_t cls, space, bytes, base, cmp;
};
constexpr uint64_t kTokMul = 0x142fcb2e01c7132dull;
enum { TB_NONE = 0, TB_BAR, TB_BARRIER, TB_LD, TB_LDU, TB_ST, TB_BRA, TB_ADD, TB_SUB, TB_MUL, TB_MAD, TB_FMA, TB_DIV,
       TB_SIN, TB_COS, TB_EX2, TB_LG2, TB_RCP, TB_RSQRT, TB_SQRT, TB_MOV, TB_SETP, TB_AND, TB_OR, TB_SHL, TB_SHR,
       TB_CVT, TB_SELP, TB_CVTA, TB_RET, TB_EXIT };
// token value: [4:0] base code  [7:5] element bytes code (1:1 2:2 3:4 4:8)  [8] float type  [9] int type
//              [11:10] vector (1:v2 2:v4)  [12] sync  [15:13] space + 1  [16] approx  [19:17] compare
constexpr uint32_t tv_base(uint32_t b) { return b; }
constexpr uint32_t tv_type(uint32_t code, bool f, bool i) { return (code << 5) | (f ? 1u << 8 : 0u) | (i ? 1u << 9 : 0u); }
struct TokDef { uint64_t key; uint32_t val; };
__constant__ TokDef kTokDefs[] = {
  {ffb_pk("bar"), TB_BAR}, {ffb_pk("barrier"), TB_BARRIER}, {ffb_pk("ld"), TB_LD}, {ffb_pk("ldu"), TB_LDU},
  {ffb_pk("st"), TB_ST}, {ffb_pk("bra"), TB_BRA}, {ffb_pk("add"), TB_ADD}, {ffb_pk("sub"), TB_SUB},
  {ffb_pk("mul"), TB_MUL}, {ffb_pk("mad"), TB_MAD}, {ffb_pk("fma"), TB_FMA}, {ffb_pk("div"), TB_DIV},
  {ffb_pk("sin"), TB_SIN}, {ffb_pk("cos"), TB_COS}, {ffb_pk("ex2"), TB_EX2}, {ffb_pk("lg2"), TB_LG2},
  {ffb_pk("rcp"), TB_RCP}, {ffb_pk("rsqrt"), TB_RSQRT}, {ffb_pk("sqrt"), TB_SQRT}, {ffb_pk("mov"), TB_MOV},
  {ffb_pk("setp"), TB_SETP}, {ffb_pk("and"), TB_AND}, {ffb_pk("or"), TB_OR}, {ffb_pk("shl"), TB_SHL},
  {ffb_pk("shr"), TB_SHR}, {ffb_pk("cvt"), TB_CVT}, {ffb_pk("selp"), TB_SELP}, {ffb_pk("cvta"), TB_CVTA},
  {ffb_pk("ret"), TB_RET}, {ffb_pk("exit"), TB_EXIT},
  {ffb_pk("b8"), tv_type(1, false, false)}, {ffb_pk("s8"), tv_type(1, false, false)}, {ffb_pk("u8"), tv_type(1, false, false)},
  {ffb_pk("b16"), tv_type(2, false, false)}, {ffb_pk("s16"), tv_type(2, false, false)}, {ffb_pk("u16"), tv_type(2, false, false)},
  {ffb_pk("f16"), tv_type(2, false, false)}, {ffb_pk("bf16"), tv_type(2, false, false)},
  {ffb_pk("b32"), tv_type(3, false, false)}, {ffb_pk("s32"), tv_type(3, false, true)}, {ffb_pk("u32"), tv_type(3, false, true)},
  {ffb_pk("f32"), tv_type(3, true, false)}, {ffb_pk("b64"), tv_type(4, false, false)}, {ffb_pk("s64"), tv_type(4, false, true)},
  {ffb_pk("u64"), tv_type(4, false, true)}, {ffb_pk("f64"), tv_type(4, true, false)},
  {ffb_pk("v2"), 1u << 10}, {ffb_pk("v4"), 2u << 10}, {ffb_pk("sync"), 1u << 12},
  {ffb_pk("global"), (uint32_t)(FFB_SP_GLOBAL + 1) << 13}, {ffb_pk("shared"), (uint32_t)(FFB_SP_SHARED + 1) << 13},
  {ffb_pk("local"), (uint32_t)(FFB_SP_LOCAL + 1) << 13}, {ffb_pk("param"), (uint32_t)(FFB_SP_PARAM + 1) << 13},
  {ffb_pk("const"), (uint32_t)(FFB_SP_PARAM + 1) << 13}, {ffb_pk("approx"), 1u << 16},
  {ffb_pk("lt"), (uint32_t)FFB_CMP_LT << 17}, {ffb_pk("ge"), (uint32_t)FFB_CMP_GE << 17}, {ffb_pk("le"), (uint32_t)FFB_CMP_LE << 17},
  {ffb_pk("gt"), (uint32_t)FFB_CMP_GT << 17}, {ffb_pk("eq"), (uint32_t)FFB_CMP_EQ << 17}, {ffb_pk("ne"), (uint32_t)FFB_CMP_NE << 17},
};
constexpr int kNumTokDefs = sizeof(kTokDefs) / sizeof(kTokDefs[0]);
struct TokTable { const uint64_t* key; const uint32_t* val; };

FFB_D uint32_t tok_lookup(const TokTable& tt, uint64_t pk) {
  const uint32_t i = (uint32_t)((pk * kTokMul) >> 56);
  return tt.key[i] == pk ? tt.val[i] : 0u;
}

// the decision part of classify_opcode, from what the token loop collected
FFB_D OpcodeInfo finish_opcode(uint32_t base, uint32_t elem_code, uint32_t vec, uint32_t space, uint32_t cmp, uint32_t flags) {
  OpcodeInfo r;
  const uint32_t elem = elem_code == 0 ? 4u : (1u << (elem_code - 1));
  r.bytes = elem * (vec == 0 ? 1u : (vec == 1 ? 2u : 4u));
  r.cmp = cmp;
  r.space = FFB_SP_NONE;
  r.base = FFB_BASE_OTHER;
  switch (base) {
    case TB_MOV: r.base = FFB_BASE_MOV; break;
    case TB_CVT: r.base = FFB_BASE_CVT; break;
    case TB_CVTA: r.base = FFB_BASE_CVTA; break;
    case TB_ADD: r.base = FFB_BASE_ADD; break;
    case TB_SUB: r.base = FFB_BASE_SUB; break;
    case TB_MUL: r.base = FFB_BASE_MUL; break;
    case TB_MAD: r.base = FFB_BASE_MAD; break;
    case TB_FMA: r.base = FFB_BASE_FMA; break;
    case TB_SHL: r.base = FFB_BASE_SHL; break;
    case TB_SETP: r.base = FFB_BASE_SETP; break;
    case TB_RET: r.base = FFB_BASE_RET; break;
    case TB_EXIT: r.base = FFB_BASE_EXIT; break;
    default: break;
  }
  // decision order of ptx.py:108-128
  const uint32_t bit = 1u << base;
  constexpr uint32_t kArith = (1u << TB_ADD) | (1u << TB_SUB) | (1u << TB_MUL) | (1u << TB_MAD) | (1u << TB_FMA) | (1u << TB_DIV);
  constexpr uint32_t kSfu = (1u << TB_SIN) | (1u << TB_COS) | (1u << TB_EX2) | (1u << TB_LG2) | (1u << TB_RCP) | (1u << TB_RSQRT);
  constexpr uint32_t kAlu = (1u << TB_MOV) | (1u << TB_SETP) | (1u << TB_AND) | (1u << TB_OR) | (1u << TB_SHL) | (1u << TB_SHR) |
                            (1u << TB_CVT) | (1u << TB_SELP);
  if (base == TB_BAR || base == TB_BARRIER || (flags & 8u)) r.cls = FFB_CLS_SYNC;
  else if (base == TB_LD || base == TB_LDU) { r.cls = FFB_CLS_MEMLOAD; r.space = space ? space - 1 : FFB_SP_NONE; }
  else if (base == TB_ST) { r.cls = FFB_CLS_MEMSTORE; r.space = space ? space - 1 : FFB_SP_NONE; }
  else if (base == TB_BRA) r.cls = FFB_CLS_BRANCH;
  else if (bit & kArith) r.cls = (flags & 1u) ? FFB_CLS_FP32 : ((flags & 2u) ? FFB_CLS_INT : FFB_CLS_OTHER);
  else if (bit & kSfu) r.cls = FFB_CLS_SFU;
  else if (base == TB_SQRT) r.cls = (flags & 4u) ? FFB_CLS_SFU : FFB_CLS_OTHER;
  else if (bit & kAlu) r.cls = FFB_CLS_ALU;
  else r.cls = FFB_CLS_OTHER;
  return r;
}

FFB_D OpcodeInfo classify_opcode(const TokTable& tt, const uint8_t* s, int o0, int o1) {
  uint64_t pk = 0;
  int tl = 0, ti = 0;
  uint32_t base = TB_NONE, elem_code = 0, vec = 0, space = 0, cmp = 0, flags = 0;   // flags: 1 f, 2 i, 4 approx, 8 last-is-sync
  for (int i = o0; i <= o1; ++i) {
    const unsigned c = i < o1 ? s[i] : (unsigned)'.';
    if (c != '.') {
      if (tl < 8) pk |= (uint64_t)c << (8 * tl);
      ++tl;
      continue;
    }
    const uint32_t v = tl > 8 ? 0u : tok_lookup(tt, pk);
    flags &= ~8u;
    if (ti == 0) base = v & 31u;
    else {
      const uint32_t ec = (v >> 5) & 7u;
      if (ec) elem_code = ec;
      flags |= (v >> 8) & 3u;                       // float / int type seen (ptx.py:116-119)
      const uint32_t vc = (v >> 10) & 3u;
      if (vc) vec = vc;
      if (v & (1u << 12)) flags |= 8u;
      const uint32_t sp = (v >> 13) & 7u;
      if (sp && !space) space = sp;                 // first space token wins (ptx.py:131-135)
    }
    if (v & (1u << 16)) flags |= 4u;
    if (!cmp) cmp = (v >> 17) & 7u;                 // first compare token, any position (cfg.py:222)
    pk = 0; tl = 0; ++ti;
  }
  return finish_opcode(base, elem_code, vec, space, cmp, flags);
}

// ---- operand description (alignment.py:31-47, cfg.py:184-188) ----------------------------------
// Hash of s[a,b) with every blank run that contains a newline collapsed to one ' ' (what the
// reference's "strip each line, join with one space" does to a multi-line statement).
FFB_COLD uint64_t norm_hash(const uint8_t* s, int a, int b) {
  FfbHasher x;
  ffb_hash_init(x);
  int i = a;
  while (i < b) {
    const unsigned c = s[i];
    if (!ffb_is_ws(c)) { ffb_hash_byte(x, c); ++i; continue; }
    int j = i;
    bool nl = false;
    while (j < b && ffb_is_ws(s[j])) { nl = nl || s[j] == '\n'; ++j; }
    if (nl) ffb_hash_byte(x, ' ');
    else for (int k = i; k < j; ++k) ffb_hash_byte(x, s[k]);
    i = j;
  }
  return ffb_hash_done(x);
}

FFB_D bool span_eq(const uint8_t* s, int a, int b, const char* lit, int n) {
  if (b - a != n) return false;
  for (int i = 0; i < n; ++i)
    if (s[a + i] != (uint8_t)lit[i]) return false;
  return true;
}
FFB_D bool span_ends(const uint8_t* s, int a, int b, const char* lit, int n) {
  if (b - a < n) return false;
  for (int i = 0; i < n; ++i)
    if (s[b - n + i] != (uint8_t)lit[i]) return false;
  return true;
}

// Python int(text, 0) on s[a,b) (already stripped).  0: not a literal, 1: value in *out, 2: too big.
FFB_COLD int py_int_literal(const uint8_t* s, int a, int b, int64_t* out) {
  int i = a;
  bool neg = false;
  if (i < b && (s[i] == '+' || s[i] == '-')) { neg = s[i] == '-'; ++i; }
  if (i >= b) return 0;
  unsigned base = 10;
  bool prefixed = false;
  if (s[i] == '0' && i + 1 < b) {
    const unsigned p = s[i + 1] | 32u;
    if (p == 'x') base = 16; else if (p == 'o') base = 8; else if (p == 'b') base = 2;
    if (base != 10) { prefixed = true; i += 2; }
  }
  uint64_t v = 0;
  bool big = false, any = false, prev_us = false, nonzero_lead = false, first_zero = false;
  int ndig = 0;
  if (prefixed && i < b && s[i] == '_') ++i;              // "0x_ff" is legal
  for (; i < b; ++i) {
    const unsigned c = s[i];
    if (c == '_') {
      if (prev_us || !any) return 0;
      prev_us = true;
      continue;
    }
    unsigned d;
    if (ffb_is_digit(c)) d = c - '0';
    else if (base == 16 && ((c | 32u) - 'a') < 6u) d = (c | 32u) - 'a' + 10;
    else return 0;
    if (d >= base) return 0;
    if (ndig == 0) { first_zero = d == 0; }
    if (d != 0) nonzero_lead = true;
    ++ndig;
    any = true;
    prev_us = false;
    if (v > (0x0fffffffffffffffull - d) / base) big = true; else v = v * base + d;
  }
  if (!any || prev_us) return 0;
  if (!prefixed && first_zero && nonzero_lead) return 0;   // "010" is rejected, "00" is zero
  if (big || v >= (1ull << 60)) return 2;
  *out = neg ? -(int64_t)v : (int64_t)v;
  return 1;
}

FFB_COLD uint64_t describe_operand(const uint8_t* s, int a, int b) {
  const uint64_t h = norm_hash(s, a, b);
  if (s[a] == '%') {
    if (span_eq(s, a, b, "%tid.x", 6)) return ffb_op_make(FFB_OPK_TIDX, h);
    if ((b - a >= 5 && span_eq(s, a, a + 5, "%tid.", 5)) || span_eq(s, a, b, "%laneid", 7) || span_eq(s, a, b, "%warpid", 7))
      return ffb_op_make(FFB_OPK_UNKNOWN, h);
    bool uni = span_ends(s, a, b, "%gridid", 7) || span_ends(s, a, b, "WARP_SZ", 7);
    if (!uni && b - a >= 2 && s[b - 2] == '.' && (s[b - 1] == 'x' || s[b - 1] == 'y' || s[b - 1] == 'z'))
      uni = span_ends(s, a, b - 2, "%ctaid", 6) || span_ends(s, a, b - 2, "%nctaid", 7) || span_ends(s, a, b - 2, "%ntid", 5);
    return ffb_op_make(uni ? FFB_OPK_UNIFORM_REG : FFB_OPK_REG, h);
  }
  int64_t v = 0;
  const int lit = py_int_literal(s, a, b, &v);
  if (lit == 1) return ffb_op_make(FFB_OPK_INT, (uint64_t)v);
  if (lit == 2) return ffb_op_make(FFB_OPK_BIGINT, h);
  return ffb_op_make(FFB_OPK_UNIFORM, h);
}

// alignment.py:21 address regex on the operand s[a,b) (starts with '[').  Returns the address
// kind and, for registers, the descriptor of the base name.
FFB_COLD uint32_t describe_address(const uint8_t* s, int a, int b, uint64_t* desc) {
  *desc = 0;
  if (b - a < 2 || s[b - 1] != ']') return FFB_ADDR_NOMATCH;
  const int i0 = a + 1, i1 = b - 1;
  int plus = -1;
  for (int i = i0; i < i1; ++i) {
    if (s[i] == ']') return FFB_ADDR_NOMATCH;
    if (s[i] == '+' && plus < 0) plus = i;
  }
  const int l1 = plus < 0 ? i1 : plus;
  if (l1 == i0) return FFB_ADDR_NOMATCH;
  if (plus >= 0) {                       // `\+\s*-?\d+\s*` up to the closing bracket
    int r0 = plus + 1, r1 = i1;
    while (r0 < r1 && ffb_is_ws(s[r0])) ++r0;
    while (r1 > r0 && ffb_is_ws(s[r1 - 1])) --r1;
    if (r0 < r1 && s[r0] == '-') ++r0;
    if (r0 >= r1) return FFB_ADDR_NOMATCH;
    for (int i = r0; i < r1; ++i)
      if (!ffb_is_digit(s[i])) return FFB_ADDR_NOMATCH;
  }
  int b0 = i0, b1 = l1;
  while (b0 < b1 && ffb_is_ws(s[b0])) ++b0;
  while (b1 > b0 && ffb_is_ws(s[b1 - 1])) --b1;
  if (b0 < b1 && s[b0] == '%') {
    *desc = ffb_op_make(FFB_OPK_REG, norm_hash(s, b0, b1));
    return FFB_ADDR_REG;
  }
  return FFB_ADDR_SYMBOL;
}

// ---- directives (ptx.py:37-40,244-254) -----------------------------------------------------------
FFB_D int scan_ws(const uint8_t* s, int i, int e) { while (i < e && ffb_is_ws(s[i])) ++i; return i; }
FFB_D int scan_word(const uint8_t* s, int i, int e, bool dollar) {
  while (i < e && (ffb_is_word(s[i]) || (dollar && s[i] == '$'))) ++i;
  return i;
}
FFB_D int scan_digits(const uint8_t* s, int i, int e, uint64_t* v) {
  uint64_t x = 0;
  while (i < e && ffb_is_digit(s[i])) { if (x < (1ull << 59)) x = x * 10 + (s[i] - '0'); ++i; }
  *v = x;
  return i;
}
FFB_D uint32_t type_bytes(const uint8_t* s, int a, int b, uint32_t dflt) {
  if (b - a > 8) return dflt;
  uint64_t pk = 0;
  for (int i = a; i < b; ++i) pk |= (uint64_t)s[i] << (8 * (i - a));
  switch (pk) {
    case ffb_pk("b8"): case ffb_pk("s8"): case ffb_pk("u8"): return 1;
    case ffb_pk("b16"): case ffb_pk("s16"): case ffb_pk("u16"): case ffb_pk("f16"): case ffb_pk("bf16"): return 2;
    case ffb_pk("b32"): case ffb_pk("s32"): case ffb_pk("u32"): case ffb_pk("f32"): return 4;
    case ffb_pk("b64"): case ffb_pk("s64"): case ffb_pk("u64"): case ffb_pk("f64"): return 8;
    default: return dflt;
  }
}
// `.reg .cls %name<N>` -> count in *n, class token span in [*c0,*c1); false if not a match.
FFB_COLD bool parse_reg_decl(const uint8_t* s, int a, int e, uint64_t* n, int* c0, int* c1) {
  if (e - a < 4 || !span_eq(s, a, a + 4, ".reg", 4)) return false;
  int i = scan_ws(s, a + 4, e);
  if (i == a + 4 || i >= e || s[i] != '.') return false;
  int j = scan_word(s, i + 1, e, false);
  if (j == i + 1) return false;
  int k = scan_ws(s, j, e);
  if (k == j || k >= e || s[k] != '%') return false;
  int m = k + 1;
  while (m < e && (ffb_is_alpha(s[m]) || s[m] == '_')) ++m;
  if (m == k + 1 || m >= e || s[m] != '<') return false;
  int d = scan_digits(s, m + 1, e, n);
  if (d == m + 1 || d >= e || s[d] != '>') return false;
  if (scan_ws(s, d + 1, e) != e) return false;
  *c0 = i + 1; *c1 = j;
  return true;
}
// `.shared [.align N] .type name[N]` -> bytes; false if not a match.
FFB_COLD bool parse_shared_decl(const uint8_t* s, int a, int e, uint64_t* bytes) {
  if (e - a < 7 || !span_eq(s, a, a + 7, ".shared", 7)) return false;
  int i = scan_ws(s, a + 7, e);
  if (i == a + 7) return false;
  if (e - i >= 6 && span_eq(s, i, i + 6, ".align", 6)) {
    uint64_t dummy;
    int p = scan_ws(s, i + 6, e);
    int q = scan_digits(s, p, e, &dummy);
    int r = scan_ws(s, q, e);
    if (p > i + 6 && q > p && r > q) i = r;
  }
  if (i >= e || s[i] != '.') return false;
  int j = scan_word(s, i + 1, e, false);
  if (j == i + 1) return false;
  const uint32_t elem = type_bytes(s, i + 1, j, 1);
  int k = scan_ws(s, j, e);
  if (k == j) return false;
  int m = scan_word(s, k, e, true);
  if (m == k) return false;
  uint64_t count = 1;
  if (m < e && s[m] == '[') {
    int d = scan_digits(s, m + 1, e, &count);
    if (d == m + 1 || d >= e || s[d] != ']') return false;
    m = d + 1;
  }
  if (scan_ws(s, m, e) != e) return false;
  *bytes = (uint64_t)elem * count;
  return true;
}

// ---- per-line walk (ptx.py:227-270) -------------------------------------------------------------
struct LineSummary {
  bool nonblank, has_semi, pend_out0, defer, unterminated;
  int n0, n_after;        // instructions if pending-in is 0 / statements after the first ';'
  int lab0, lab_after;    // labels likewise
  int dcl0, dcl_after;    // .reg declarations likewise
};

struct Emit {
  // where this lane's results go (record mode) and its accumulators
  const LexArgs* a;
  TokTable tok;          // shared-memory token table
  const uint8_t* cls;    // shared-memory byte-class table
  int64_t seg;            // segment index
  int64_t seg_begin;      // global offset of the segment
  int64_t abase;          // global offset of smem index 0
  int64_t ins_at, lab_at; // next global record slots
  int64_t ins_limit, lab_limit;   // first slot NOT owned by this segment
  int dcl_at;
  uint32_t line;          // source line of the current line
  uint64_t c0, c1, c2;    // nine 21-bit class counters, three per word (no dynamically indexed array)
  unsigned long long shared_bytes, regs;
};

// Finds the ';' that closes a statement opened at `from` on a line ending at `e`, looking
// past the line (continuation lines) up to `hi`.  Tracks braces from `depth` so a body end
// stops the search.  Returns position or -1 (not in tile) / -2 (body ended first).
FFB_D int find_closing_semi(const uint8_t* s, int from, int hi, int depth) {
  for (int i = from; i < hi; ++i) {
    const unsigned c = s[i];
    if (c == ';') return i;
    if (c == '{') ++depth;
    else if (c == '}') { if (--depth == 0) return -2; }
  }
  return -1;
}

// kMode: 0 = summary only (never reaches here), 1 = class counts, 2 = class counts + records
template <int kMode>
FFB_D void do_statement(const uint8_t* s, int b, int e, Emit& em) {
  // s[b,e): statement text without the ';', possibly spanning lines; b is a non-blank byte
  while (e > b && ffb_is_ws(s[e - 1])) --e;
  if (e <= b) return;
  int i = b;
  bool has_pred = false, neg = false;
  int p0 = 0, p1 = 0;
  if (s[i] == '@') {                                   // ptx.py:42  ^@(!?%[\w$]+)\s+
    int j = i + 1;
    const bool n = j < e && s[j] == '!';
    if (n) ++j;
    if (j < e && s[j] == '%') {
      int k = j + 1;
      while (k < e && ffb_is_name_char(s[k])) ++k;
      if (k > j + 1 && k < e && ffb_is_ws(s[k])) {
        has_pred = true; neg = n; p0 = j; p1 = k;
        i = scan_ws(s, k, e);
      }
    }
  }
  const int o0 = i;
  int o1 = o0;
  while (o1 < e && !ffb_is_ws(s[o1])) ++o1;
  const OpcodeInfo oc = classify_opcode(em.tok, s, o0, o1);
  {
    const uint64_t inc = 1ull << (21 * (oc.cls % 3u));
    em.c0 += oc.cls < 3u ? inc : 0ull; em.c1 += (oc.cls >= 3u && oc.cls < 6u) ? inc : 0ull; em.c2 += oc.cls >= 6u ? inc : 0ull;
  }
  if (kMode < 2) { em.ins_at += 1; return; }

  FfbInsRec rec;
  rec.line = em.line;
  rec.off = (uint32_t)(em.abase + b - em.seg_begin);
  rec.len = (uint32_t)(e - b);
  rec.pred = has_pred ? norm_hash(s, p0, p1) : 0ull;
  rec.aux = 0;
  rec.op[0] = rec.op[1] = rec.op[2] = rec.op[3] = 0;
  FfbSpanRec* sp = em.a->spans ? em.a->spans + em.ins_at : nullptr;
  if (sp) {
    sp->pred_off = has_pred ? (uint32_t)(em.abase + p0 - (neg ? 1 : 0) - em.seg_begin) : 0;
    sp->pred_len = has_pred ? (uint32_t)(p1 - p0 + (neg ? 1 : 0)) : 0;
    sp->opc_off = (uint32_t)(em.abase + o0 - em.seg_begin);
    sp->opc_len = (uint32_t)(o1 - o0);
  }
  // operands: split at depth-0 commas (ptx.py:144-162).  Phase 1 only records the spans, so that
  // the per-operand work below starts at the same instruction for every lane of the warp
  // (describing operands inside this byte loop would run one lane at a time).
  int depth = 0, ps = -1, pe = -1, count = 0, last_s = -1, last_e = -1;
  int s0 = 0, e0 = 0, s1 = 0, e1 = 0, s2 = 0, e2 = 0, s3 = 0, e3 = 0, s4 = 0, e4 = 0, as = -1, ae = -1;
  bool extra_reg = false;
  const bool is_mem = oc.cls == FFB_CLS_MEMLOAD || oc.cls == FFB_CLS_MEMSTORE;
  const bool aux_is_op4 = !is_mem && oc.cls != FFB_CLS_BRANCH;
  for (int q = o1; q <= e; ++q) {
    const unsigned c = q < e ? s[q] : 0u;
    const unsigned kc = q < e ? em.cls[c] : 0u;
    depth += (int)((kc >> 6) & 1u) - (int)((kc >> 7) & 1u);
    if (q == e || (c == ',' && depth == 0)) {
      if (ps >= 0) {
        if (count == 0) { s0 = ps; e0 = pe; } else if (count == 1) { s1 = ps; e1 = pe; }
        else if (count == 2) { s2 = ps; e2 = pe; } else if (count == 3) { s3 = ps; e3 = pe; }
        else if (count == 4) { s4 = ps; e4 = pe; if (!aux_is_op4 && s[ps] == '%') extra_reg = true; }
        else if (s[ps] == '%') extra_reg = true;
        if (is_mem && as < 0 && s[ps] == '[') { as = ps; ae = pe; }
        if (sp && count < FFB_MAX_SPAN_OPS) {
          sp->op_off[count] = (uint32_t)(em.abase + ps - em.seg_begin);
          sp->op_len[count] = (uint32_t)(pe - ps);
        }
        last_s = ps; last_e = pe;
        ++count;
      }
      ps = -1;
    } else if (!(kc & CC_WS)) {
      if (ps < 0) ps = q;
      pe = q + 1;
    }
  }
  // Phase 2: describe the operands, slot by slot
  const bool dst_reg = count > 0 && s[s0] == '%';
  if (count > 0) rec.op[0] = describe_operand(s, s0, e0);
  if (count > 1) rec.op[1] = describe_operand(s, s1, e1);
  if (count > 2) rec.op[2] = describe_operand(s, s2, e2);
  if (count > 3) rec.op[3] = describe_operand(s, s3, e3);
  uint32_t addr_kind = FFB_ADDR_ABSENT;
  if (aux_is_op4) { if (count > 4) rec.aux = describe_operand(s, s4, e4); }
  else if (is_mem) { if (as >= 0) addr_kind = describe_address(s, as, ae, &rec.aux); }
  else rec.aux = last_s >= 0 ? ffb_op_make(FFB_OPK_REG, norm_hash(s, last_s, last_e)) : 0ull;
  if (sp) sp->n_ops = (uint32_t)count;
  rec.meta = oc.cls | (oc.space << 4) | ((oc.bytes & 63u) << 7) | (oc.base << 13) | ((has_pred ? 1u : 0u) << 18) |
             ((neg ? 1u : 0u) << 19) | ((uint32_t)(count > 7 ? 7 : count) << 20) | (oc.cmp << 23) | (addr_kind << 26) |
             ((dst_reg ? 1u : 0u) << 28) | ((extra_reg ? 1u : 0u) << 29);
  if (em.ins_at < em.ins_limit) {
    em.a->ins[em.ins_at] = rec;
    if (em.a->meta) em.a->meta[em.ins_at] = rec.meta;
  }
  em.ins_at += 1;
}

template <int kMode>
FFB_D void do_directive(const uint8_t* s, int b, int e, Emit& em, int* n_decl) {
  while (e > b && ffb_is_ws(s[e - 1])) --e;
  uint64_t n = 0;
  int c0 = 0, c1 = 0;
  if (parse_reg_decl(s, b, e, &n, &c0, &c1)) {
    *n_decl += 1;
    if (kMode > 0) {
      em.regs += n;
      if (kMode == 2 && em.a->decls && em.dcl_at < FFB_MAX_DECLS) {
        FfbDeclRec d;
        d.cls_off = (uint32_t)(em.abase + c0 - em.seg_begin);
        d.cls_len = (uint32_t)(c1 - c0);
        d.count = n;
        em.a->decls[em.seg * FFB_MAX_DECLS + em.dcl_at] = d;
      }
      em.dcl_at += 1;
    }
    return;
  }
  uint64_t bytes = 0;
  if (parse_shared_decl(s, b, e, &bytes)) {
    if (kMode > 0) em.shared_bytes += bytes;
  }
}

}  // namespace
