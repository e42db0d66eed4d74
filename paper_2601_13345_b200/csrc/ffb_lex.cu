// K1: GPU byte-lexer, opcode classifier and per-kernel class histogram.
//
// Restates (never copies) pkg/src/ptxwatt/ptx.py:99-313 of the reference: comment stripping
// (:139-141), kernel location and brace matching (:165-187), the line / ';' driven statement
// loop with labels, bare braces, directives and multi-line statements (:227-270), predicate
// and first-token opcode extraction (:296-313), the nine-class classifier (:99-136), access
// width (:64-76), .reg / .shared declarations (:37-40,244-254).
//
// Parallel formulation (one warp per corpus segment, i.e. per kernel):
//   T0  16-byte vector loads stage a 4 KB tile of text in shared memory;
//   T1  comment automaton, byte-parallel: each lane owns 128 bytes, lanes exchange their
//       entry state with shuffles until consistent, comment bytes are blanked in place
//       (the blanked text equals the reference's cleaned text up to trailing blanks);
//   T2  newline positions by per-lane counts + warp prefix sum  -> line table;
//   T3  one lane per line: brace depth (body end), a 2-bit "pending statement" map per line
//       composed across lanes with a shuffle scan (ptx.py's `pending` string is a 1-bit
//       state once the opener parses its own continuation), then the statement walk:
//       label / brace / directive / instruction, opcode tokens compared as packed u64 words.
//   Per-lane class counters are reduced with shuffles once per segment and stored by lane 0
//   (a segment has exactly one owner warp, so no atomics are needed on the histogram).
// In record mode the same walk also parses operands and writes one 64-byte FfbInsRec per
// instruction for the dataflow kernel (K1b).
#include "ffb_records.cuh"

// rarely taken, register-hungry paths are kept out of line so that the hot loop of the lexer
// is allocated for the common case only
#define FFB_COLD __device__ __forceinline__

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

// ---- operand description (alignment.py:31-47, cfg.py:184-188) ----------------------------------
// Hash of s[a,b) with every blank run that contains a newline collapsed to one ' ' (what the
// reference's "strip each line, join with one space" does to a multi-line statement).
FFB_D uint64_t norm_hash(const uint8_t* s, int a, int b) {
  uint64_t h = kFnvBasis;
  int i = a;
  for (; i < b; ++i) {                          // common case: no blank inside the operand
    const unsigned c = s[i];
    if (ffb_is_ws(c)) break;
    h = ffb_hash_step(h, c);
  }
  while (i < b) {
    const unsigned c = s[i];
    if (!ffb_is_ws(c)) { h = ffb_hash_step(h, c); ++i; continue; }
    int j = i;
    bool nl = false;
    while (j < b && ffb_is_ws(s[j])) { nl = nl || s[j] == '\n'; ++j; }
    if (nl) h = ffb_hash_step(h, ' ');
    else for (int k = i; k < j; ++k) h = ffb_hash_step(h, s[k]);
    i = j;
  }
  return ffb_hash_fold(h);
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

FFB_D uint64_t describe_operand(const uint8_t* s, int a, int b) {
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

// The statement loop of one line s[b,e) (newline excluded, possibly truncated at the body
// end).  pending_in: the line starts inside an unfinished statement.  hi/depth_in serve the
// look-ahead of a statement this line opens.  kMode 0 only fills the summary.
template <int kMode>
FFB_COLD LineSummary walk_line(const uint8_t* s, int b, int e, bool pending_in, int hi, int depth_in,
                            bool at_seg_end, Emit& em) {
  LineSummary r;
  r.nonblank = r.has_semi = r.pend_out0 = r.defer = r.unterminated = false;
  r.n0 = r.n_after = r.lab0 = r.lab_after = r.dcl0 = r.dcl_after = 0;
  int line_b = b;
  while (b < e && ffb_is_ws(s[b])) ++b;
  while (e > b && ffb_is_ws(s[e - 1])) --e;
  if (b >= e) { r.pend_out0 = false; return r; }
  r.nonblank = true;
  bool pending = pending_in;
  bool after_first = false;       // past the first ';' of the line
  int pos = b;
  // depth at `pos` is needed only when a statement is opened: count braces lazily
  while (pos < e) {
    if (!pending) {
      int k = pos;
      while (k < e && ffb_is_label_char(s[k])) ++k;
      if (k > pos && k < e && s[k] == ':') {                       // ptx.py:232-236
        if (kMode > 0) {
          if (kMode == 2) {
            FfbLabelRec L;
            const uint64_t h0 = norm_hash(s, pos, k);
            L.hash = h0; L.index = (uint32_t)(em.ins_at - em.a->ins_base[em.seg]);
            L.off = (uint32_t)(em.abase + pos - em.seg_begin);
            if (em.lab_at < em.lab_limit) em.a->labels[em.lab_at] = L;
          }
          em.lab_at += 1;
        }
        if (after_first) r.lab_after += 1;
        r.lab0 += 1;
        pos = scan_ws(s, k + 1, e);
        continue;
      }
      if (e - pos == 1 && (s[pos] == '{' || s[pos] == '}')) break;   // ptx.py:237-239
      if (s[pos] == '.') {                                        // ptx.py:240-256
        int semi = pos;
        while (semi < e && s[semi] != ';') ++semi;
        int nd = 0;
        do_directive<kMode>(s, pos, semi, em, &nd);
        r.dcl0 += nd;
        if (after_first) r.dcl_after += nd;
        if (semi < e) { if (!after_first) { r.has_semi = true; after_first = true; } pos = scan_ws(s, semi + 1, e); }
        else pos = e;
        continue;
      }
    }
    int semi = pos;
    while (semi < e && s[semi] != ';') ++semi;
    if (pending) {
      // continuation of a statement an earlier line opened: that line's lane parses it
      if (semi >= e) { pos = e; break; }                          // still pending (ptx.py:257-262)
      if (!after_first) { r.has_semi = true; after_first = true; }
      pending = false;
      pos = scan_ws(s, semi + 1, e);
      continue;
    }
    if (semi >= e) {
      // this line opens a multi-line statement: find its ';' further down the tile
      int d = depth_in;
      for (int i = line_b; i < pos; ++i) { if (s[i] == '{') ++d; else if (s[i] == '}') --d; }
      const int close = find_closing_semi(s, pos, hi, d);
      if (close == -2 || (close == -1 && at_seg_end)) { r.unterminated = true; r.pend_out0 = true; pos = e; break; }
      if (close == -1) { r.defer = true; r.pend_out0 = true; pos = e; break; }
      r.n0 += 1;
      if (after_first) r.n_after += 1;
      if (kMode > 0) do_statement<kMode>(s, pos, close, em);
      r.pend_out0 = true;
      pending = true;
      pos = e;
      break;
    }
    // ordinary statement s[pos, semi)
    {
      int q = semi;
      while (q > pos && ffb_is_ws(s[q - 1])) --q;
      if (q > pos) {
        r.n0 += 1;
        if (after_first) r.n_after += 1;
        if (kMode > 0) do_statement<kMode>(s, pos, semi, em);
      }
    }
    if (!after_first) { r.has_semi = true; after_first = true; }
    pos = scan_ws(s, semi + 1, e);
  }
  return r;
}

// ---- the kernel --------------------------------------------------------------------------------
// kRecords: also write FfbInsRec / FfbLabelRec (and the optional span / decl records)
template <bool kRecords>
__global__ void __launch_bounds__(kWarps * 32, kRecords ? 2 : 4)   // record mode needs ~128 registers (measured: capping at 64 spills and is 1.5x slower)
lex_corpus_kernel(LexArgs a) {
  constexpr int kMain = kRecords ? 2 : 1;
  FFB_DYN_SMEM(smem_raw);
  __shared__ uint8_t s_cls[256];
  __shared__ uint64_t s_tok_key[256];
  __shared__ uint32_t s_tok_val[256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* s = smem_raw + (size_t)wid * kWarpSmem;
  uint16_t* nl = reinterpret_cast<uint16_t*>(s + kTile + kPad);
  for (int c = threadIdx.x; c < 256; c += kWarps * 32) { s_cls[c] = char_class((unsigned)c); s_tok_key[c] = ~0ull; s_tok_val[c] = 0; }
  __syncthreads();
  for (int c = threadIdx.x; c < kNumTokDefs; c += kWarps * 32) {
    const uint32_t slot = (uint32_t)((kTokDefs[c].key * kTokMul) >> 56);
    s_tok_key[slot] = kTokDefs[c].key; s_tok_val[slot] = kTokDefs[c].val;
  }
  __syncthreads();

  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(a.work, 1ull);
    w = __shfl_sync(kFull, w, 0);
    if (w >= (unsigned long long)a.n_segs) break;
    const int64_t seg = a.order ? (int64_t)a.order[w] : (int64_t)w;
    const int64_t seg_begin = a.seg_off[seg], seg_end = a.seg_off[seg + 1];

    // ---- warp-uniform segment state ----
    int phase = PH_SEARCH;
    int cm_state = S_CODE;            // comment automaton state at `cur`
    int64_t noblk_from_g = 0x7fffffffffffffffLL;   // from here on "/*" is plain text (unterminated comment)
    int64_t blk_close_g = -1;         // a "*/" is known to exist up to here
    int depth = 0;
    bool pending = false;             // ptx.py's `pending` string is non-empty
    uint32_t line_no = 1;             // source line of the byte at `cur`
    uint32_t status = FFB_OK;
    int64_t cur = seg_begin;
    int64_t scan_from_g = seg_begin;  // SEARCH / HEADER resume position
    int64_t body_pos_g = 0;           // first body byte (after '{')
    int64_t name_off = 0, name_len = 0, body_end_off = 0;
    uint32_t n_instr = 0, n_labels = 0, n_decls = 0;

    Emit em;
    em.a = &a; em.seg = seg; em.seg_begin = seg_begin; em.abase = 0; em.line = 0;
    em.tok.key = s_tok_key; em.tok.val = s_tok_val; em.cls = s_cls;
    em.ins_at = kRecords ? a.ins_base[seg] : 0;
    em.lab_at = kRecords ? a.lab_base[seg] : 0;
    em.ins_limit = (kRecords && a.ins_cap) ? em.ins_at + a.ins_cap[seg] : 0x7fffffffffffffffLL;
    em.lab_limit = (kRecords && a.lab_cap) ? em.lab_at + a.lab_cap[seg] : 0x7fffffffffffffffLL;
    em.dcl_at = 0;
    em.c0 = em.c1 = em.c2 = 0;
    em.shared_bytes = 0; em.regs = 0;

    while (phase != PH_DONE && status == FFB_OK && cur < seg_end) {
      // ================= T0: stage the tile =================
      const int64_t abase = cur & ~(int64_t)15;
      const int64_t hi_g = (abase + kTile < seg_end) ? abase + kTile : seg_end;
      const int lo = (int)(cur - abase), hi = (int)(hi_g - abase);
      const bool at_seg_end = hi_g == seg_end;
      __syncwarp();
      for (int v = lane; v < kTile / 16; v += 32) {
        const int64_t g = abase + (int64_t)v * 16;
        uint4 val;
        if (g + 16 <= a.n_bytes) val = *reinterpret_cast<const uint4*>(a.text + g);
        else { val.x = val.y = val.z = val.w = 0x0a0a0a0au; }
        *reinterpret_cast<uint4*>(s + v * 16) = val;
      }
      __syncwarp();
      for (int i = hi + lane; i < kTile + kPad; i += 32) s[i] = '\n';
      __syncwarp();
      em.abase = abase;

      // ================= T1: comments =================
      const int chunk_base = lane * kLaneBytes;
      const int c0 = max(chunk_base, lo), c1 = min(chunk_base + kLaneBytes, hi);
      uint32_t slash[4], unused4[4];
      chunk_masks(s + chunk_base, 0x2f2f2f2fu, 0x2f2f2f2fu, c0 - chunk_base, c1 - chunk_base, slash, unused4);
      const bool has_slash = (slash[0] | slash[1] | slash[2] | slash[3]) != 0;
      int st_in = S_CODE, st_out = S_CODE, last_open = -1;
      int noblk_from = noblk_from_g >= abase + kTile ? 0x7fffffff : (noblk_from_g <= abase ? 0 : (int)(noblk_from_g - abase));
      for (int attempt = 0; attempt < 2; ++attempt) {
        bool need = true;
        st_in = S_CODE;
        for (int guard = 0; guard < 40; ++guard) {
          if (need) {
            last_open = -1;
            if (c0 >= c1) st_out = st_in;
            else if (!has_slash && st_in == S_CODE) st_out = S_CODE;
            else st_out = cm_run(s, c0, c1, st_in, false, slash, chunk_base, noblk_from, &last_open);
            need = false;
          }
          int left = __shfl_up_sync(kFull, st_out, 1);
          if (lane == 0) left = cm_state;
          const bool changed = left != st_in;
          if (!__any_sync(kFull, changed)) break;
          if (changed) { st_in = left; need = true; }
        }
        // a block comment still open at the tile end must have its "*/" somewhere behind
        const int end_state = __shfl_sync(kFull, st_out, 31);
        if (end_state < S_BLK || attempt == 1 || blk_close_g >= abase + hi) break;
        int64_t found = -1;
        const int64_t from = abase + hi - ((end_state == S_BLK_STAR || end_state == S_LBLK_STAR) ? 1 : 0);
        for (int64_t g0 = from; g0 < seg_end - 1 && found < 0; g0 += 32) {
          const int64_t g = g0 + lane;
          const bool hit = g + 1 < seg_end && a.text[g] == '*' && a.text[g + 1] == '/';
          const unsigned mask = __ballot_sync(kFull, hit);
          if (mask) found = g0 + __ffs((int)mask) - 1;
        }
        if (found >= 0) { blk_close_g = found + 2; break; }
        // unterminated: the last "/*" of this tile and everything behind it is ordinary text
        int lo_open = last_open;
#pragma unroll
        for (int dd = 16; dd > 0; dd >>= 1) { const int o = __shfl_xor_sync(kFull, lo_open, dd); lo_open = o > lo_open ? o : lo_open; }
        if (lo_open < 0) break;                       // opened in an earlier tile: cannot happen, keep going
        noblk_from_g = abase + lo_open;
        noblk_from = lo_open;
      }
      const bool dirty = (has_slash || st_in != S_CODE) && c0 < c1;
      if (__any_sync(kFull, dirty)) {
        int dummy = -1;
        if (dirty) cm_run(s, c0, c1, st_in, true, slash, chunk_base, noblk_from, &dummy);
        __syncwarp();
      }

      // ================= T2: line table =================
      uint32_t nlm[4], nlb[4];
      chunk_masks(s + chunk_base, 0x0a0a0a0au, 0x8a8a8a8au, c0 - chunk_base, c1 - chunk_base, nlm, nlb);
      const int my_nl = __popc(nlm[0]) + __popc(nlm[1]) + __popc(nlm[2]) + __popc(nlm[3]);
      int total_nl = 0;
      int at = warp_excl_sum(my_nl, &total_nl);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t m = nlm[k];
        while (m) {
          const int bit = __ffs((int)m) - 1;
          m &= m - 1;
          const int i = chunk_base + 32 * k + bit;
          const bool in_block = (nlb[k] >> bit) & 1u;
          if (at < kMaxLines) nl[at] = (uint16_t)(i | (in_block ? 0x8000 : 0));
          if (in_block) s[i] = '\n';
          ++at;
        }
      }
      const int n_real = total_nl < kMaxLines ? total_nl : kMaxLines;
      // the text may end without a newline: close the last line at `hi`
      const bool virtual_last = at_seg_end && total_nl < kMaxLines;
      if (virtual_last && lane == 0) nl[n_real] = (uint16_t)hi;
      const int n_lines = n_real + (virtual_last ? 1 : 0);
      __syncwarp();
      if (n_lines == 0) { status = FFB_E_CAPACITY; break; }         // a line longer than the tile
      const int region_end = virtual_last ? hi : (nl[n_real - 1] & 0x7fff) + 1;
      int consume_to = region_end;     // smem index where the next tile starts
      bool skip_rest = false;

      // ================= T3a: locate the kernel (ptx.py:165-187) =================
      if (phase == PH_SEARCH) {
        int from = (int)(scan_from_g - abase);
        if (from < lo) from = lo;
        for (;;) {
          int cand = 0x7fffffff;
          for (int i = max(c0, from); i < min(c1, region_end); ++i)
            if (s[i] == '.' && s[i + 1] == 'e' && s[i + 2] == 'n' && s[i + 3] == 't' && s[i + 4] == 'r' && s[i + 5] == 'y') { cand = i; break; }
          cand = warp_min(cand);
          if (cand == 0x7fffffff) { scan_from_g = abase + region_end; break; }
          int q = cand + 6;
          while (q < hi && ffb_is_ws(s[q])) ++q;
          int r = q;
          bool ok = q > cand + 6 && q < hi && ffb_is_name_start(s[q]);
          if (ok) { r = q + 1; while (r < hi && ffb_is_name_char(s[r])) ++r; }
          if ((q >= hi || (ok && r >= hi)) && !at_seg_end) {
            // the match runs off the staged bytes: restart the tile at the candidate
            if (cand == lo) status = FFB_E_CAPACITY;
            consume_to = cand; scan_from_g = abase + cand; skip_rest = true;
            break;
          }
          if (!ok) { from = cand + 1; continue; }
          bool take = true;
          if (a.want_name) {
            take = (r - q) == a.want_len;
            for (int i = 0; take && i < a.want_len; ++i) take = s[q + i] == a.want_name[i];
          }
          if (!take) { from = r; continue; }
          name_off = abase + q - seg_begin; name_len = r - q;
          phase = PH_HEADER; scan_from_g = abase + r;
          break;
        }
      }
      if (status != FFB_OK) break;
      if (phase == PH_HEADER && !skip_rest) {
        int from = (int)(scan_from_g - abase);
        if (from < lo) from = lo;
        int cand = 0x7fffffff;
        for (int i = max(c0, from); i < min(c1, region_end); ++i)
          if (s[i] == '{') { cand = i; break; }
        cand = warp_min(cand);
        if (cand == 0x7fffffff) {
          if (scan_from_g < abase + region_end) scan_from_g = abase + region_end;
        } else {
          phase = PH_BODY; depth = 1; pending = false;
          body_pos_g = abase + cand + 1;
        }
      }

      // ================= T3b: body lines (ptx.py:227-270) =================
      if (phase == PH_BODY && !skip_rest) {
        int pos = body_pos_g > cur ? (int)(body_pos_g - abase) : lo;
        if (pos <= region_end) {
          int first = 0;
          for (int l = lane; l < n_lines; l += 32) first += ((nl[l] & 0x7fff) < pos) ? 1 : 0;
          first = (int)warp_sum_u64((unsigned long long)first);
          for (int l0 = first; l0 < n_lines; l0 += 32) {
            const int li = l0 + lane;
            const bool live = li < n_lines;
            int b = 0, e = 0;
            if (live) {
              b = li == 0 ? lo : (nl[li - 1] & 0x7fff) + 1;
              e = nl[li] & 0x7fff;
              if (b < pos) b = pos;               // the line that holds the opening brace
            }
            // ---- feature scan: one uniform pass over the batch's lines ----
            const int len = live ? e - b : 0;
            int maxlen = len;
#pragma unroll
            for (int dd = 16; dd > 0; dd >>= 1) { const int o = __shfl_xor_sync(kFull, maxlen, dd); maxlen = o > maxlen ? o : maxlen; }
            int fb = 0x7fffffff, lb = -1, n_semi = 0, n_colon = 0, n_nonws = 0;
            unsigned seen = 0;
            for (int i = 0; i < maxlen; ++i) {
              if (i < len) {
                const unsigned k = s_cls[s[b + i]];
                seen |= k;
                n_semi += (k >> 1) & 1; n_colon += (k >> 4) & 1;
                if (!(k & CC_WS)) { fb = min(fb, b + i); lb = b + i; ++n_nonws; }
              }
            }
            if (lb < 0) fb = -1;
            // braces are rare (vector operands, nested scopes): walk them only where they occur
            int run = 0, min_run = 0x7fffffff;
            if (seen & (CC_LBRACE | CC_RBRACE)) {
              for (int i = b; i < e; ++i) {
                const unsigned c = s[i];
                if (c == '{') ++run;
                else if (c == '}') { --run; if (run < min_run) min_run = run; }
              }
            }
            int tot_delta = 0;
            const int d_in = depth + warp_excl_sum(run, &tot_delta);
            const bool closes = live && min_run != 0x7fffffff && d_in + min_run <= 0;
            const unsigned close_mask = __ballot_sync(kFull, closes);
            const int end_lane = close_mask ? __ffs((int)close_mask) - 1 : 32;
            int close_at = -1;
            if (lane == end_lane) {
              int d = d_in;
              for (int i = b; i < e; ++i) {
                const unsigned c = s[i];
                if (c == '{') ++d;
                else if (c == '}') { if (--d == 0) { close_at = i; break; } }
              }
              e = close_at;
            }
            const bool mine = live && lane <= end_lane;
            // ---- line kind ----
            int kind = LK_COMPLEX;
            if (fb < 0) kind = LK_BLANK;
            else if (min_run == 0x7fffffff || (min_run >= 0 && run == 0)) {
              const unsigned c_first = s[fb], c_last = s[lb];
              if (c_first == '.') {
                const bool decl = (s[fb + 1] == 'r' && s[fb + 2] == 'e' && s[fb + 3] == 'g') ||
                                  (s[fb + 1] == 's' && s[fb + 2] == 'h' && s[fb + 3] == 'a');
                if (n_semi == 0 && n_colon == 0 && !decl) kind = LK_SKIP;         // ptx.py:255-256
              } else if (c_last == ';' && n_semi == 1 && n_colon == 0 && lb > fb) {
                kind = LK_STMT;       // one statement, ';' last (braces inside operands are balanced)
              } else if (c_last == ':' && n_semi == 0 && n_colon == 1 && lb - fb + 1 == n_nonws && lb > fb) {
                bool all_label = true;                                            // ptx.py:232-236
                for (int i = fb; i < lb && all_label; ++i) all_label = (s_cls[s[i]] & CC_LABEL) != 0;
                if (all_label) kind = LK_LABEL;
              }
            }
            if (lane == end_lane) kind = LK_COMPLEX;
            // ---- structure of the line if it starts outside a statement ----
            LineSummary sm;
            sm.nonblank = kind != LK_BLANK; sm.has_semi = kind == LK_STMT;
            sm.pend_out0 = sm.defer = sm.unterminated = false;
            sm.n0 = kind == LK_STMT ? 1 : 0; sm.n_after = 0;
            sm.lab0 = kind == LK_LABEL ? 1 : 0; sm.lab_after = 0; sm.dcl0 = sm.dcl_after = 0;
            if (mine && kind == LK_COMPLEX) sm = walk_line<0>(s, b, e, false, hi, d_in, at_seg_end, em);
            // pending map: f0 = state after the line when it starts clean, f1 = when it starts
            // inside a statement; blank lines are the identity (ptx.py:230 `while line`)
            unsigned f0 = 0, f1 = 1;
            if (mine && sm.nonblank) { f0 = sm.pend_out0 ? 1u : 0u; f1 = sm.has_semi ? f0 : 1u; }
            unsigned m0 = f0, m1 = f1;          // inclusive composition over lanes 0..lane
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
              const unsigned o0 = __shfl_up_sync(kFull, m0, dd), o1 = __shfl_up_sync(kFull, m1, dd);
              if (lane >= dd) { const unsigned t0 = o0 ? m1 : m0, t1 = o1 ? m1 : m0; m0 = t0; m1 = t1; }
            }
            unsigned e0 = __shfl_up_sync(kFull, m0, 1), e1 = __shfl_up_sync(kFull, m1, 1);
            if (lane == 0) { e0 = 0; e1 = 1; }
            const bool p_in = pending ? (e1 != 0) : (e0 != 0);
            // the statement a line opens is only real if the line's tail is reached outside a
            // statement: always after a ';', otherwise only when the line starts clean
            const bool tail_real = mine && (!p_in || sm.has_semi);
            const unsigned defer_mask = __ballot_sync(kFull, tail_real && sm.defer);
            const int defer_lane = defer_mask ? __ffs((int)defer_mask) - 1 : 32;
            const bool run_line = mine && lane < defer_lane;
            const bool bad = run_line && tail_real && sm.unterminated;
            int n_ins = 0, n_lab = 0, n_dcl = 0;
            if (run_line) {
              if (p_in) { if (sm.has_semi) { n_ins = sm.n_after; n_lab = sm.lab_after; n_dcl = sm.dcl_after; } }
              else { n_ins = sm.n0; n_lab = sm.lab0; n_dcl = sm.dcl0; }
            }
            int tot_ins = 0, tot_lab = 0, tot_dcl = 0;
            const int ins_ex = warp_excl_sum(n_ins, &tot_ins);
            const int lab_ex = warp_excl_sum(n_lab, &tot_lab);
            const int dcl_ex = warp_excl_sum(n_dcl, &tot_dcl);
            // ---- main walk ----
            {
              const int64_t ins0 = em.ins_at, lab0 = em.lab_at;
              const int dcl0 = em.dcl_at;
              em.ins_at = ins0 + ins_ex; em.lab_at = lab0 + lab_ex; em.dcl_at = dcl0 + dcl_ex;
              em.line = line_no + (uint32_t)li;
              if (run_line) {
                if (p_in || kind == LK_COMPLEX) walk_line<kMain>(s, b, e, p_in, hi, d_in, at_seg_end, em);
                else if (kind == LK_STMT) do_statement<kMain>(s, fb, lb, em);
                else if (kind == LK_LABEL) {
                  if (kMain == 2) {
                    FfbLabelRec L;
                    L.hash = norm_hash(s, fb, lb); L.index = (uint32_t)(em.ins_at - a.ins_base[seg]);
                    L.off = (uint32_t)(abase + fb - seg_begin);
                    if (em.lab_at < em.lab_limit) a.labels[em.lab_at] = L;
                  }
                }
              }
              em.ins_at = ins0 + tot_ins; em.lab_at = lab0 + tot_lab; em.dcl_at = dcl0 + tot_dcl;
            }
            n_instr += (uint32_t)tot_ins; n_labels += (uint32_t)tot_lab; n_decls += (uint32_t)tot_dcl;
            if (__any_sync(kFull, bad)) { status = FFB_E_MALFORMED_PTX; break; }   // ptx.py:272-273
            // ---- carry ----
            if (defer_lane < 32) {
              const int keep = l0 + defer_lane;          // lines consumed by this tile
              if (keep == 0) { status = FFB_E_CAPACITY; break; }     // statement longer than the tile
              if (defer_lane > 0) {
                const unsigned pm0 = __shfl_sync(kFull, m0, defer_lane - 1), pm1 = __shfl_sync(kFull, m1, defer_lane - 1);
                pending = pending ? (pm1 != 0) : (pm0 != 0);
              }
              depth = __shfl_sync(kFull, d_in, defer_lane);
              consume_to = (nl[keep - 1] & 0x7fff) + 1;
              // the deferred line may be the one holding the opening brace
              if (body_pos_g > abase + consume_to) { /* resume position already recorded */ }
              break;
            }
            const int last_lane = end_lane < 32 ? end_lane : min(31, n_lines - 1 - l0);
            {
              const unsigned pm0 = __shfl_sync(kFull, m0, last_lane), pm1 = __shfl_sync(kFull, m1, last_lane);
              pending = pending ? (pm1 != 0) : (pm0 != 0);
            }
            if (end_lane < 32) {
              phase = PH_DONE;
              body_end_off = abase + __shfl_sync(kFull, close_at, end_lane) - seg_begin;
              break;
            }
            depth += tot_delta;
            pos = lo;
          }
        }
      }
      if (status != FFB_OK) break;
      if (phase == PH_DONE) break;

      // ================= advance =================
      int nlc = 0;
      for (int l = lane; l < n_real; l += 32) nlc += ((nl[l] & 0x7fff) < consume_to) ? 1 : 0;
      nlc = (int)warp_sum_u64((unsigned long long)nlc);
      cm_state = S_CODE;
      if (nlc > 0) {
        const unsigned last = nl[nlc - 1];
        if ((int)(last & 0x7fff) == consume_to - 1 && (last & 0x8000)) cm_state = S_BLK;
      }
      line_no += (uint32_t)nlc;
      const int64_t next = abase + consume_to;
      if (next <= cur) { status = FFB_E_CAPACITY; break; }
      cur = next;
    }

    // ================= segment epilogue =================
    if (status == FFB_OK) {
      if (phase == PH_SEARCH) status = FFB_E_NO_KERNEL;                                // ptx.py:186-187
      else if (phase == PH_HEADER || phase == PH_BODY) status = FFB_E_MALFORMED_PTX;   // :175, :184
      else if (pending) status = FFB_E_MALFORMED_PTX;                                  // :272-273
      else if (n_instr == 0) status = FFB_E_MALFORMED_PTX;                             // :274-275
    }
    if (kRecords && status == FFB_OK && ((a.ins_cap && (int64_t)n_instr > a.ins_cap[seg]) || (a.lab_cap && (int64_t)n_labels > a.lab_cap[seg])))
      status = FFB_E_CAPACITY;            // single-pass mode: the segment outgrew its record slots
    uint32_t tot[FFB_N_CLASSES];
#pragma unroll
    for (int c = 0; c < FFB_N_CLASSES; ++c) {
      const uint64_t word = c < 3 ? em.c0 : (c < 6 ? em.c1 : em.c2);
      tot[c] = (uint32_t)warp_sum_u64((word >> (21 * (c % 3))) & 0x1fffffull);
    }
    const unsigned long long sh = warp_sum_u64(em.shared_bytes), rg = warp_sum_u64(em.regs);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < FFB_N_CLASSES; ++c) a.hist[seg * FFB_N_CLASSES + c] = tot[c];
      FfbSegInfo inf;
      inf.status = status; inf.n_instr = n_instr; inf.n_labels = n_labels; inf.n_decls = n_decls;
      inf.static_shared = sh; inf.regs_declared = rg;
      inf.name_off = (uint32_t)name_off; inf.name_len = (uint32_t)name_len;
      inf.body_off = (uint32_t)(body_pos_g ? body_pos_g - seg_begin : 0); inf.body_end = (uint32_t)body_end_off;
      a.info[seg] = inf;
    }
  }
}

// Batch classifier: one thread per opcode string (ptx.py:99-136 and :64-76 as pure functions).
__global__ void __launch_bounds__(256)
classify_opcodes_kernel(const uint8_t* text, const int64_t* off, int64_t n, uint32_t* out) {
  __shared__ uint64_t s_tok_key[256];
  __shared__ uint32_t s_tok_val[256];
  s_tok_key[threadIdx.x] = ~0ull; s_tok_val[threadIdx.x] = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < kNumTokDefs; c += 256) {
    const uint32_t slot = (uint32_t)((kTokDefs[c].key * kTokMul) >> 56);
    s_tok_key[slot] = kTokDefs[c].key; s_tok_val[slot] = kTokDefs[c].val;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  TokTable tt; tt.key = s_tok_key; tt.val = s_tok_val;
  const int64_t b = off[i], e = off[i + 1];
  const OpcodeInfo oc = classify_opcode(tt, text + b, 0, (int)(e - b));
  out[3 * i] = oc.cls; out[3 * i + 1] = oc.space; out[3 * i + 2] = oc.bytes;
}

}  // namespace

extern "C" int32_t ffb_classify_opcodes(FfbContext* ctx, const uint8_t* d_text, const int64_t* d_off, int64_t n,
                                        uint32_t* d_out, void* stream) {
  if (!ctx || !d_text || !d_off || !d_out || n < 0) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_classify_opcodes: bad argument");
  if (n == 0) return FFB_OK;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));
  FFB_LAUNCH(classify_opcodes_kernel, (unsigned)((n + 255) / 256), 256, 0, stream, d_text, d_off, n, d_out);
  return ffb_check_launch(ctx, "classify_opcodes_kernel");
}

namespace {
}  // namespace

extern "C" int32_t ffb_lex_corpus(FfbContext* ctx, const FfbLexDesc* d, void* stream_) {
  if (!ctx || !d || !d->d_text || !d->d_seg_off || !d->d_hist || !d->d_info || d->n_segs < 0)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: bad argument");
  if (d->n_bytes % 16 != 0)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: n_bytes must be the padded size (multiple of 16)");
  if (d->n_segs == 0) return FFB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));
  int32_t rc = ffb_reserve(ctx, &ctx->d_lex, 4096);
  if (rc) return rc;
  LexArgs a = {};
  a.text = d->d_text; a.n_bytes = d->n_bytes; a.seg_off = d->d_seg_off; a.n_segs = d->n_segs;
  a.order = d->d_order; a.work = (unsigned long long*)ctx->d_lex.p;
  a.hist = d->d_hist; a.info = d->d_info;
  a.ins_base = d->d_ins_base; a.lab_base = d->d_lab_base; a.ins_cap = d->d_ins_cap; a.lab_cap = d->d_lab_cap;
  a.ins = (FfbInsRec*)d->d_ins; a.labels = (FfbLabelRec*)d->d_labels;
  a.spans = d->d_spans; a.decls = d->d_decls; a.meta = d->d_meta;
  a.want_name = nullptr; a.want_len = 0;
  if (d->h_kernel_name && d->kernel_name_len > 0) {
    if (d->kernel_name_len > 2048) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: kernel name too long");
    rc = ffb_stage_reserve(ctx, (size_t)d->kernel_name_len);
    if (rc) return rc;
    memcpy(ctx->h_stage, d->h_kernel_name, (size_t)d->kernel_name_len);
    uint8_t* dn = (uint8_t*)ctx->d_lex.p + 64;
    FFB_CUDA(ctx, cudaMemcpyAsync(dn, ctx->h_stage, (size_t)d->kernel_name_len, cudaMemcpyHostToDevice, stream));
    FFB_CUDA(ctx, cudaEventRecord(ctx->stage_free, stream));
    ctx->stage_busy = true;
    a.want_name = dn; a.want_len = d->kernel_name_len;
  }
  const bool records = d->d_ins != nullptr;
  if (records && (!d->d_ins_base || !d->d_lab_base || !d->d_labels))
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: record mode needs ins/label buffers and their bases");
  FFB_CUDA(ctx, cudaMemsetAsync(a.work, 0, 8, stream));
  const size_t smem = (size_t)kWarps * kWarpSmem;
  int64_t ctas = (d->n_segs + kWarps - 1) / kWarps;
  const int64_t max_ctas = (int64_t)ctx->sm_count * 4;
  if (ctas > max_ctas) ctas = max_ctas;
  if (records) {
    FFB_CUDA(ctx, cudaFuncSetAttribute(lex_corpus_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FFB_LAUNCH(lex_corpus_kernel<true>, (unsigned)ctas, kWarps * 32, smem, stream, a);
  } else {
    FFB_CUDA(ctx, cudaFuncSetAttribute(lex_corpus_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FFB_LAUNCH(lex_corpus_kernel<false>, (unsigned)ctas, kWarps * 32, smem, stream, a);
  }
  return ffb_check_launch(ctx, "lex_corpus_kernel");
}
