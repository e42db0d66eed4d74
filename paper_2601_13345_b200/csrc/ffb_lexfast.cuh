// K1 fast path: byte-parallel lexer for REGULAR segments, with a device-side hand-over of
// everything else to the exact walk in ffb_lex.cu (same results either way; a segment is
// finished by exactly one of the two kernels).
//
// "Regular" is what compilers emit and what the reference's parse_ptx (ptx.py:207-293) handles
// without its `pending` machinery: 7-bit text whose only blanks are ' ' '\t' '\r' '\n', no "/*"
// anywhere before the end of the kernel body, and body lines that are - after cutting a
// trailing "// ..." comment (ptx.py:141) - one of
//     blank | `name:` | bare `{` / `}` | `.directive [;]` | `[@p] opcode operands ;`
// with braces inside a statement balanced.  Anything else (multi-line statements, several
// statements on a line, label + statement on one line, block comments, CR/LF, a kernel name
// filter ...) marks the segment; marked segments are appended to a work list that the exact
// kernel consumes in the same stream.  No host round trip, no CPU path.
//
// One warp per segment (dynamic queue), 4 KB tiles:
//   M  each lane loads coalesced 16-byte units and, still in registers, derives 16-bit position
//      masks by SWAR (newline, ';', "rare" = ':' '{' '}' '/', blank, '.', and in record mode
//      ',' and opening / closing brackets) plus a reject flag for bytes outside the regular
//      alphabet; text and masks go to shared memory (conflict-free 16 B / 2 B stores);
//   T  lane L owns mask words 4L..4L+3: popcounts + one warp scan give the newline table and
//      per-word prefix counts, so "how many ';' / rare bytes in [b,e)" is two rank queries;
//   S  `.entry NAME` and the opening '{' by warp-min over mask bits (ptx.py:165-176);
//   P1 one lane per line: rank queries split lines into plain and careful (any rare byte);
//      plain lines are classified from first/last byte and the ';' count;
//      careful lines are compacted and resolved 32 at a time, visiting only their rare bytes
//      (comment cut, label, braces); a warp scan of the brace deltas finds the line that closes
//      the body;
//   P2 one lane per statement, parsed from 64-bit windows of the masks: predicate, opcode
//      tokens (packed words, perfect-hash table), top-level commas, operand spans; operands,
//      addresses and literals are described from packed 16-byte loads.  Statements the windows
//      cannot express are compacted and take the byte-serial do_statement of the exact kernel.
//      Record slots come from ballots, not atomics.
// Both modes run as ONE barrier-paced CTA per SM (kLockstep): the warps of a scheduler then run the
// same phase of this long loop together and share fetched instruction lines.
#pragma once
#include "ffb_lex_shared.cuh"

namespace {

#ifdef FFB_SIMT_EMUL
#define FFB_PREFETCH_L2(p) ((void)(p))
#else
#define FFB_PREFETCH_L2(p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p))
#endif
#ifndef FFB_LEX_PREFETCH
#define FFB_LEX_PREFETCH 1
#endif
constexpr bool kPrefetch = FFB_LEX_PREFETCH != 0;
constexpr int kFWarps = 4;
#ifndef FFB_LEX_REC_CTAS
#define FFB_LEX_REC_CTAS 1                       // barrier-paced record-mode CTAs per SM (16 warps per SM in all)
#endif
constexpr int kFRecCtasPerSm = FFB_LEX_REC_CTAS;
constexpr int kFRecLockWarps = 16 / kFRecCtasPerSm;   // warps of the barrier-paced record-mode CTA
constexpr int kFTile = 4096;
constexpr int kFPad = 64;
constexpr int kFWords = kFTile / 32;              // 32-byte mask words per tile
constexpr int kFMaxLines = 256;
// per-warp shared memory (byte offsets)
constexpr int kFOffNlm = kFTile + kFPad;                        // u32[128] newline mask; later u16[256] careful / slow lists
constexpr int kFOffMA = kFOffNlm + kFWords * 4;                 // uint4[128 + 4] {semi, rare, blank, dot} per 32-byte word (+ zero sentinels)
constexpr int kFOffP = kFOffMA + (kFWords + 4) * 16;            // u32[128 + 4] prefix counts (semi | rare << 16) + total
constexpr int kFOffNl = kFOffP + (kFWords + 4) * 4;             // u16[kFMaxLines + 8] newline positions
constexpr int kFOffInfo = kFOffNl + (kFMaxLines + 8) * 2;       // u32[kFMaxLines] line info
constexpr int kFOffMB = kFOffInfo + kFMaxLines * 4;             // record mode: uint4[128 + 4] {comma, bracket, bracket out of turn, parity} (+ zero sentinels)
constexpr int kFWarpSmemHist = kFOffMB;
constexpr int kFWarpSmemRec = kFOffMB + (kFWords + 4) * 16;
static_assert(kFWarpSmemHist % 16 == 0 && kFWarpSmemRec % 16 == 0 && kFOffNlm % 16 == 0 && kFOffMA % 16 == 0 && kFOffP % 16 == 0 &&
              kFOffInfo % 16 == 0 && kFOffMB % 16 == 0, "smem layout");

enum { FK_BLANK = 0, FK_STMT, FK_LABEL, FK_DIR, FK_DECL, FK_OPEN, FK_CLOSE, FK_BAD };
constexpr uint32_t kH80 = 0x80808080u;

FFB_D uint32_t fk_pack(int kind, int b, int e) { return (uint32_t)b | ((uint32_t)e << 13) | ((uint32_t)kind << 26); }

// bit 7 of every byte that DIFFERS from the replicated byte c4 (exact for 7-bit text; a byte
// >= 0x80 may disturb its neighbour, such tiles are rejected before the masks are used)
FFB_D uint32_t ne80(uint32_t w, uint32_t c4) { return (w ^ c4) + 0x7f7f7f7fu; }
// four words of bit-7 flags -> 16 dense bits (bit 4j+k <-> byte k of word j)
FFB_D uint32_t pack16(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  const uint32_t q01 = (m0 >> 7) | (m1 >> 3), q23 = (m2 >> 7) | (m3 >> 3);
  return ((q01 * 0x01020408u) >> 24) | (((q23 * 0x01020408u) >> 16) & 0xff00u);
}

// 8 x 8 bit-matrix transpose of the eight bytes (lo, hi): afterwards bit r of byte c is bit c of input byte r
// (three delta swaps, Hacker's Delight 7-3, on the two 32-bit halves)
FFB_D void transpose8x8(uint32_t& lo, uint32_t& hi) {
  uint32_t t;
  t = (lo ^ (lo >> 7)) & 0x00aa00aau; lo ^= t ^ (t << 7);
  t = (hi ^ (hi >> 7)) & 0x00aa00aau; hi ^= t ^ (t << 7);
  t = (lo ^ (lo >> 14)) & 0x0000ccccu; lo ^= t ^ (t << 14);
  t = (hi ^ (hi >> 14)) & 0x0000ccccu; hi ^= t ^ (t << 14);
  t = (lo ^ __funnelshift_r(lo, hi, 28)) & 0xf0f0f0f0u;
  lo ^= t ^ (t << 28); hi ^= t >> 4;
}

// number of ';' (low half) and rare bytes (high half) at tile positions < x
FFB_D uint32_t rank2(const uint4* MA, const uint32_t* P, int x) {
  const int w = x >> 5;
  const uint32_t low = (1u << (x & 31)) - 1u;
  const uint2 m = *reinterpret_cast<const uint2*>(MA + w);
  return P[w] + (uint32_t)__popc(m.x & low) + ((uint32_t)__popc(m.y & low) << 16);
}

// ---- bit-window statement parser ----------------------------------------------------------------
// A statement of at most 64 bytes is parsed from 64-bit windows of the tile masks: bit i of a
// window is the class of byte kb + i.  Everything the windows cannot express exactly (longer
// statements, nested brackets, empty operands, odd predicates) returns false and goes through
// do_statement, the byte-serial walk shared with the exact kernel.
FFB_D uint64_t win64(uint32_t a, uint32_t b, uint32_t c, int sh) {
  return (uint64_t)__funnelshift_r(a, b, sh) | ((uint64_t)__funnelshift_r(b, c, sh) << 32);
}
FFB_D uint64_t low_mask(int n) { return n >= 64 ? ~0ull : ((1ull << n) - 1ull); }      // bits [0, n), 0 <= n
FFB_D uint64_t high_mask(int n) { return n >= 64 ? 0ull : (~0ull << n); }              // bits [n, 64), 0 <= n
FFB_D uint64_t range_mask(int lo, int hi) {                                            // bits [lo, hi) of a window, any ints
  lo = lo < 0 ? 0 : lo; hi = hi > 64 ? 64 : hi;
  return lo >= hi ? 0ull : (low_mask(hi) & high_mask(lo));
}
FFB_D uint64_t prefix_xor64(uint64_t x) {
  x ^= x << 1; x ^= x << 2; x ^= x << 4; x ^= x << 8; x ^= x << 16; x ^= x << 32;
  return x;
}
// s[p, p+len) as a little-endian u64, len <= 8 (three aligned word loads, no byte loop)
FFB_D uint64_t load_packed(const uint8_t* s, int p, int len) {
  if (len <= 0) return 0ull;
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(s + (p & ~3));
  const uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2];
  const int sh = (p & 3) * 8;
  uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
  if (len <= 4) { hi = 0u; lo &= 0xffffffffu >> (32 - 8 * len); }
  else hi &= 0xffffffffu >> (64 - 8 * len);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

// ---- cold paths, kept OUT of line -----------------------------------------------------------------
// The hot loop has to fit the instruction cache (the first version of this kernel inlined every
// byte-serial helper several times, grew to 17 K instructions and spent 80% of its issue slots
// waiting for instruction fetch, ncu r1l).  Everything rare is a real call: arguments by value,
// results in registers, so that no hot variable is forced into local memory.
#define FFB_NOINLINE __device__ __noinline__
FFB_NOINLINE uint64_t cold_norm_hash(const uint8_t* s, int a, int b) { return norm_hash(s, a, b); }
FFB_NOINLINE uint64_t cold_describe_operand(const uint8_t* s, int a, int b) { return describe_operand(s, a, b); }
struct AddrDesc { uint64_t desc; uint32_t kind; };
FFB_NOINLINE AddrDesc cold_describe_address(const uint8_t* s, int a, int b) {
  AddrDesc r;
  r.kind = describe_address(s, a, b, &r.desc);
  return r;
}
struct DeclResult { unsigned long long regs, shared; int n_reg_decl; };
FFB_NOINLINE DeclResult cold_directive(const uint8_t* s, int b, int e) {
  DeclResult r;
  r.regs = 0; r.shared = 0; r.n_reg_decl = 0;
  while (e > b && ffb_is_ws(s[e - 1])) --e;
  uint64_t n = 0, bytes = 0;
  int c0 = 0, c1 = 0;
  if (parse_reg_decl(s, b, e, &n, &c0, &c1)) { r.regs = n; r.n_reg_decl = 1; }
  else if (parse_shared_decl(s, b, e, &bytes)) r.shared = bytes;
  return r;
}
// the byte-serial statement walk of the exact kernel; returns the opcode class
template <int kMode>
FFB_NOINLINE uint32_t cold_statement(const LexArgs* a, const uint64_t* tok_key, const uint32_t* tok_val, const uint8_t* cls,
                                     const uint8_t* s, int kb, int ke, long long ins_at, long long ins_limit, uint32_t line,
                                     long long abase, long long seg_begin) {
  Emit em;
  em.a = a; em.seg = 0; em.seg_begin = seg_begin; em.abase = abase; em.line = line;
  em.tok.key = tok_key; em.tok.val = tok_val; em.cls = cls;
  em.ins_at = ins_at; em.lab_at = 0; em.ins_limit = ins_limit; em.lab_limit = 0; em.dcl_at = 0;
  em.c0 = em.c1 = em.c2 = 0; em.shared_bytes = 0; em.regs = 0;
  do_statement<kMode>(s, kb, ke, em);
  const uint64_t w = em.c0 ? em.c0 : (em.c1 ? em.c1 : em.c2);
  return (em.c0 ? 0u : (em.c1 ? 3u : 6u)) + ((w >> 42) ? 2u : ((w >> 21) ? 1u : 0u));
}

// s[p, p+len) as two little-endian u64, 1 <= len <= 16 (five aligned word loads)
FFB_D void load_packed16(const uint8_t* s, int p, int len, uint64_t* lo, uint64_t* hi) {
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(s + (p & ~3));
  const uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2], w3 = wp[3], w4 = wp[4];
  const int sh = (p & 3) * 8;
  const uint64_t l = (uint64_t)__funnelshift_r(w0, w1, sh) | ((uint64_t)__funnelshift_r(w1, w2, sh) << 32);
  const uint64_t h = (uint64_t)__funnelshift_r(w2, w3, sh) | ((uint64_t)__funnelshift_r(w3, w4, sh) << 32);
  if (len <= 8) { *lo = l & low_mask(8 * len); *hi = 0ull; }
  else { *lo = l; *hi = h & low_mask(8 * (len - 8)); }
}
// the last k (<= 8) bytes of the first `len` (>= k) bytes of the packed pair
FFB_D uint64_t packed_tail(uint64_t lo, uint64_t hi, int len, int k) {
  const int sh = 8 * (len - k);
  const uint64_t v = sh == 0 ? lo : (sh >= 64 ? hi >> (sh - 64) : (lo >> sh) | (hi << (64 - sh)));
  return v & low_mask(8 * k);
}
// name hash of s[a,b) when the span holds no newline (every statement of the fast path sits on one
// line, so norm_hash's blank-run rule never fires): 8-byte chunks straight from packed loads
FFB_D uint64_t hash_bytes(const uint8_t* s, int a, int len) {
  uint64_t h = kHashBasis;
#pragma unroll 1
  for (int off = 0; off < len; off += 8) h = ffb_hash_chunk(h, load_packed(s, a + off, len - off < 8 ? len - off : 8));
  return ffb_hash_fold(h ^ (uint64_t)(uint32_t)len);
}
FFB_D uint64_t hash_span(const uint8_t* s, int a, int b) {
  if (b <= a) return cold_norm_hash(s, a, b);
  if (b - a > 16) return hash_bytes(s, a, b - a);
  uint64_t lo, hi;
  load_packed16(s, a, b - a, &lo, &hi);
  return ffb_hash_packed(lo, hi, (uint32_t)(b - a));
}

// describe_operand (alignment.py:31-47, cfg.py:184-188) for operands of at most 16 bytes, from two
// packed words: same descriptor, no byte loops.  The few shapes that need Python's full int(text, 0)
// grammar (prefixed or '_'-separated literals) and longer operands use describe_operand itself.
FFB_D uint64_t describe_fast(const uint8_t* s, int a, int b) {
  const int len = b - a;
  if (len > 16) {
    // long operands are vector lists and symbols; registers and numbers this long take the byte walk
    const unsigned f = s[a];
    if (f == '%' || f == '+' || f == '-' || ffb_is_digit(f)) return cold_describe_operand(s, a, b);
    return ffb_op_make(FFB_OPK_UNIFORM, hash_bytes(s, a, len));
  }
  uint64_t lo, hi;
  load_packed16(s, a, len, &lo, &hi);
  const uint64_t h = ffb_hash_packed(lo, hi, (uint32_t)len);
  const unsigned c0 = (unsigned)(lo & 0xffu);
  if (c0 == '%') {
    // special registers start with %t %l %w %g %n, or are long enough to END in "%gridid" / "WARP_SZ" / "%ctaid.x"
    const unsigned c1 = (unsigned)((lo >> 8) & 0xffu) - 'a';
    if (len < 8 && !(c1 < 26u && ((1u << c1) & ((1u << ('t' - 'a')) | (1u << ('l' - 'a')) | (1u << ('w' - 'a')) | (1u << ('g' - 'a')) | (1u << ('n' - 'a'))))))
      return ffb_op_make(FFB_OPK_REG, h);
    if (len == 6 && lo == ffb_pk("%tid.x")) return ffb_op_make(FFB_OPK_TIDX, h);
    if ((len >= 5 && (lo & 0xffffffffffull) == ffb_pk("%tid.")) || (len == 7 && (lo == ffb_pk("%laneid") || lo == ffb_pk("%warpid"))))
      return ffb_op_make(FFB_OPK_UNKNOWN, h);
    bool uni = false;
    if (len >= 7) {
      const uint64_t t7 = packed_tail(lo, hi, len, 7);
      uni = t7 == ffb_pk("%gridid") || t7 == ffb_pk("WARP_SZ");
    }
    if (!uni && len >= 2) {
      const uint64_t t2 = packed_tail(lo, hi, len, 2);
      const unsigned ax = (unsigned)(t2 >> 8);
      if ((t2 & 0xffu) == '.' && (ax == 'x' || ax == 'y' || ax == 'z')) {
        const int L = len - 2;
        uni = (L >= 6 && packed_tail(lo, hi, L, 6) == ffb_pk("%ctaid")) || (L >= 7 && packed_tail(lo, hi, L, 7) == ffb_pk("%nctaid")) ||
              (L >= 5 && packed_tail(lo, hi, L, 5) == ffb_pk("%ntid"));
      }
    }
    return ffb_op_make(uni ? FFB_OPK_UNIFORM_REG : FFB_OPK_REG, h);
  }
  // Python int(text, 0)
  const bool sign = c0 == '+' || c0 == '-';
  const int m = len - (sign ? 1 : 0);
  if (m <= 0) return ffb_op_make(FFB_OPK_UNIFORM, h);
  uint64_t dl = lo, dh = hi;
  if (sign) { dl = (lo >> 8) | (hi << 56); dh = hi >> 8; }
  const unsigned d0 = (unsigned)(dl & 0xffu);
  if (!ffb_is_digit(d0)) return ffb_op_make(FFB_OPK_UNIFORM, h);
  constexpr uint64_t k30 = 0x3030303030303030ull, k76 = 0x7676767676767676ull, k80 = 0x8080808080808080ull,
                     k5f = 0x5f5f5f5f5f5f5f5full, k7f = 0x7f7f7f7f7f7f7f7full;
  const uint64_t pl = dl | (k30 & ~low_mask(8 * (m < 8 ? m : 8))), ph = dh | (k30 & ~low_mask(8 * (m > 8 ? m - 8 : 0)));
  const uint64_t nd = ((((pl ^ k30) + k76) | ((ph ^ k30) + k76)) | pl | ph) & k80;          // some byte is not 0-9
  if (nd) {
    const uint64_t other = (((pl ^ k30) + k76) & ((pl ^ k5f) + k7f)) | (((ph ^ k30) + k76) & ((ph ^ k5f) + k7f)) | pl | ph;
    const unsigned d1 = (unsigned)((dl >> 8) & 0xffu) | 32u;
    const bool prefixed = d0 == '0' && m >= 2 && (d1 == 'x' || d1 == 'o' || d1 == 'b');
    if (prefixed || !(other & k80)) return cold_describe_operand(s, a, b);    // 0x.. / 0o.. / 0b.. or digits with '_'
    return ffb_op_make(FFB_OPK_UNIFORM, h);                                // base 10 meets a foreign byte: not a literal
  }
  uint64_t v = 0;
  bool nonzero = false;
#pragma unroll 1
  for (int k = 0; k < m; ++k) {
    const unsigned d = (unsigned)(((k < 8 ? dl >> (8 * k) : dh >> (8 * (k - 8)))) & 0xfu);
    nonzero = nonzero || d != 0;
    v = v * 10u + d;
  }
  if (d0 == '0' && nonzero) return ffb_op_make(FFB_OPK_UNIFORM, h);       // "010": rejected by int(.., 0)
  const int64_t sv = c0 == '-' ? -(int64_t)v : (int64_t)v;
  return ffb_op_make(FFB_OPK_INT, (uint64_t)sv);
}

// describe_address (alignment.py:21) for the canonical shapes `[base]`, `[base+N]`, `[base+-N]` of at
// most 16 bytes without blanks or inner brackets (the caller checks those on the mask windows and
// that the operand starts with '[').  Returns false for anything else: the byte-serial version decides.
FFB_D bool address_fast(const uint8_t* s, int a, int b, uint32_t* kind, uint64_t* desc) {
  const int len = b - a;
  uint64_t lo, hi;
  load_packed16(s, a, len, &lo, &hi);
  if (packed_tail(lo, hi, len, 1) != ']') return false;
  constexpr uint64_t k80 = 0x8080808080808080ull, k7f = 0x7f7f7f7f7f7f7f7full, k2b = 0x2b2b2b2b2b2b2b2bull,
                     k30 = 0x3030303030303030ull, k76 = 0x7676767676767676ull;
  const uint64_t pl = ~((lo ^ k2b) + k7f) & k80, ph = ~((hi ^ k2b) + k7f) & k80;      // '+' bytes
  int plus = -1;
  if (pl) plus = (__ffsll((long long)pl) - 1) >> 3; else if (ph) plus = 8 + ((__ffsll((long long)ph) - 1) >> 3);
  const int base_end = plus >= 0 ? plus : len - 1;
  *desc = 0;
  if (base_end <= 1) { *kind = FFB_ADDR_NOMATCH; return true; }          // empty base
  if (plus >= 0) {                                                       // `+ -? digits` up to the bracket
    int d0 = plus + 1;
    const int sh0 = 8 * d0;
    const unsigned c = (unsigned)((sh0 >= 64 ? hi >> (sh0 - 64) : lo >> sh0) & 0xffu);
    if (c == '-') ++d0;
    const int m = len - 1 - d0;
    if (m <= 0) { *kind = FFB_ADDR_NOMATCH; return true; }
    const int sh = 8 * d0;                                               // digits start at byte d0 (1..15)
    const uint64_t dl = sh >= 64 ? hi >> (sh - 64) : (lo >> sh) | (hi << (64 - sh)), dh = sh >= 64 ? 0ull : hi >> sh;
    const uint64_t ml = low_mask(8 * (m < 8 ? m : 8)), mh = low_mask(8 * (m > 8 ? m - 8 : 0));
    const uint64_t ql = (dl & ml) | (k30 & ~ml), qh = (dh & mh) | (k30 & ~mh);
    if (((((ql ^ k30) + k76) | ((qh ^ k30) + k76)) | ql | qh) & k80) { *kind = FFB_ADDR_NOMATCH; return true; }
  }
  if (((lo >> 8) & 0xffu) != '%') { *kind = FFB_ADDR_SYMBOL; return true; }
  const int blen = base_end - 1;
  uint64_t bl = (lo >> 8) | (hi << 56), bh = hi >> 8;
  if (blen <= 8) { bl &= low_mask(8 * blen); bh = 0ull; } else bh &= low_mask(8 * (blen - 8));
  *desc = ffb_op_make(FFB_OPK_REG, ffb_hash_packed(bl, bh, (uint32_t)blen));
  *kind = FFB_ADDR_REG;
  return true;
}

// ---- opcode memo ----------------------------------------------------------------------------------
// PTX repeats a few hundred opcode strings ("ld.global.f32", "mad.lo.s32" ...).  classify_opcode
// (ptx.py:99-136) depends on that string alone, so every CTA keeps a table  text (compared exactly) ->
// opcode part of the meta word  in shared memory: a statement costs one probe instead of a token loop.
// Two tables: 256 slots of 32 B for opcodes of at most 24 bytes, 32 slots of 64 B for 25..56 bytes (mma / tex /
// wmma shapes); longer opcodes always take the token walk.
// The table is READ while tiles are parsed and WRITTEN only between two CTA barriers: a lane that misses
// classifies its opcode with the token walk and queues (key, value); behind the barrier that paces the tile loop
// every thread sees the queue length of the finished iteration (two queues, alternating, so nobody can be writing
// the one being read), one lane enters the queued opcodes, a second barrier ends the insert phase.  No atomics on
// the table, no fences, nothing for racecheck to flag - and 512 lanes missing `add.s32` at once leave one entry.
constexpr int kMemoSlots = 256, kMemoProbes = 8;
constexpr int kLongSlots = 32, kLongProbes = 4, kLongWords = 14;
constexpr int kPendMax = 32;                                    // queued inserts per iteration (more: retried later)
constexpr uint32_t kMemoValid = 1u << 31;
struct Memo {
  uint4* tab;                    // [2 * kMemoSlots] then the long table (uint32 [kLongSlots][16]); NULL: no memo (token walk only)
  uint32_t* pend;                // [kPendMax][16] queue of this iteration: 14 key words, value, length
  unsigned int* n_pend;
};
// packed key words of s[p, p+len): word i holds bytes 4i..4i+3, zero beyond len
FFB_D uint32_t key_word(const uint32_t* wp, int sh, int i, int q, uint32_t pm) {
  if (i > q) return 0u;
  const uint32_t v = __funnelshift_r(wp[i], wp[i + 1], sh);
  return i == q ? (v & pm) : v;
}
struct MemoKey { uint32_t k0, k1, k2, k3, k4, k5, slot; };
FFB_D void memo_key(const uint8_t* s, int p, int len, MemoKey& k) {          // 1 <= len <= 24
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(s + (p & ~3));
  const uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2], w3 = wp[3], w4 = wp[4], w5 = wp[5], w6 = wp[6];
  const int sh = (p & 3) * 8;
  const int q = len >> 2;
  const uint32_t pm = (1u << ((len & 3) * 8)) - 1u;
  uint32_t v;
  v = __funnelshift_r(w0, w1, sh); k.k0 = q > 0 ? v : (v & pm);
  v = __funnelshift_r(w1, w2, sh); k.k1 = q > 1 ? v : (q == 1 ? (v & pm) : 0u);
  v = __funnelshift_r(w2, w3, sh); k.k2 = q > 2 ? v : (q == 2 ? (v & pm) : 0u);
  v = __funnelshift_r(w3, w4, sh); k.k3 = q > 3 ? v : (q == 3 ? (v & pm) : 0u);
  v = __funnelshift_r(w4, w5, sh); k.k4 = q > 4 ? v : (q == 4 ? (v & pm) : 0u);
  v = __funnelshift_r(w5, w6, sh); k.k5 = q > 5 ? v : (q == 5 ? (v & pm) : 0u);
  uint32_t h = (k.k0 * 0x9e3779b1u) ^ (k.k1 * 0x85ebca77u) ^ (k.k2 * 0xc2b2ae3du) ^ (k.k3 * 0x27d4eb2fu) ^ (k.k4 * 0x165667b1u) ^ (k.k5 * 0xd3a2646du);
  h ^= h >> 15;
  k.slot = (h * 0x2c1b3c6du) >> 24;
}
FFB_D uint32_t memo_probe(const uint4* memo, const MemoKey& k) {             // value with kMemoValid set, or 0
  uint32_t sl = k.slot;
#pragma unroll 1
  for (int pr = 0; pr < kMemoProbes; ++pr) {
    const uint4 e1 = memo[2 * sl + 1];
    if (!(e1.z & kMemoValid)) break;                   // empty slot: the opcode is not in the table
    const uint4 e0 = memo[2 * sl];
    if (e1.x == k.k4 && e1.y == k.k5 && e0.x == k.k0 && e0.y == k.k1 && e0.z == k.k2 && e0.w == k.k3) return e1.z;
    sl = (sl + 1u) & (kMemoSlots - 1);
  }
  return 0u;
}
FFB_D uint32_t opcode_bits(const OpcodeInfo& oc) {     // the opcode's share of FfbInsRec.meta
  return oc.cls | (oc.space << 4) | ((oc.bytes & 63u) << 7) | (oc.base << 13) | (oc.cmp << 23);
}
FFB_D uint32_t long_hash(const uint32_t* wp, int sh, int q, uint32_t pm) {
  uint32_t h = 0x811c9dc5u;
#pragma unroll 1
  for (int i = 0; i <= q && i < kLongWords; ++i) h = (h ^ key_word(wp, sh, i, q, pm)) * 0x01000193u;
  h ^= h >> 15;
  return (h * 0x2c1b3c6du) >> 27;
}
// miss (or an opcode of 25..56 bytes): probe the long table if that is where it belongs, else the token walk of the
// exact kernel; the result is queued for the next insert phase
FFB_NOINLINE uint32_t cold_opcode(const uint64_t* tok_key, const uint32_t* tok_val, const uint8_t* s, int p0, int p1, const uint32_t* lmemo,
                                  uint32_t* pend, unsigned int* n_pend) {
  TokTable tt;
  tt.key = tok_key; tt.val = tok_val;
  const int len = p1 - p0;
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(s + (p0 & ~3));
  const int sh = (p0 & 3) * 8, q = len >> 2;
  const uint32_t pm = (1u << ((len & 3) * 8)) - 1u;
  if (lmemo && len > 24 && len <= 4 * kLongWords) {
    uint32_t sl = long_hash(wp, sh, q, pm);
#pragma unroll 1
    for (int pr = 0; pr < kLongProbes; ++pr) {
      const uint32_t* e = lmemo + 16 * sl;
      const uint32_t val = e[14];
      if (!(val & kMemoValid)) break;
      bool same = true;
#pragma unroll 1
      for (int i = 0; i < kLongWords && same; ++i) same = e[i] == key_word(wp, sh, i, q, pm);
      if (same) return val;
      sl = (sl + 1u) & (kLongSlots - 1);
    }
  }
  const uint32_t val = opcode_bits(classify_opcode(tt, s, p0, p1)) | kMemoValid;
  if (pend && len <= 4 * kLongWords) {
    const unsigned int at = atomicAdd(n_pend, 1u);
    if (at < (unsigned int)kPendMax) {
      uint32_t* e = pend + 16 * at;
#pragma unroll 1
      for (int i = 0; i < kLongWords; ++i) e[i] = key_word(wp, sh, i, q, pm);
      e[14] = val; e[15] = (uint32_t)len;
    }
  }
  return val;
}
// insert phase (one lane, between two CTA barriers): the queued opcodes enter their table unless already there
FFB_NOINLINE void memo_apply(uint4* tab, const uint32_t* pend, unsigned int n) {
  uint32_t* lmemo = reinterpret_cast<uint32_t*>(tab + 2 * kMemoSlots);
  for (unsigned int j = 0; j < n && j < (unsigned int)kPendMax; ++j) {
    const uint32_t* e = pend + 16 * j;
    const uint32_t val = e[14], len = e[15];
    if (len <= 24u) {
      uint32_t h = (e[0] * 0x9e3779b1u) ^ (e[1] * 0x85ebca77u) ^ (e[2] * 0xc2b2ae3du) ^ (e[3] * 0x27d4eb2fu) ^ (e[4] * 0x165667b1u) ^ (e[5] * 0xd3a2646du);
      h ^= h >> 15;
      uint32_t sl = (h * 0x2c1b3c6du) >> 24;
      for (int pr = 0; pr < kMemoProbes; ++pr) {
        const uint4 e1 = tab[2 * sl + 1], e0 = tab[2 * sl];
        if (!(e1.z & kMemoValid)) { tab[2 * sl] = make_uint4(e[0], e[1], e[2], e[3]); tab[2 * sl + 1] = make_uint4(e[4], e[5], val, 1u); break; }
        if (e1.x == e[4] && e1.y == e[5] && e0.x == e[0] && e0.y == e[1] && e0.z == e[2] && e0.w == e[3]) break;
        sl = (sl + 1u) & (kMemoSlots - 1);
      }
    } else {
      uint32_t h = 0x811c9dc5u;
      const int q = (int)(len >> 2);
      for (int i = 0; i <= q && i < kLongWords; ++i) h = (h ^ e[i]) * 0x01000193u;
      h ^= h >> 15;
      uint32_t sl = (h * 0x2c1b3c6du) >> 27;
      for (int pr = 0; pr < kLongProbes; ++pr) {
        uint32_t* d = lmemo + 16 * sl;
        if (!(d[14] & kMemoValid)) { for (int i = 0; i < kLongWords; ++i) d[i] = e[i]; d[14] = val; d[15] = len; break; }
        bool same = true;
        for (int i = 0; i < kLongWords && same; ++i) same = d[i] == e[i];
        if (same) break;
        sl = (sl + 1u) & (kLongSlots - 1);
      }
    }
  }
}
// opcode s[p0, p1) -> opcode bits of the meta word
FFB_D uint32_t opcode_of(const TokTable& tok, const Memo& memo, const uint8_t* s, int p0, int p1) {
  const int len = p1 - p0;
  uint32_t val = 0;
  if (memo.tab && len <= 24) {
    MemoKey k;
    memo_key(s, p0, len, k);
    val = memo_probe(memo.tab, k);
  }
  if (!val) val = cold_opcode(tok.key, tok.val, s, p0, p1, memo.tab ? reinterpret_cast<const uint32_t*>(memo.tab + 2 * kMemoSlots) : nullptr,
                              memo.pend, memo.n_pend);
  return val & ~kMemoValid;
}

template <int kMode>
FFB_D bool fast_statement(const uint8_t* s, const uint4* MA, const uint4* MB, const Memo& memo, int kb, int ke, Emit& em) {
  const int n = ke - kb;
  const int w0 = kb >> 5, sh = kb & 31;
  const uint64_t valid = low_mask(n);
  const uint64_t BL = win64(MA[w0].z, MA[w0 + 1].z, MA[w0 + 2].z, sh) & valid;
  // ---- predicate  ^@(!?%[\w$]+)\s+  (ptx.py:42) ----
  int o0 = 0, p0 = 0, p1 = 0;
  bool has_pred = false, neg = false;
  if (s[kb] == '@') {
    if (!BL) return false;
    const int t1 = __ffsll((long long)BL) - 1;
    int j = kb + 1;
    neg = s[j] == '!';
    if (neg) ++j;
    if (s[j] != '%' || kb + t1 <= j + 1) return false;
#pragma unroll 1
    for (int k = j + 1; k < kb + t1; ++k)
      if (!ffb_is_name_char(s[k])) return false;
    const uint64_t rest = ~BL & valid & high_mask(t1);
    if (!rest) return false;
    has_pred = true; p0 = j; p1 = kb + t1;
    o0 = __ffsll((long long)rest) - 1;
  }
  // ---- opcode tokens (ptx.py:99-136, :64-76) ----
  const uint64_t after = BL & high_mask(o0);
  if (!after && n > 64) return false;
  const int o1 = after ? __ffsll((long long)after) - 1 : n;
  uint32_t ob;
  if (kMode == 1) {
    // histogram mode needs the class only: the first token, whether the last one is "sync", and - for the
    // arithmetic bases and sqrt alone - the type / approx tokens in between (ptx.py:104-128).  Shorter than a
    // probe of the memo (measured: 481 vs 460 GB/s).
    uint64_t D = win64(MA[w0].w, MA[w0 + 1].w, MA[w0 + 2].w, sh) & valid & low_mask(o1) & high_mask(o0);
    uint32_t flags = 0;
    const int t0e = D ? __ffsll((long long)D) - 1 : o1;
    const int len0 = t0e - o0;
    const uint32_t base = (len0 > 8 ? 0u : tok_lookup(em.tok, load_packed(s, kb + o0, len0))) & 31u;
    if (D) {
      const int ld = 63 - __clzll((long long)D);
      if (o1 - ld - 1 == 4 && load_packed(s, kb + ld + 1, 4) == ffb_pk("sync")) flags |= 8u;
      constexpr uint32_t kScan = (1u << TB_ADD) | (1u << TB_SUB) | (1u << TB_MUL) | (1u << TB_MAD) | (1u << TB_FMA) | (1u << TB_DIV) | (1u << TB_SQRT);
      if ((kScan >> base) & 1u) {
        int ts = t0e + 1;
        D &= D - 1;
#pragma unroll 1
        for (;;) {
          const int te = D ? __ffsll((long long)D) - 1 : o1;
          const int len = te - ts;
          const uint32_t v = len > 8 ? 0u : tok_lookup(em.tok, load_packed(s, kb + ts, len));
          flags |= (v >> 8) & 3u;
          if (v & (1u << 16)) flags |= 4u;
          if (!D) break;
          D &= D - 1;
          ts = te + 1;
        }
      }
    }
    ob = finish_opcode(base, 0, 0, 0, 0, flags).cls;
  } else {
    // record mode: one probe of the CTA's opcode memo (ptx.py:99-136, :64-76)
    ob = opcode_of(em.tok, memo, s, kb + o0, kb + o1);
  }
  OpcodeInfo oc;
  oc.cls = ob & 15u; oc.space = (ob >> 4) & 7u; oc.bytes = (ob >> 7) & 63u; oc.base = (ob >> 13) & 31u; oc.cmp = (ob >> 23) & 7u;
  if (kMode == 2) {
    // ---- operands: top-level commas (ptx.py:144-162) ----
    // a second set of windows, anchored at the end of the opcode, so that the operand list may
    // itself be 64 bytes long (mma / tex / vector forms with a long opcode in front)
    const int ko = kb + o1, m = n - o1;
    if (m > 64) return false;
    // phase T left {commas, brackets, brackets out of turn, parity} in MB; the parity in front of the list is the
    // list's depth 0 (the kernel body itself sits inside a brace)
    uint64_t BO, CM, XX, BD, IN;
    {
      const int wo = ko >> 5, so = ko & 31;
      const uint64_t R = low_mask(m);
      const uint4 b0 = MB[wo], b1 = MB[wo + 1], b2 = MB[wo + 2];
      BO = win64(MA[wo].z, MA[wo + 1].z, MA[wo + 2].z, so) & R;
      CM = win64(b0.x, b1.x, b2.x, so) & R; XX = win64(b0.y, b1.y, b2.y, so) & R; BD = win64(b0.z, b1.z, b2.z, so) & R;
      IN = win64(b0.w, b1.w, b2.w, so);
    }
    const uint64_t NB = ~BO & low_mask(m);
    uint64_t inside = 0;
    if (XX) {                                         // brackets must alternate open / close (depth 0 or 1) and balance
      if ((IN ^ XX) & 1ull) { IN = ~IN; BD = XX & ~BD; }
      if (BD || ((IN >> (m - 1)) & 1ull)) return false;
      inside = IN;
    }
    const uint64_t C0 = CM & ~inside;
    const bool is_mem = oc.cls == FFB_CLS_MEMLOAD || oc.cls == FFB_CLS_MEMSTORE;
    const bool aux_is_op4 = !is_mem && oc.cls != FFB_CLS_BRANCH;
    FfbInsRec rec;
    rec.op[0] = rec.op[1] = rec.op[2] = rec.op[3] = 0; rec.aux = 0;
    int count = 0, as = -1, ae = -1, last_s = -1, last_e = -1;
    bool extra_reg = false, dst_reg = false;
    {
      uint64_t rem = C0, nb = NB;                     // commas and non-blank bytes not yet consumed
      for (;;) {
        const uint64_t below = (rem & (0ull - rem)) - 1ull;       // bits in front of the next comma (all bits when none is left)
        const uint64_t seg = nb & below;
        if (!seg) {
          if (C0) return false;                       // empty operand between commas: the walk drops it
          break;
        }
        const int a = ko + __ffsll((long long)seg) - 1, b = ko + 64 - __clzll((long long)seg);
        const unsigned c_first = s[a];
        if (count == 0) dst_reg = c_first == '%';
        if (count < 4 || (count == 4 && aux_is_op4)) {
          const uint64_t d = describe_fast(s, a, b);
          if (count == 0) rec.op[0] = d; else if (count == 1) rec.op[1] = d; else if (count == 2) rec.op[2] = d;
          else if (count == 3) rec.op[3] = d; else rec.aux = d;
        } else if (c_first == '%') extra_reg = true;
        if (is_mem && as < 0 && c_first == '[') { as = a; ae = b; }
        last_s = a; last_e = b;
        ++count;
        if (!rem) break;
        nb &= ~((below << 1) | 1ull);                 // drop the operand and its comma
        rem &= rem - 1;
      }
    }
    uint32_t addr_kind = FFB_ADDR_ABSENT;
    if (is_mem) {
      if (as >= 0) {
        const uint64_t span = low_mask(ae - ko) & high_mask(as - ko);
        const bool canonical = ae - as <= 16 && !(BO & span) && (XX & span) == ((1ull << (as - ko)) | (1ull << (ae - ko - 1)));
        if (!canonical || !address_fast(s, as, ae, &addr_kind, &rec.aux)) {
          const AddrDesc ad = cold_describe_address(s, as, ae);
          addr_kind = ad.kind; rec.aux = ad.desc;
        }
      }
    }
    else if (!aux_is_op4) rec.aux = last_s >= 0 ? ffb_op_make(FFB_OPK_REG, hash_span(s, last_s, last_e)) : 0ull;
    rec.line = em.line;
    rec.off = (uint32_t)(em.abase + kb - em.seg_begin);
    rec.len = (uint32_t)(NB ? o1 + 64 - __clzll((long long)NB) : o1);
    rec.pred = has_pred ? hash_span(s, p0, p1) : 0ull;
    rec.meta = ob | ((has_pred ? 1u : 0u) << 18) | ((neg ? 1u : 0u) << 19) | ((uint32_t)(count > 7 ? 7 : count) << 20) | (addr_kind << 26) |
               ((dst_reg ? 1u : 0u) << 28) | ((extra_reg ? 1u : 0u) << 29);
    if (em.ins_at < em.ins_limit) {
      em.a->ins[em.ins_at] = rec;
      if (em.a->meta) em.a->meta[em.ins_at] = rec.meta;
    }
  }
  const uint64_t inc = 1ull << (21 * (oc.cls % 3u));
  em.c0 += oc.cls < 3u ? inc : 0ull; em.c1 += (oc.cls >= 3u && oc.cls < 6u) ? inc : 0ull; em.c2 += oc.cls >= 6u ? inc : 0ull;
  return true;
}

// A line without rare bytes, or what is left of a careful one: s[b,e) holds no ':' and no
// comment; braces, if any, are balanced.  nsemi = number of ';' in it.
FFB_D int classify_plain(const uint8_t* s, int b, int e, int nsemi, int* kb, int* ke) {
  int fb = b;
#pragma unroll 1
  while (fb < e && s[fb] <= ' ') ++fb;
  if (fb >= e) return FK_BLANK;
  int lb = e - 1;
#pragma unroll 1
  while (s[lb] <= ' ') --lb;
  const unsigned c0 = s[fb];
  *kb = fb;
  if (c0 == '.') {                                               // ptx.py:240-256
    if (nsemi == 0) *ke = lb + 1;
    else if (nsemi == 1 && s[lb] == ';') *ke = lb;
    else return FK_BAD;                                          // text behind the first ';'
    const bool decl = (s[fb + 1] == 'r' && s[fb + 2] == 'e' && s[fb + 3] == 'g') ||
                      (s[fb + 1] == 's' && s[fb + 2] == 'h' && s[fb + 3] == 'a');
    return decl ? FK_DECL : FK_DIR;
  }
  if (nsemi != 1 || s[lb] != ';') return FK_BAD;                 // pending / several statements
  if (lb == fb) return FK_BLANK;                                 // a lone ';' (ptx.py:268-269)
  *ke = lb;
  return FK_STMT;
}

// A line with rare bytes.  s[b,e) is the raw line (scanned whole for "/*"), classification
// starts at bc >= b (the byte after the kernel's opening brace on that one line).  Only the rare
// bytes themselves are visited (bits of the line's window of the rare mask); the ';' count comes
// from the window of the ';' mask.  Lines longer than one window are walked byte by byte.
struct CarefulScan { int cut, ncolon, colon_at, nsemi, run, minrun, nbrace; bool ss; };
FFB_D void careful_visit(const uint8_t* s, int i, int bc, int e, CarefulScan& c) {
  const unsigned ch = s[i];
  if (ch == '/') {
    const unsigned c2 = s[i + 1];
    if (c2 == '*') c.ss = true;
    else if (c2 == '/' && c.cut == e) c.cut = i;
  }
  if (i >= bc && i < c.cut) {
    if (ch == ':') { if (c.ncolon++ == 0) c.colon_at = i; }
    else if (ch == '{') { ++c.run; ++c.nbrace; }
    else if (ch == '}') { --c.run; ++c.nbrace; if (c.run < c.minrun) c.minrun = c.run; }
  }
}
FFB_NOINLINE uint64_t careful_scan_bytes(const uint8_t* s, int b, int bc, int e) {     // long lines; returns the packed scan
  CarefulScan c;
  c.cut = e; c.ncolon = 0; c.colon_at = -1; c.nsemi = 0; c.run = 0; c.minrun = 0; c.nbrace = 0; c.ss = false;
  for (int i = b; i < e; ++i) careful_visit(s, i, bc, e, c);
  for (int i = bc; i < c.cut; ++i) c.nsemi += s[i] == ';' ? 1 : 0;
  // cut:13 | colon_at+1:13 | flags: ss, ncolon (0,1,2+), nsemi (0,1,2+), brace state (0 none, 1 balanced, 2 bad)
  const uint32_t bs = c.nbrace == 0 ? 0u : ((c.run == 0 && c.minrun >= 0) ? 1u : 2u);
  return (uint64_t)c.cut | ((uint64_t)(c.colon_at + 1) << 13) | ((c.ss ? 1ull : 0ull) << 26) | ((uint64_t)(c.ncolon > 2 ? 2 : c.ncolon) << 27) |
         ((uint64_t)(c.nsemi > 2 ? 2 : c.nsemi) << 29) | ((uint64_t)bs << 31);
}
FFB_D int resolve_careful(const uint8_t* s, const uint4* MA, int b, int bc, int e, int* kb, int* ke, bool* slashstar) {
  int cut, ncolon, colon_at, nsemi;
  bool braces, balanced;
  const int n = e - b;
  if (n <= 128) {                                                // one or two 64-byte windows
    CarefulScan c;
    c.cut = e; c.ncolon = 0; c.colon_at = -1; c.nsemi = 0; c.run = 0; c.minrun = 0; c.nbrace = 0; c.ss = false;
    uint64_t SW0 = 0, SW1 = 0;
#pragma unroll 1
    for (int wb = b; wb < e; wb += 64) {
      const int w0 = wb >> 5, sh = wb & 31, nn = e - wb;
      const uint4 a0 = MA[w0], a1 = MA[w0 + 1], a2 = MA[w0 + 2];
      uint64_t RW = win64(a0.y, a1.y, a2.y, sh) & low_mask(nn);
      const uint64_t SW = win64(a0.x, a1.x, a2.x, sh) & low_mask(nn);
      if (wb == b) SW0 = SW; else SW1 = SW;
#pragma unroll 1
      while (RW) {
        careful_visit(s, wb + __ffsll((long long)RW) - 1, bc, e, c);
        RW &= RW - 1;
      }
    }
    cut = c.cut; ncolon = c.ncolon; colon_at = c.colon_at;
    nsemi = __popcll(SW0 & range_mask(bc - b, cut - b)) + __popcll(SW1 & range_mask(bc - b - 64, cut - b - 64));
    braces = c.nbrace != 0; balanced = c.run == 0 && c.minrun >= 0;
    *slashstar = c.ss;
  } else {
    const uint64_t r = careful_scan_bytes(s, b, bc, e);
    cut = (int)(r & 0x1fffu); colon_at = (int)((r >> 13) & 0x1fffu) - 1;
    *slashstar = ((r >> 26) & 1u) != 0; ncolon = (int)((r >> 27) & 3u); nsemi = (int)((r >> 29) & 3u);
    braces = ((r >> 31) & 3u) != 0u; balanced = ((r >> 31) & 3u) == 1u;
  }
  int fb = bc;
#pragma unroll 1
  while (fb < cut && s[fb] <= ' ') ++fb;
  if (fb >= cut) return FK_BLANK;
  int lb = cut - 1;
#pragma unroll 1
  while (s[lb] <= ' ') --lb;
  *kb = fb;
  if (ncolon) {                                                  // ptx.py:232-236, label alone on its line
    if (ncolon != 1 || colon_at != lb || lb == fb) return FK_BAD;
#pragma unroll 1
    for (int i = fb; i < lb; ++i)
      if (!ffb_is_label_char(s[i])) return FK_BAD;
    *ke = lb;
    return FK_LABEL;
  }
  if (braces) {
    if (fb == lb) return s[fb] == '{' ? FK_OPEN : FK_CLOSE;      // ptx.py:237-239
    if (!balanced) return FK_BAD;
  }
  return classify_plain(s, fb, cut, nsemi, kb, ke);
}

// first set bit of the lane's four mask words at tile position >= from (and < lim) for which
// pred(pos) holds; 0x7fffffff if none
template <typename Pred>
FFB_D int lane_first(const uint32_t w[4], int lane, int from, int lim, Pred pred) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int base = lane * 128 + 32 * k;
    if (from >= base + 32) continue;
    uint32_t m = w[k];
    if (from > base) m &= 0xffffffffu << (from - base);
    while (m) {
      const int pos = base + __ffs((int)m) - 1;
      m &= m - 1;
      if (pos >= lim) return 0x7fffffff;
      if (pred(pos)) return pos;
    }
  }
  return 0x7fffffff;
}

FFB_D bool in_line_comment(const uint8_t* s, int at, int lo) {   // is a "//" open between the line start and `at`?
  for (int i = at - 1; i >= lo && s[i] != '\n'; --i)        // stops at the newline right before `at` too
    if (s[i] == '/' && s[i + 1] == '/') return true;
  return false;
}

// kLockstep: one CTA fills the SM and its warps meet at a barrier before every tile, so that the
// warps of a scheduler run the same phase of the (long) tile loop together and share fetched
// instruction lines; without it 70% of the issue slots of the record-mode kernel waited for
// instruction fetch (ncu r1o).
template <bool kRecords, bool kLockstep>
__global__ void __launch_bounds__(kLockstep ? (kRecords ? kFRecLockWarps * 32 : 768) : kFWarps * 32, kLockstep ? (kRecords ? kFRecCtasPerSm : 1) : (kRecords ? 4 : 6))
lex_fast_kernel(LexArgs a) {
  constexpr int kMain = kRecords ? 2 : 1;
  FFB_DYN_SMEM(smem_raw);
  __shared__ uint8_t s_cls[256];
  __shared__ uint64_t s_tok_key[256];
  __shared__ uint32_t s_tok_val[256];
  __shared__ uint4 s_memo[2 * kMemoSlots + 4 * kLongSlots];     // short-opcode table, then the long-opcode table
  __shared__ uint32_t s_pend[2][kPendMax * 16];                 // opcodes queued for the next insert phase (alternating)
  __shared__ unsigned int s_npend[2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint8_t* s = smem_raw + (size_t)wid * (kRecords ? kFWarpSmemRec : kFWarpSmemHist);
  uint32_t* NLM = reinterpret_cast<uint32_t*>(s + kFOffNlm);
  uint16_t* clist = reinterpret_cast<uint16_t*>(s + kFOffNlm);
  uint4* MA = reinterpret_cast<uint4*>(s + kFOffMA);
  uint4* MB = reinterpret_cast<uint4*>(s + kFOffMB);
  uint32_t* P = reinterpret_cast<uint32_t*>(s + kFOffP);
  uint16_t* nl = reinterpret_cast<uint16_t*>(s + kFOffNl);
  uint32_t* linfo = reinterpret_cast<uint32_t*>(s + kFOffInfo);
  for (int c = threadIdx.x; c < 256; c += (int)blockDim.x) { s_cls[c] = char_class((unsigned)c); s_tok_key[c] = ~0ull; s_tok_val[c] = 0; }
  for (int c = threadIdx.x; c < 2 * kMemoSlots + 4 * kLongSlots; c += (int)blockDim.x) s_memo[c] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x < 2) s_npend[threadIdx.x] = 0u;
  __syncthreads();
  for (int c = threadIdx.x; c < kNumTokDefs; c += (int)blockDim.x) {
    const uint32_t slot = (uint32_t)((kTokDefs[c].key * kTokMul) >> 56);
    s_tok_key[slot] = kTokDefs[c].key; s_tok_val[slot] = kTokDefs[c].val;
  }
  for (int i = lane; i < kFPad; i += 32) s[kFTile + i] = '\n';      // never overwritten
  if (lane < 4) {                                                   // windows and rank2(kFTile) read past the last word
    MA[kFWords + lane] = make_uint4(0u, 0u, 0u, 0u);
    if (kRecords) MB[kFWords + lane] = make_uint4(0u, 0u, 0u, 0u);
  }
  __syncthreads();

  // one segment in flight per warp; the loop below handles ONE tile per trip
  bool have = false, done = false, reject = false;
  int iter = 0;                                                    // trips of the tile loop: the same number in every thread of the CTA
  int64_t seg = 0, seg_begin = 0, seg_end = 0, cur = 0, scan_from_g = 0, body_pos_g = 0;
  int64_t name_off = 0, name_len = 0, body_end_off = 0, ins_base = 0, lab_base = 0;
  int phase = PH_SEARCH, depth = 0;
  uint32_t line_no = 1, n_instr = 0, n_labels = 0, n_decls = 0, n_slow_seg = 0;
  Emit em;
  em.a = &a; em.abase = 0; em.line = 0; em.dcl_at = 0;
  em.tok.key = s_tok_key; em.tok.val = s_tok_val; em.cls = s_cls;
  em.seg = 0; em.seg_begin = 0; em.ins_at = 0; em.lab_at = 0; em.ins_limit = 0; em.lab_limit = 0;
  em.c0 = em.c1 = em.c2 = 0; em.shared_bytes = 0; em.regs = 0;

  for (;;) {
    if (!have && !done) {
      unsigned long long wq = 0;
      if (lane == 0) wq = atomicAdd(a.work, 1ull);
      wq = __shfl_sync(kFull, wq, 0);
      if (wq >= (unsigned long long)a.n_segs) done = true;
      else {
        have = true;
        seg = a.order ? (int64_t)a.order[wq] : (int64_t)wq;
        seg_begin = a.seg_off[seg]; seg_end = a.seg_off[seg + 1];
        phase = PH_SEARCH; depth = 0; reject = false; line_no = 1;
        cur = seg_begin; scan_from_g = seg_begin; body_pos_g = 0;
        name_off = 0; name_len = 0; body_end_off = 0;
        n_instr = 0; n_labels = 0; n_decls = 0; n_slow_seg = 0;
        ins_base = kRecords ? a.ins_base[seg] : 0; lab_base = kRecords ? a.lab_base[seg] : 0;
        em.seg = seg; em.seg_begin = seg_begin; em.ins_at = ins_base; em.lab_at = lab_base;
        em.ins_limit = (kRecords && a.ins_cap) ? ins_base + a.ins_cap[seg] : 0x7fffffffffffffffLL;
        em.lab_limit = (kRecords && a.lab_cap) ? lab_base + a.lab_cap[seg] : 0x7fffffffffffffffLL;
        em.c0 = em.c1 = em.c2 = 0; em.shared_bytes = 0; em.regs = 0;
      }
    }
    if (kLockstep) {
      if (!__syncthreads_or(done ? 0 : 1)) break;
      if (kRecords) {
        // insert phase of the opcode memo: what the previous iteration queued (nobody writes that queue now)
        const int prev = (iter & 1) ^ 1;
        const unsigned int np = s_npend[prev];
        if (np) {
          if (threadIdx.x == 0) memo_apply(s_memo, s_pend[prev], np);
          __syncthreads();
          if (threadIdx.x == 0) s_npend[prev] = 0u;              // every thread has read the count; the queue refills after the NEXT barrier
        }
      }
    }
    else if (done) break;
    Memo memo;
    memo.tab = (kRecords && kLockstep) ? s_memo : nullptr;
    memo.pend = (kRecords && kLockstep) ? s_pend[iter & 1] : nullptr;
    memo.n_pend = &s_npend[iter & 1];
    ++iter;
    if (done) continue;                                          // idle warps keep meeting the barrier

    if (cur < seg_end) do {
      const int64_t abase = cur & ~(int64_t)15;
      const int64_t hi_g = (abase + kFTile < seg_end) ? abase + kFTile : seg_end;
      const int lo = (int)(cur - abase), hi = (int)(hi_g - abase);
      const bool at_seg_end = hi_g == seg_end;
      em.abase = abase;
      __syncwarp();

      // ================= M: load, masks, stage =================
      // the tile after this one starts its way from DRAM to L2 now (one 128-byte line per lane): all warps of the
      // barrier-paced CTA reach their loads together, nothing else hides that latency
      if (kPrefetch) {
        const int64_t pf = abase + kFTile + (int64_t)lane * 128;
        if (pf + 128 <= a.n_bytes && pf < seg_end) FFB_PREFETCH_L2(a.text + pf);
      }
      uint32_t badacc = 0;
#pragma unroll 1
      for (int v0 = 0; v0 < 8; v0 += 2) {                        // rolled on purpose: code size (see the note on cold paths)
        uint4 q[2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int64_t g = abase + (int64_t)((v0 + v) * 32 + lane) * 16;
          if (g + 16 <= a.n_bytes && g < hi_g) q[v] = *reinterpret_cast<const uint4*>(a.text + g);
          else q[v].x = q[v].y = q[v].z = q[v].w = 0x0a0a0a0au;
        }
        // Bit-sliced byte classes.  The 16 bytes of a unit are two 8 x 8 bit matrices; transposed, byte c of a
        // matrix holds bit c of its eight bytes.  Gathering byte c of the four matrices of the lane's two units
        // gives plane P[c] (bit i = bit c of byte i: bits 0-15 first unit, 16-31 second), and every class mask is
        // three-input logic on the eight planes - about a quarter of the instructions of testing each byte
        // against each character (the first version: 410 instructions per unit, 23% of the record-mode kernel).
        uint32_t keep[2], tl[2][2], th[2][2];                    // [unit][matrix]: transposed low / high words
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int u = (v0 + v) * 32 + lane, us = u * 16;
          uint32_t w[4] = {q[v].x, q[v].y, q[v].z, q[v].w};
          keep[v] = 0xffffu;
          if (us < lo || us + 16 > hi) {                         // unit straddles the tile's live range
            keep[v] = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int p = us + 4 * j + k;
                if (p >= lo && p < hi) keep[v] |= 1u << (4 * j + k);
                else w[j] = (w[j] & ~(0xffu << (8 * k))) | (0x0au << (8 * k));
              }
          }
          *reinterpret_cast<uint4*>(s + us) = make_uint4(w[0], w[1], w[2], w[3]);
          transpose8x8(w[0], w[1]);
          transpose8x8(w[2], w[3]);
          tl[v][0] = w[0]; th[v][0] = w[1]; tl[v][1] = w[2]; th[v][1] = w[3];
        }
        uint32_t P[8];
        {
          const uint32_t x0 = __byte_perm(tl[0][0], tl[0][1], 0x5140), y0 = __byte_perm(tl[0][0], tl[0][1], 0x7362);
          const uint32_t x1 = __byte_perm(tl[1][0], tl[1][1], 0x5140), y1 = __byte_perm(tl[1][0], tl[1][1], 0x7362);
          P[0] = __byte_perm(x0, x1, 0x5410); P[1] = __byte_perm(x0, x1, 0x7632);
          P[2] = __byte_perm(y0, y1, 0x5410); P[3] = __byte_perm(y0, y1, 0x7632);
          const uint32_t z0 = __byte_perm(th[0][0], th[0][1], 0x5140), r0 = __byte_perm(th[0][0], th[0][1], 0x7362);
          const uint32_t z1 = __byte_perm(th[1][0], th[1][1], 0x5140), r1 = __byte_perm(th[1][0], th[1][1], 0x7362);
          P[4] = __byte_perm(z0, z1, 0x5410); P[5] = __byte_perm(z0, z1, 0x7632);
          P[6] = __byte_perm(r0, r1, 0x5410); P[7] = __byte_perm(r0, r1, 0x7632);
        }
        // high nibble 0 / 2 / 3 / 5 / 7, low nibble 0 8 9 a b c d e f
        const uint32_t LOW = ~P[7] & ~P[6] & ~P[5];              // byte < 0x20
        const uint32_t H0 = LOW & ~P[4];
        const uint32_t h23 = ~P[7] & ~P[6] & P[5], H2 = h23 & ~P[4], H3 = h23 & P[4];
        const uint32_t h57 = ~P[7] & P[6] & P[4], H5 = h57 & ~P[5], H7 = h57 & P[5];
        const uint32_t x10 = P[3] & ~P[2], x11 = P[3] & P[2];
        const uint32_t La = x10 & P[1] & ~P[0], L9 = x10 & ~P[1] & P[0], Lb = x10 & P[1] & P[0], L8 = x10 & ~P[1] & ~P[0];
        const uint32_t Ld = x11 & ~P[1] & P[0], Lf = x11 & P[1] & P[0], Le = x11 & P[1] & ~P[0], Lc = x11 & ~P[1] & ~P[0];
        const uint32_t L0 = ~P[3] & ~P[2] & ~P[1] & ~P[0];
        const uint32_t NL = H0 & La, TABCR = H0 & (L9 | Ld), SP = H2 & L0;
        const uint32_t BLANK = (LOW | SP) & ~NL;                 // <= 0x20 and not '\n' (only \t \r ' ' pass the reject test)
        const uint32_t SEMI = H3 & Lb, DOT = H2 & Le;
        const uint32_t RARE = (H2 & Lf) | (H3 & La) | (H7 & (Lb | Ld));                  // '/' ':' '{' '}'
        // bytes >= 0x80, and control bytes other than \t \n \r (CR only ever sits in front of a newline or inside a
        // comment, where Python's strip() / \s treat it like a space)
        badacc |= P[7] | (LOW & ~NL & ~TABCR);
        uint32_t COMMA = 0, OPEN = 0, CLOSE = 0;
        if (kRecords) {
          COMMA = H2 & Lc;
          OPEN = (H2 & L8) | (Lb & (H7 | H5));                   // '(' '{' '['
          CLOSE = (H2 & L9) | (Ld & (H7 | H5));                  // ')' '}' ']'
        }
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int u = (v0 + v) * 32 + lane, sh = 16 * v;
          reinterpret_cast<uint16_t*>(NLM)[u] = (uint16_t)((NL >> sh) & keep[v]);
          uint16_t* m16 = reinterpret_cast<uint16_t*>(MA + (u >> 1)) + (u & 1);     // field f of word u/2: halfword 2f + (u&1)
          m16[0] = (uint16_t)(SEMI >> sh);
          m16[2] = (uint16_t)(RARE >> sh);
          m16[4] = (uint16_t)(BLANK >> sh);
          m16[6] = (uint16_t)(DOT >> sh);
          if (kRecords) {
            uint16_t* x16 = reinterpret_cast<uint16_t*>(MB + (u >> 1)) + (u & 1);
            x16[0] = (uint16_t)(COMMA >> sh);
            x16[2] = (uint16_t)(OPEN >> sh);
            x16[4] = (uint16_t)(CLOSE >> sh);
          }
        }
      }
      __syncwarp();
      if (__any_sync(kFull, badacc != 0)) { reject = true; break; }

      // ================= T: line table and prefix counts =================
      uint32_t rw[4], dw[4];                                     // this lane's rare / dot words (S phase)
      int total_nl = 0;
      {
        const uint4 nw = *reinterpret_cast<const uint4*>(NLM + 4 * lane);
        const uint4 m0 = MA[4 * lane], m1 = MA[4 * lane + 1], m2 = MA[4 * lane + 2], m3 = MA[4 * lane + 3];
        rw[0] = m0.y; rw[1] = m1.y; rw[2] = m2.y; rw[3] = m3.y;
        dw[0] = m0.w; dw[1] = m1.w; dw[2] = m2.w; dw[3] = m3.w;
        const uint32_t c0 = (uint32_t)__popc(m0.x) | ((uint32_t)__popc(m0.y) << 16);
        const uint32_t c1 = (uint32_t)__popc(m1.x) | ((uint32_t)__popc(m1.y) << 16);
        const uint32_t c2 = (uint32_t)__popc(m2.x) | ((uint32_t)__popc(m2.y) << 16);
        const uint32_t c3 = (uint32_t)__popc(m3.x) | ((uint32_t)__popc(m3.y) << 16);
        int tot_sr = 0;
        const uint32_t ex = (uint32_t)warp_excl_sum((int)(c0 + c1 + c2 + c3), &tot_sr);
        *reinterpret_cast<uint4*>(P + 4 * lane) = make_uint4(ex, ex + c0, ex + c0 + c1, ex + c0 + c1 + c2);
        if (lane == 31) P[kFWords] = (uint32_t)tot_sr;
        const uint32_t nwv[4] = {nw.x, nw.y, nw.z, nw.w};
        int at = warp_excl_sum(__popc(nw.x) + __popc(nw.y) + __popc(nw.z) + __popc(nw.w), &total_nl);
        __syncwarp();                                            // NLM fully read before it becomes the careful list
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t m = nwv[k];
          while (m) {
            const int bit = __ffs((int)m) - 1;
            m &= m - 1;
            if (at < kFMaxLines) nl[at] = (uint16_t)(lane * 128 + 32 * k + bit);
            ++at;
          }
        }
      }
      if (kRecords) {
        // bracket parity by a prefix-xor over the whole tile (brackets alternate open / close in everything the
        // window parser accepts): MB becomes {commas, brackets, brackets that do not alternate from parity 0,
        // parity}.  A statement reads the parity in front of its operand list (the kernel body itself sits inside
        // a brace) and takes everything relative to it.
        uint4 b[4];
        uint32_t X[4], par = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) { b[k] = MB[4 * lane + k]; X[k] = b[k].y | b[k].z; par ^= (uint32_t)__popc(X[k]); }
        uint32_t carry = (uint32_t)__popc(__ballot_sync(kFull, par & 1u) & lt_mask) & 1u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t px = X[k];
          px ^= px << 1; px ^= px << 2; px ^= px << 4; px ^= px << 8; px ^= px << 16;
          const uint32_t incl = px ^ (0u - carry), excl = incl ^ X[k];
          MB[4 * lane + k] = make_uint4(b[k].x, X[k], (b[k].y & excl) | (b[k].z & ~excl), incl);
          carry ^= (uint32_t)__popc(X[k]) & 1u;
        }
      }
      const int n_real = total_nl < kFMaxLines ? total_nl : kFMaxLines;
      const bool virtual_last = at_seg_end && total_nl < kFMaxLines;   // text may end without a newline
      if (virtual_last && lane == 0) nl[n_real] = (uint16_t)hi;
      const int n_lines = n_real + (virtual_last ? 1 : 0);
      __syncwarp();
      if (n_lines == 0) { reject = true; break; }                // a line longer than the tile
      const int region_end = virtual_last ? hi : nl[n_real - 1] + 1;

      // ================= S: kernel header (ptx.py:165-176) =================
      if (phase == PH_SEARCH) {
        int from = (int)(scan_from_g - abase);
        if (from < lo) from = lo;
        for (;;) {
          int cand = lane_first(dw, lane, from, region_end, [&](int p) {
            return s[p + 1] == 'e' && s[p + 2] == 'n' && s[p + 3] == 't' && s[p + 4] == 'r' && s[p + 5] == 'y'; });
          cand = warp_min(cand);
          if (cand == 0x7fffffff) { scan_from_g = abase + region_end; break; }
          if (in_line_comment(s, cand, lo)) { from = cand + 1; continue; }
          int q = cand + 6;
          while (q < region_end && s[q] <= ' ') ++q;
          if (q >= region_end) {                                 // `\s+NAME` may continue in the next tile
            if (!at_seg_end) reject = true; else scan_from_g = abase + region_end;
            break;
          }
          if (s[q] == '/') { reject = true; break; }             // a comment inside the match: exact kernel
          if (q == cand + 6 || !ffb_is_name_start(s[q])) { from = cand + 1; continue; }
          int r = q + 1;
          while (r < region_end && ffb_is_name_char(s[r])) ++r;
          name_off = abase + q - seg_begin; name_len = r - q;
          phase = PH_HEADER; scan_from_g = abase + r;
          break;
        }
        if (reject) break;
      }
      if (phase == PH_HEADER) {
        int from = (int)(scan_from_g - abase);
        if (from < lo) from = lo;
        for (;;) {
          int cand = lane_first(rw, lane, from, region_end, [&](int p) { return s[p] == '{'; });
          cand = warp_min(cand);
          if (cand == 0x7fffffff) { if (scan_from_g < abase + region_end) scan_from_g = abase + region_end; break; }
          if (in_line_comment(s, cand, lo)) { from = cand + 1; continue; }
          phase = PH_BODY; depth = 1; body_pos_g = abase + cand + 1;
          break;
        }
      }

      // ================= P1: line kinds =================
      int pos = 0x7fffffff, first = n_lines;                     // first body byte / line of this tile
      if (phase == PH_BODY) {
        pos = body_pos_g > cur ? (int)(body_pos_g - abase) : lo;
        first = 0;
        if (pos > lo) {
          for (int l = lane; l < n_lines; l += 32) first += (nl[l] < pos) ? 1 : 0;
          first = (int)warp_sum_u64((unsigned long long)first);
        }
      }
      int n_car = 0, bad_line = 0x7fffffff, ss_line = 0x7fffffff;
      for (int l0 = 0; l0 < n_lines; l0 += 32) {
        const int li = l0 + lane;
        const bool live = li < n_lines;
        bool careful = false;
        if (live) {
          const int b = li == 0 ? lo : nl[li - 1] + 1, e = nl[li];
          const uint32_t r = rank2(MA, P, e) - rank2(MA, P, b);
          careful = (r >> 16) != 0 || (li == first && pos > b);
          if (!careful && li >= first) {
            int kb = 0, ke = 0;
            const int kind = classify_plain(s, b, e, (int)(r & 0xffffu), &kb, &ke);
            linfo[li] = fk_pack(kind, kb, ke);
            if (kind == FK_BAD && li < bad_line) bad_line = li;
          }
        }
        const unsigned cm = __ballot_sync(kFull, careful);
        if (careful) clist[n_car + __popc(cm & lt_mask)] = (uint16_t)li;
        n_car += __popc(cm);
      }
      __syncwarp();
      int end_line = 0x7fffffff, close_at = 0;
      for (int c0 = 0; c0 < n_car; c0 += 32) {
        const int ci = c0 + lane;
        const bool live = ci < n_car;
        int li = 0x7fffffff, kind = FK_BLANK, kb = 0, ke = 0;
        if (live) {
          li = clist[ci];
          const int b = li == 0 ? lo : nl[li - 1] + 1, e = nl[li];
          const int bc = (li == first && pos > b) ? pos : b;
          bool ss = false;
          kind = resolve_careful(s, MA, b, bc, e, &kb, &ke, &ss);
          if (ss && li < ss_line) ss_line = li;
          if (li >= first) {
            linfo[li] = fk_pack(kind, kb, ke);
            if (kind == FK_BAD && li < bad_line) bad_line = li;
          } else kind = FK_BLANK;
        }
        if (end_line == 0x7fffffff) {                            // brace depth over the body lines, in order
          const int delta = kind == FK_OPEN ? 1 : (kind == FK_CLOSE ? -1 : 0);
          int tot = 0;
          const int d_after = depth + warp_excl_sum(delta, &tot) + delta;
          const unsigned closing = __ballot_sync(kFull, kind == FK_CLOSE && d_after == 0);
          if (closing) {
            const int src = __ffs((int)closing) - 1;
            end_line = __shfl_sync(kFull, li, src);
            close_at = __shfl_sync(kFull, kb, src);
          } else depth += tot;
        }
      }
      __syncwarp();
      const int n_eff = end_line < n_lines ? end_line : n_lines;
      bad_line = warp_min(bad_line);
      ss_line = warp_min(ss_line);
      if (bad_line < n_eff || ss_line < n_eff || (end_line != 0x7fffffff && ss_line <= end_line)) { reject = true; break; }

      // ================= P2: statements, labels, declarations =================
      const uint32_t tile_ins0 = n_instr;
      int n_slow = 0;
      uint16_t* slist = clist;                                   // the careful list is dead by now
      // Record mode parses the statements of a tile in rounds of SIMILAR LENGTH (histogram mode, whose parser
      // is short, loses more to the sort than it gains: 416 -> 388 GB/s, so it keeps line order): a statement's record slot is
      // fixed by its line order, so the processing order is free, and lines of the same length have
      // similar token / operand counts - the lanes of a round then follow the same path through the
      // parser far more often (the union of 32 unrelated statements costs ~4x one statement's path).
      // Counting sort by length: histogram, scan, scatter of (line | slot << 8) into the dead newline table.
      uint16_t* sorted = nl;
      uint32_t* bcnt = P;                                          // 64 bucket counters (the prefix counts are dead too)
      if (kRecords) { bcnt[lane] = 0; bcnt[lane + 32] = 0; __syncwarp(); }
      int n_stmt = 0;
      for (int l0 = first & ~31; l0 < n_eff; l0 += 32) {
        const int li = l0 + lane;
        const bool live = li >= first && li < n_eff;
        const uint32_t inf = live ? linfo[li] : 0u;
        const int kind = (int)(inf >> 26), kb = (int)(inf & 0x1fffu), ke = (int)((inf >> 13) & 0x1fffu);
        const unsigned stm = __ballot_sync(kFull, kind == FK_STMT);
        const unsigned lbm = __ballot_sync(kFull, kind == FK_LABEL);
        const unsigned dcm = __ballot_sync(kFull, kind == FK_DECL);
        const int64_t my_ins = ins_base + n_instr + __popc(stm & lt_mask);
        if (kRecords) { if (kind == FK_STMT) atomicAdd(&bcnt[min(ke - kb, 63)], 1u); }
        else {
          bool slow = false;
          if (kind == FK_STMT) {
            em.ins_at = my_ins;
            em.line = line_no + (uint32_t)li;
            slow = !fast_statement<kMain>(s, MA, MB, memo, kb, ke, em);
          }
          const unsigned slm = __ballot_sync(kFull, slow);
          if (slow) slist[n_slow + __popc(slm & lt_mask)] = (uint16_t)(li | ((int)(my_ins - ins_base - tile_ins0) << 8));
          n_slow += __popc(slm);
        }
        if (kRecords && kind == FK_LABEL) {
          const int64_t slot = lab_base + n_labels + __popc(lbm & lt_mask);
          FfbLabelRec L;
          L.hash = hash_span(s, kb, ke); L.index = (uint32_t)(my_ins - ins_base);
          L.off = (uint32_t)(abase + kb - seg_begin);
          if (slot < em.lab_limit) a.labels[slot] = L;
        }
        int nd = 0;
        if (dcm) {
          if (kind == FK_DECL) {
            const DeclResult dr = cold_directive(s, kb, ke);
            em.regs += dr.regs; em.shared_bytes += dr.shared; nd = dr.n_reg_decl;
          }
          nd = (int)warp_sum_u64((unsigned long long)nd);
        }
        n_instr += (uint32_t)__popc(stm); n_labels += (uint32_t)__popc(lbm); n_decls += (uint32_t)nd;
        n_stmt += __popc(stm);
      }
      __syncwarp();
      if (kRecords) {
        int tot = 0;
        const uint32_t c0 = bcnt[2 * lane], c1 = bcnt[2 * lane + 1];
        const uint32_t base_of = (uint32_t)warp_excl_sum((int)(c0 + c1), &tot);     // bucket starts
        __syncwarp();
        bcnt[2 * lane] = base_of; bcnt[2 * lane + 1] = base_of + c0;
        __syncwarp();
        uint32_t seen = 0;
        for (int l0 = first & ~31; l0 < n_eff; l0 += 32) {
          const int li = l0 + lane;
          const bool live = li >= first && li < n_eff;
          const uint32_t inf = live ? linfo[li] : 0u;
          const bool st = (int)(inf >> 26) == FK_STMT;
          const unsigned stm = __ballot_sync(kFull, st);
          if (st) {
            const uint32_t slot = seen + __popc(stm & lt_mask);                      // statement index within the tile
            const uint32_t at = atomicAdd(&bcnt[min((int)((inf >> 13) & 0x1fffu) - (int)(inf & 0x1fffu), 63)], 1u);
            sorted[at] = (uint16_t)(li | (slot << 8));
          }
          seen += __popc(stm);
        }
        __syncwarp();
      }
      for (int i0 = 0; kRecords && i0 < n_stmt; i0 += 32) {
        const int i = i0 + lane;
        bool slow = false;
        uint32_t ent = 0;
        if (i < n_stmt) {
          ent = sorted[i];
          const int li = (int)(ent & 255u);
          const uint32_t inf = linfo[li];
          em.ins_at = ins_base + tile_ins0 + (ent >> 8);
          em.line = line_no + (uint32_t)li;
          slow = !fast_statement<kMain>(s, MA, MB, memo, (int)(inf & 0x1fffu), (int)((inf >> 13) & 0x1fffu), em);
        }
        const unsigned slm = __ballot_sync(kFull, slow);
        if (slow) slist[n_slow + __popc(slm & lt_mask)] = (uint16_t)ent;
        n_slow += __popc(slm);
      }
      __syncwarp();
      n_slow_seg += (uint32_t)n_slow;
      for (int i0 = 0; i0 < n_slow; i0 += 32) {                 // statements the windows could not express
        const int i = i0 + lane;
        if (i < n_slow) {
          const unsigned ent = slist[i];
          const int li = (int)(ent & 255u);
          const uint32_t inf = linfo[li];
          const uint32_t cls = cold_statement<kMain>(&a, s_tok_key, s_tok_val, s_cls, s, (int)(inf & 0x1fffu), (int)((inf >> 13) & 0x1fffu),
                                                     ins_base + tile_ins0 + (ent >> 8), em.ins_limit, line_no + (uint32_t)li, abase, seg_begin);
          const uint64_t inc = 1ull << (21 * (cls % 3u));
          em.c0 += cls < 3u ? inc : 0ull; em.c1 += (cls >= 3u && cls < 6u) ? inc : 0ull; em.c2 += cls >= 6u ? inc : 0ull;
        }
      }
      if (end_line != 0x7fffffff) {
        phase = PH_DONE;
        body_end_off = abase + close_at - seg_begin;
        break;
      }

      // ================= advance =================
      line_no += (uint32_t)n_real;
      const int64_t next = abase + region_end;
      if (next <= cur) { reject = true; break; }
      cur = next;
    } while (0);
    if (!(phase == PH_DONE || reject || cur >= seg_end)) continue;   // more tiles of this segment

    // ================= segment epilogue =================
    // only complete, well-formed kernels are finished here; every error status comes from the exact kernel
    bool ok = !reject && phase == PH_DONE && n_instr > 0;   // (an empty segment ends here too: nothing found)
    if (kRecords && ok && ((a.ins_cap && (int64_t)n_instr > a.ins_cap[seg]) || (a.lab_cap && (int64_t)n_labels > a.lab_cap[seg]))) ok = false;
    have = false;
    if (!ok) {
      if (lane == 0) a.fb_list[atomicAdd(a.fb_count, 1ull)] = (int32_t)seg;
      continue;
    }
#pragma unroll 1
    for (int c = 0; c < FFB_N_CLASSES; ++c) {
      const uint64_t word = c < 3 ? em.c0 : (c < 6 ? em.c1 : em.c2);
      const uint32_t tot = (uint32_t)warp_sum_u64((word >> (21 * (c % 3))) & 0x1fffffull);
      if (lane == 0) a.hist[seg * FFB_N_CLASSES + c] = tot;
    }
    const unsigned long long sh = warp_sum_u64(em.shared_bytes), rg = warp_sum_u64(em.regs);
    if (lane == 0) {
      FfbSegInfo inf;
      inf.status = FFB_OK; inf.n_instr = n_instr; inf.n_labels = n_labels; inf.n_decls = n_decls;
      inf.static_shared = sh; inf.regs_declared = rg;
      inf.name_off = (uint32_t)name_off; inf.name_len = (uint32_t)name_len;
      inf.body_off = (uint32_t)(body_pos_g - seg_begin); inf.body_end = (uint32_t)body_end_off;
      a.info[seg] = inf;
      if (n_slow_seg) atomicAdd(a.fb_count + 2, (unsigned long long)n_slow_seg);   // statistics only
    }
  }
}

}  // namespace
