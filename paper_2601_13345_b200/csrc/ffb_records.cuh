// Device-side record formats shared by the lexer (K1) and the dataflow kernel (K1b),
// plus the character classes and hashing both use.  Mirrored in include/ffb.h for callers
// that want to read the records back (the Python shim does, to rebuild PtxModule objects).
#pragma once
#include "ffb_common.cuh"

// ---- character classes -------------------------------------------------------------------
// Whitespace = Python str.strip()/split() on ASCII = regex \s on str: \t \n \v \f \r FS GS RS US ' '
FFB_HD bool ffb_is_ws(unsigned c) { return c <= 32u && ((0x1F0003E00ull >> c) & 1ull); }
FFB_HD bool ffb_is_digit(unsigned c) { return c - '0' < 10u; }
FFB_HD bool ffb_is_alpha(unsigned c) { return ((c | 32u) - 'a') < 26u; }
FFB_HD bool ffb_is_word(unsigned c) { return ffb_is_alpha(c) || ffb_is_digit(c) || c == '_'; }       // \w (ASCII)
FFB_HD bool ffb_is_label_char(unsigned c) { return ffb_is_word(c) || c == '$' || c == '.'; }        // [\w$.]
FFB_HD bool ffb_is_name_char(unsigned c) { return ffb_is_word(c) || c == '$'; }                     // [\w$]
FFB_HD bool ffb_is_name_start(unsigned c) { return ffb_is_alpha(c) || c == '_' || c == '$'; }        // [A-Za-z_$]

// ---- packed short tokens -----------------------------------------------------------------
// Tokens of at most 8 bytes are compared as one little-endian u64.
constexpr uint64_t ffb_pk(const char* s) {
  uint64_t v = 0;
  int i = 0;
  for (; s[i] && i < 8; ++i) v |= (uint64_t)(unsigned char)s[i] << (8 * i);
  return v;
}

// ---- 61-bit name hash ----------------------------------------------------------------------
// The text is cut into 8-byte little-endian chunks (the last one zero-padded); every chunk is
// mixed with one multiply-xorshift, the length goes in at the end.  Tokens of at most 16 bytes
// (registers, literals, labels) are hashed from two packed words without a byte loop
// (ffb_hash_packed); the streaming form below gives the same value for any length.
constexpr uint64_t kHashBasis = 0xcbf29ce484222325ull, kHashMul = 0x9e3779b97f4a7c15ull;
FFB_HD uint64_t ffb_hash_chunk(uint64_t h, uint64_t c) { h = (h ^ c) * kHashMul; return h ^ (h >> 31); }
FFB_HD uint64_t ffb_hash_fold(uint64_t h) { h ^= h >> 29; h *= 0xbf58476d1ce4e5b9ull; h ^= h >> 32; return h & 0x1fffffffffffffffull; }
struct FfbHasher { uint64_t h, pk; uint32_t n; };
FFB_HD void ffb_hash_init(FfbHasher& x) { x.h = kHashBasis; x.pk = 0; x.n = 0; }
FFB_HD void ffb_hash_byte(FfbHasher& x, unsigned c) {
  x.pk |= (uint64_t)(c & 0xffu) << (8u * (x.n & 7u));
  if ((++x.n & 7u) == 0u) { x.h = ffb_hash_chunk(x.h, x.pk); x.pk = 0; }
}
FFB_HD uint64_t ffb_hash_done(const FfbHasher& x) {
  uint64_t h = x.h;
  if (x.n & 7u) h = ffb_hash_chunk(h, x.pk);
  return ffb_hash_fold(h ^ (uint64_t)x.n);
}
// len <= 16 bytes packed little-endian into (lo, hi), unused bytes zero
FFB_HD uint64_t ffb_hash_packed(uint64_t lo, uint64_t hi, uint32_t len) {
  uint64_t h = kHashBasis;
  if (len > 0) h = ffb_hash_chunk(h, lo);
  if (len > 8) h = ffb_hash_chunk(h, hi);
  return ffb_hash_fold(h ^ (uint64_t)len);
}

// ---- operand descriptor --------------------------------------------------------------------
// bits 63..61 kind, bits 60..0 payload (name hash, or two's-complement value for INT)
enum : uint64_t {
  FFB_OPK_NONE = 0,      // operand absent
  FFB_OPK_REG = 1,       // %name looked up in the scale table            (alignment.py:41-42)
  FFB_OPK_TIDX = 2,      // exactly %tid.x                       -> scale 1 (alignment.py:34-35)
  FFB_OPK_UNKNOWN = 3,   // %tid.y/.z, %laneid, %warpid          -> None   (alignment.py:36-37)
  FFB_OPK_UNIFORM = 4,   // uniform special or any non-% operand -> scale 0 (alignment.py:38-47)
  FFB_OPK_INT = 5,       // Python int(text, 0) literal, |v| < 2^60       (scale 0, value kept)
  FFB_OPK_BIGINT = 6,    // int literal outside that range
  FFB_OPK_UNIFORM_REG = 7,  // %-prefixed uniform special (%ctaid.x, %ntid.y, %gridid ...) -> scale 0
};
FFB_HD uint64_t ffb_op_make(uint64_t kind, uint64_t payload) { return (kind << 61) | (payload & 0x1fffffffffffffffull); }
FFB_HD uint64_t ffb_op_kind(uint64_t d) { return d >> 61; }
FFB_HD uint64_t ffb_op_hash(uint64_t d) { return d & 0x1fffffffffffffffull; }
FFB_HD int64_t ffb_op_int(uint64_t d) { return (int64_t)(d << 3) >> 3; }

// ---- instruction record (64 B) ---------------------------------------------------------------
// meta: [3:0] class  [6:4] space  [12:7] access bytes  [17:13] base id  [18] has predicate
//       [19] predicate negated  [22:20] operand count (7 = seven or more)  [25:23] compare
//       [27:26] address kind  [28] first operand starts with '%'  [29] operands beyond slot 5
//       hold a generic register
enum { FFB_BASE_OTHER = 0, FFB_BASE_MOV, FFB_BASE_CVT, FFB_BASE_CVTA, FFB_BASE_ADD, FFB_BASE_SUB,
       FFB_BASE_MUL, FFB_BASE_MAD, FFB_BASE_FMA, FFB_BASE_SHL, FFB_BASE_SETP, FFB_BASE_RET,
       FFB_BASE_EXIT };
enum { FFB_CMP_NONE = 0, FFB_CMP_LT, FFB_CMP_GE, FFB_CMP_LE, FFB_CMP_GT, FFB_CMP_EQ, FFB_CMP_NE };
enum { FFB_ADDR_ABSENT = 0, FFB_ADDR_NOMATCH, FFB_ADDR_SYMBOL, FFB_ADDR_REG };

struct __align__(16) FfbInsRec {
  uint32_t meta;
  uint32_t line;       // 1-based source line of the statement's first line
  uint32_t off;        // statement start, bytes from the segment start
  uint32_t len;        // statement length in bytes (raw text, up to but excluding ';')
  uint64_t pred;       // hash of the predicate register name (without '!'), 0 if none
  uint64_t aux;        // memory: address-base descriptor; Branch: descriptor of the LAST operand;
                       // otherwise descriptor of operand 4 (FFB_OPK_NONE if absent)
  uint64_t op[4];      // descriptors of operands 0..3
};
static_assert(sizeof(FfbInsRec) == 64, "FfbInsRec layout");

FFB_HD uint32_t ffb_meta_cls(uint32_t m) { return m & 15u; }
FFB_HD uint32_t ffb_meta_space(uint32_t m) { return (m >> 4) & 7u; }
FFB_HD uint32_t ffb_meta_bytes(uint32_t m) { return (m >> 7) & 63u; }
FFB_HD uint32_t ffb_meta_base(uint32_t m) { return (m >> 13) & 31u; }
FFB_HD bool ffb_meta_has_pred(uint32_t m) { return (m >> 18) & 1u; }
FFB_HD bool ffb_meta_pred_neg(uint32_t m) { return (m >> 19) & 1u; }
FFB_HD uint32_t ffb_meta_nops(uint32_t m) { return (m >> 20) & 7u; }
FFB_HD uint32_t ffb_meta_cmp(uint32_t m) { return (m >> 23) & 7u; }
FFB_HD uint32_t ffb_meta_addr(uint32_t m) { return (m >> 26) & 3u; }
FFB_HD bool ffb_meta_dst_reg(uint32_t m) { return (m >> 28) & 1u; }
FFB_HD bool ffb_meta_extra_reg(uint32_t m) { return (m >> 29) & 1u; }

// ---- label record (16 B) ----------------------------------------------------------------------
struct __align__(16) FfbLabelRec {
  uint64_t hash;       // 61-bit name hash
  uint32_t index;      // instruction index the label points at (ptx.py:234)
  uint32_t off;        // name start, bytes from the segment start (length = len)
};
static_assert(sizeof(FfbLabelRec) == 16, "FfbLabelRec layout");
