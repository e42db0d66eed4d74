// K1b: per-kernel control-flow and affine dataflow over the lexer's instruction records
// -> trip-weighted dynamic counts and aligned_fraction (one FFB_F_* feature row per kernel).
//
// Restates pkg/src/ptxwatt: ptx.py:277-284 (branch targets must be labels), cfg.py:57-95
// (leaders, blocks, edges), :98-151 (dominators, natural loops, one loop per header),
// :154-182 (trip precedence: annotation > detected > default, floored at 1), :191-279
// (counted do-while recogniser), :43-54 (block weights), alignment.py:31-125 (register ->
// %tid.x scale map, single textual pass) and :128-147 (weighted aligned fraction),
// features.py:62-81 (dynamic counts).
//
// Launched as TWO kernels for feature rows (flow_kernel<1>: CFG, loops, trips, weights; flow_kernel<2>: the textual
// dataflow pass) and as one (flow_kernel<0>) when the caller wants the detail outputs; see the template's comment.
// One WARP per kernel (dynamic queue, longest first).  Lane-parallel: label table, leaders, block
// numbering, edges, predecessor lists, the "last match" scans of the trip recogniser, weights and
// the textual dataflow pass (32 statements per round).  Lane 0 alone: DFS, dominators and loop
// bodies, which are sequential graph walks.  The CFG working arrays live in a context-owned HBM
// scratch indexed by the same exclusive scans as the records.
//
// Dominators: the reference iterates full bit-sets to the maximal fixed point.  For blocks
// reachable from block 0 that equals the dominator tree (computed here with the
// Cooper-Harvey-Kennedy iteration over a reverse post-order); blocks NOT reachable keep the
// full set, i.e. every block "dominates" them — reproduced explicitly (dominates()).
#include "ffb_records.cuh"

#include <math.h>

#ifdef FFB_SIMT_EMUL
#define FFB_PREFETCH(p) ((void)(p))
#else
#define FFB_PREFETCH(p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p))
#endif

namespace {

constexpr int kFlowWarps = 4;
constexpr int kMapSlots = 512;                    // shared-memory register -> scale map per warp (8 KB)
constexpr int kMapFill = 384;
constexpr int kLeadWords = 256;                   // flow_kernel<1>: leader flags of kernels up to 8 192 statements as a shared-memory bit set
constexpr int kLabSlots = 128;                    // flow_kernel<1>: label tables of up to this many slots (<= 63 labels) in shared memory
constexpr int kBodyList = 32;                     // loop bodies up to this many blocks are scanned through a compact list                     // entries kept on chip; later names spill to the HBM table
constexpr int64_t kNoneScale = INT64_MIN;            // alignment.py "None"
constexpr int64_t kBigScale = INT64_MIN + 1;         // |scale| beyond 2^62: known, never aligned
constexpr uint32_t kNoBlock = 0xffffffffu;

// two-kernel form: state of one PTX kernel between the CFG kernel and the dataflow kernel (everything else -
// block_of, weight - already lives in the context's scratch)
struct FlowMid { uint32_t status, nb, n_edges, n_loops; };

struct FlowArgs {
  int64_t n_segs;
  const FfbSegInfo* info;
  const int64_t* ins_base;
  const int64_t* lab_base;
  const FfbInsRec* ins;
  const FfbLabelRec* labels;
  const uint32_t* meta_arr;     // optional compact meta words
  const int32_t* order;
  unsigned long long* work;     // work-queue counters (one per kernel of the two-kernel form)
  struct FlowMid* mid;          // [K] what the CFG kernel hands to the dataflow kernel
  double default_trip;
  int parallel_pass;            // 0: textual pass on lane 0 only (test switch)
  const uint64_t* ann_hash;     // device copies
  const double* ann_trip;
  int n_ann;
  uint8_t* ann_hit;             // [n_ann] set when a loop header carries the label
  double* feat;
  uint32_t* status;
  FfbFlowInfo* flow;
  // scratch (see host side for the carve-up)
  uint32_t* block_of;           // [N]
  uint32_t* block_start;        // [N + 2K]
  int32_t* succ0;               // [N + 2K]
  int32_t* succ1;
  uint32_t* pred_ptr;           // [N + 2K]
  uint32_t* pred_list;          // [2(N + 2K)]
  int32_t* rpo_num;             // [N + 2K]
  uint32_t* rpo_order;
  int32_t* idom;
  uint32_t* mark;
  uint32_t* stack;
  double* weight;               // [N + 2K]
  uint64_t* lab_key;            // [4L + 8K]
  uint32_t* lab_first;
  uint32_t* lab_last;
  uint64_t* sc_key;             // [4N + 8K]
  int64_t* sc_val;
  // detail outputs (optional)
  uint32_t* out_block_start;
  int32_t* out_edges;
  FfbLoopRec* out_loops;
  uint8_t* out_loop_body;
  int64_t loop_body_cap;
  double* out_weights;
};

// ---- tiny open-addressing tables ----------------------------------------------------------------
// capacities are powers of two
// keys are 61-bit name hashes that went through ffb_hash_fold already (multiply + xorshift): their bits are
// uniform, so a fold of the two halves is a good slot without another 64-bit multiply
FFB_D uint32_t slot_of(uint64_t h, uint32_t cap) { return ((uint32_t)h ^ (uint32_t)(h >> 32)) & (cap - 1u); }

struct LabelTable {
  uint64_t* key; uint32_t* first; uint32_t* last; uint32_t cap;
  FFB_D void clear() { for (uint32_t i = 0; i < cap; ++i) key[i] = 0; }
  FFB_D uint32_t find(uint64_t h) const {          // slot or cap
    uint32_t s = slot_of(h, cap);
    for (uint32_t n = 0; n < cap; ++n) {
      if (key[s] == 0) return cap;
      if (key[s] == h + 1) return s;
      s = (s + 1) & (cap - 1u);
    }
    return cap;
  }
  FFB_D void define(uint64_t h, uint32_t order, uint32_t /*unused*/) {
    uint32_t s = slot_of(h, cap);
    for (;;) {
      if (key[s] == 0) { key[s] = h + 1; first[s] = order; last[s] = order; return; }
      if (key[s] == h + 1) { last[s] = order; return; }
      s = (s + 1) & (cap - 1u);
    }
  }
};

struct ScaleTable {
  uint64_t* key; int64_t* val; uint32_t cap;
  FFB_D void clear() { for (uint32_t i = 0; i < cap; ++i) key[i] = 0; }
  FFB_D int64_t get(uint64_t h) const {
    uint32_t s = slot_of(h, cap);
    for (uint32_t n = 0; n < cap; ++n) {
      if (key[s] == 0) return kNoneScale;
      if (key[s] == h + 1) return val[s];
      s = (s + 1) & (cap - 1u);
    }
    return kNoneScale;
  }
  FFB_D void put(uint64_t h, int64_t v) {
    uint32_t s = slot_of(h, cap);
    for (;;) {
      if (key[s] == 0 || key[s] == h + 1) { key[s] = h + 1; val[s] = v; return; }
      s = (s + 1) & (cap - 1u);
    }
  }
};

// ---- scale arithmetic with saturation -------------------------------------------------------------
FFB_D bool sc_known(int64_t v) { return v != kNoneScale; }
FFB_D int64_t sc_add(int64_t a, int64_t b) {
  if (!sc_known(a) || !sc_known(b)) return kNoneScale;
  if (a == kBigScale || b == kBigScale) return kBigScale;
  const int64_t lim = (int64_t)1 << 61;
  const int64_t r = a + b;     // |a|,|b| <= 2^61: no wrap
  return (r > lim || r < -lim) ? kBigScale : r;
}
FFB_D int64_t sc_neg(int64_t a) { return (!sc_known(a) || a == kBigScale) ? a : -a; }
FFB_D int64_t sc_mul(int64_t a, int64_t b) {
  if (!sc_known(a) || !sc_known(b)) return kNoneScale;
  if (a == 0 || b == 0) return 0;
  if (a == kBigScale || b == kBigScale) return kBigScale;
  const int64_t lim = (int64_t)1 << 61;
  const uint64_t ua = a < 0 ? (uint64_t)(-a) : (uint64_t)a, ub = b < 0 ? (uint64_t)(-b) : (uint64_t)b;
  if (__umul64hi(ua, ub) != 0) return kBigScale;
  const uint64_t p = ua * ub;
  if (p > (uint64_t)lim) return kBigScale;
  return ((a < 0) != (b < 0)) ? -(int64_t)p : (int64_t)p;
}

// alignment.py:31-47 on a descriptor
FFB_D int64_t operand_scale(uint64_t d, const ScaleTable& t) {
  switch (ffb_op_kind(d)) {
    case FFB_OPK_TIDX: return 1;
    case FFB_OPK_UNKNOWN: return kNoneScale;
    case FFB_OPK_REG: return t.get(ffb_op_hash(d));
    case FFB_OPK_NONE: return kNoneScale;
    default: return 0;       // UNIFORM, UNIFORM_REG, INT, BIGINT
  }
}
FFB_D bool is_int_lit(uint64_t d) { const uint64_t k = ffb_op_kind(d); return k == FFB_OPK_INT || k == FFB_OPK_BIGINT; }
FFB_D int64_t int_as_scale(uint64_t d) { return ffb_op_kind(d) == FFB_OPK_INT ? ffb_op_int(d) : kBigScale; }
FFB_D bool starts_with_percent(uint64_t d) {
  const uint64_t k = ffb_op_kind(d);
  return k == FFB_OPK_REG || k == FFB_OPK_TIDX || k == FFB_OPK_UNKNOWN || k == FFB_OPK_UNIFORM_REG;
}

// alignment.py:50-58 (_combine_mul)
FFB_D int64_t mul_scale(uint64_t a, uint64_t b, const ScaleTable& t) {
  const int64_t sa = operand_scale(a, t), sb = operand_scale(b, t);
  if (sa == 0 && sb == 0) return 0;
  if (is_int_lit(b) && sc_known(sa)) return sc_mul(sa, int_as_scale(b));
  if (is_int_lit(a) && sc_known(sb)) return sc_mul(int_as_scale(a), sb);
  return kNoneScale;
}

// dom(h, u): h in the reference's dominator set of u
FFB_D bool dominates(const int32_t* idom, const int32_t* rpo_num, uint32_t h, uint32_t u) {
  if (rpo_num[u] < 0) return true;          // unreachable blocks keep the full set (cfg.py:108-122)
  if (rpo_num[h] < 0) return h == u;
  uint32_t x = u;
  for (;;) {
    if (x == h) return true;
    if (x == 0) return false;
    x = (uint32_t)idom[x];
  }
}

// ---- warp helpers -----------------------------------------------------------------------------------
constexpr unsigned kAll = 0xffffffffu;
FFB_D int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { const int64_t o = __shfl_xor_sync(kAll, v, d); v = o > v ? o : v; }
  return v;
}
FFB_D int warp_sum_i(int v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kAll, v, d);
  return v;
}

// Register -> scale map of the textual pass (alignment.py:61-125).  The first kMapFill distinct
// names live in an open-addressing table in shared memory, so the sequential walk never leaves
// the SM for ordinary kernels (r1i: 80% of the stall samples of this kernel were lane 0 waiting
// on the HBM-resident table).  Names met after that go to the HBM table `g`, cleared lazily on
// the first spill.  Used by lane 0 only.
struct CachedScales {
  ScaleTable g;
  uint64_t* ckey; int64_t* cval;
  uint32_t used; bool spilled;
  FFB_D int64_t get(uint64_t h) {
    uint32_t c = slot_of(h, kMapSlots);
    for (;;) {
      const uint64_t k = ckey[c];
      if (k == h + 1) return cval[c];
      if (k == 0) break;
      c = (c + 1) & (kMapSlots - 1);
    }
    return spilled ? g.get(h) : kNoneScale;
  }
  FFB_D void put(uint64_t h, int64_t v) {
    uint32_t c = slot_of(h, kMapSlots);
    for (;;) {
      const uint64_t k = ckey[c];
      if (k == h + 1) { cval[c] = v; return; }
      if (k == 0) break;
      c = (c + 1) & (kMapSlots - 1);
    }
    if (used < kMapFill) { ckey[c] = h + 1; cval[c] = v; ++used; return; }
    if (!spilled) { g.clear(); spilled = true; }
    g.put(h, v);
  }
};
FFB_D int64_t operand_scale_c(uint64_t d, CachedScales& t) {
  switch (ffb_op_kind(d)) {
    case FFB_OPK_TIDX: return 1;
    case FFB_OPK_UNKNOWN: return kNoneScale;
    case FFB_OPK_REG: return t.get(ffb_op_hash(d));
    case FFB_OPK_NONE: return kNoneScale;
    default: return 0;
  }
}
FFB_D int64_t mul_scale_c(uint64_t a, uint64_t b, CachedScales& t) {
  const int64_t sa = operand_scale_c(a, t), sb = operand_scale_c(b, t);
  if (sa == 0 && sb == 0) return 0;
  if (is_int_lit(b) && sc_known(sa)) return sc_mul(sa, int_as_scale(b));
  if (is_int_lit(a) && sc_known(sb)) return sc_mul(int_as_scale(a), sb);
  return kNoneScale;
}

// ---- one statement of the textual pass, from the scales of its sources ------------------------------
// s1..s3 / sa: scales of operands 1..3 and of the `aux` descriptor (alignment.py:31-47), however the
// caller obtained them (table look-up, or the value an earlier statement of the same chunk published).
struct SrcScales { int64_t s1, s2, s3, sa; };
FFB_D int64_t mul_scale_v(uint64_t a, uint64_t b, int64_t sa, int64_t sb) {          // alignment.py:50-58
  if (sa == 0 && sb == 0) return 0;
  if (is_int_lit(b) && sc_known(sa)) return sc_mul(sa, int_as_scale(b));
  if (is_int_lit(a) && sc_known(sb)) return sc_mul(int_as_scale(a), sb);
  return kNoneScale;
}
// Non-memory statement with a register destination (alignment.py:91-125): the scale it defines.
// Returns false for setp (no definition).
FFB_D bool eval_def(uint32_t m, uint64_t op1, uint64_t op2, uint64_t op3, const SrcScales& s, int64_t* out, uint32_t* status) {
  const uint32_t nops = ffb_meta_nops(m), base = ffb_meta_base(m);
  int64_t v;
  if (base == FFB_BASE_MOV && nops == 2) v = s.s1;
  else if ((base == FFB_BASE_CVT || base == FFB_BASE_CVTA) && nops >= 2) {
    v = nops == 2 ? s.s1 : nops == 3 ? s.s2 : nops == 4 ? s.s3 : s.sa;            // LAST operand
    if (nops > 5) { *status = FFB_E_CAPACITY; v = kNoneScale; }
  } else if ((base == FFB_BASE_ADD || base == FFB_BASE_SUB) && nops == 3) {
    v = base == FFB_BASE_ADD ? sc_add(s.s1, s.s2) : sc_add(s.s1, sc_neg(s.s2));
  } else if (base == FFB_BASE_MUL && nops == 3) v = mul_scale_v(op1, op2, s.s1, s.s2);
  else if ((base == FFB_BASE_MAD || base == FFB_BASE_FMA) && nops == 4) v = sc_add(mul_scale_v(op1, op2, s.s1, s.s2), s.s3);
  else if (base == FFB_BASE_SHL && nops == 3) {
    if (!sc_known(s.s1) || !is_int_lit(op2)) v = kNoneScale;
    else {
      const int64_t sh = int_as_scale(op2);
      if (sh == kBigScale || sh < 0) { *status = FFB_E_CAPACITY; v = kNoneScale; }   // 1 << huge / negative: reference raises
      else v = s.s1 == 0 ? 0 : (sh >= 61 ? kBigScale : sc_mul(s.s1, (int64_t)1 << sh));
    }
  } else if (base == FFB_BASE_SETP) return false;
  else {
    // unmodelled producer: uniform only if it has sources and all of them are uniform
    bool all0 = nops >= 2;
    if (nops > 1) all0 = all0 && s.s1 == 0;
    if (nops > 2) all0 = all0 && s.s2 == 0;
    if (nops > 3) all0 = all0 && s.s3 == 0;
    if (nops >= 5) all0 = all0 && s.sa == 0;
    if (all0 && nops >= 6 && ffb_meta_extra_reg(m)) { *status = FFB_E_CAPACITY; all0 = false; }
    v = all0 ? 0 : kNoneScale;
  }
  *out = v;
  return true;
}
// Per-statement contributions to the dynamic counts (features.py:62-81) and the alignment sums
// (alignment.py:137-144); `sc_addr` is the scale of the address register of a global access.
struct Sums { double n_mem, mem_bytes, u_fp, u_int, u_sfu, u_alu, n_sync, al_hit, al_tot; };
FFB_D void count_statement(uint32_t m, double wgt, int64_t sc_addr, Sums& a) {
  const uint32_t cls = ffb_meta_cls(m);
  if (cls == FFB_CLS_MEMLOAD || cls == FFB_CLS_MEMSTORE) {
    const uint32_t space = ffb_meta_space(m), bytes = ffb_meta_bytes(m);
    if (space != FFB_SP_PARAM) { a.n_mem += wgt; a.mem_bytes += wgt * (double)bytes; }
    if (space == FFB_SP_GLOBAL) {
      int64_t sc = kNoneScale;
      const uint32_t ak = ffb_meta_addr(m);
      if (ak == FFB_ADDR_SYMBOL) sc = 0;
      else if (ak == FFB_ADDR_REG) sc = sc_addr;
      a.al_tot += wgt;
      if (sc_known(sc) && sc != kBigScale && (sc < 0 ? -sc : sc) == (int64_t)bytes) a.al_hit += wgt;
    }
    return;
  }
  if (cls == FFB_CLS_FP32) a.u_fp += wgt;
  else if (cls == FFB_CLS_INT) a.u_int += wgt;
  else if (cls == FFB_CLS_SFU) a.u_sfu += wgt;
  else if (cls == FFB_CLS_ALU) a.u_alu += wgt;
  else if (cls == FFB_CLS_SYNC) a.n_sync += wgt;
}
FFB_D double warp_sum_d(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kAll, v, d);
  return v;
}

// One WARP per kernel.  Lane-parallel: label table, leaders, block numbering, edges, the
// "last match" scans of the trip recogniser, weights, record staging.  Lane 0 alone: the graph
// walks (DFS, dominators, loop bodies) and the textual dataflow pass, which are sequential by
// nature.
// kPart 0: the whole analysis of a PTX kernel in one launch (the drop-in API's detail outputs, annotations).
// kPart 1 / 2: the same code as two launches - CFG, loops, trips and block weights (no scale maps: a third of the
// shared memory, more resident warps for its latency-bound scratch walks), then the textual dataflow pass - each
// half the instruction footprint of the whole.  What crosses the cut is FlowMid + the scratch arrays.
template <int kPart>
__global__ void __launch_bounds__(kFlowWarps * 32, kPart == 1 ? 8 : 6)
flow_kernel(FlowArgs a) {
  constexpr int kMs = kPart == 1 ? 1 : kMapSlots, kCh = kPart == 1 ? 1 : 64;
  __shared__ uint64_t s_ckey[kFlowWarps][kMs];
  __shared__ int64_t s_cval[kFlowWarps][kMs];
  __shared__ uint64_t s_chkey[kFlowWarps][kCh];     // chunk-local: names the 32 statements in flight define
  __shared__ uint32_t s_chmask[kFlowWarps][kCh];    //              ... and the lanes that define them
  __shared__ int64_t s_chval[kFlowWarps][kPart == 1 ? 1 : 32];                          //              ... and the values they publish
  __shared__ uint32_t s_blist[kFlowWarps][kPart == 2 ? 1 : kBodyList];   // blocks of the loop being analysed
  __shared__ uint32_t s_lead[kFlowWarps][kPart == 1 ? kLeadWords : 1];   // leader flags (labels), one bit per statement
  __shared__ uint64_t s_lkey[kFlowWarps][kPart == 1 ? kLabSlots : 1];    // small label tables (2 KB per warp)
  __shared__ uint32_t s_lfirst[kFlowWarps][kPart == 1 ? kLabSlots : 1];
  __shared__ uint32_t s_llast[kFlowWarps][kPart == 1 ? kLabSlots : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(a.work + (kPart == 2 ? 1 : 0), 1ull);
    w = __shfl_sync(kAll, w, 0);
    if (w >= (unsigned long long)a.n_segs) break;
    const int64_t k = a.order ? (int64_t)a.order[w] : (int64_t)w;
    const FfbSegInfo inf = a.info[k];
    double* feat = a.feat + k * FFB_FEAT_WIDTH;
    if (kPart != 2 && lane < FFB_FEAT_WIDTH) feat[lane] = lane == FFB_F_OVR_TEXEC ? NAN : 0.0;
    uint32_t status = inf.status;
    FfbFlowInfo fi;
    fi.n_blocks = fi.n_edges = fi.n_loops = 0; fi.reserved = 0;
    uint32_t nb = 0, n_edges = 0, n_loops = 0;
    if (kPart == 2) {                                // the CFG kernel reported this PTX kernel's status already
      const FlowMid md = a.mid[k];
      if (md.status != FFB_OK) continue;
      nb = md.nb; n_edges = md.n_edges; n_loops = md.n_loops;
    } else if (status != FFB_OK) {
      if (lane == 0) {
        a.status[k] = status; if (a.flow) a.flow[k] = fi;
        if (kPart == 1) { FlowMid md; md.status = status; md.nb = md.n_edges = md.n_loops = 0; a.mid[k] = md; }
      }
      continue;
    }
    const uint32_t n = inf.n_instr, L = inf.n_labels;
    const int64_t ib = a.ins_base[k], lb = a.lab_base[k];
    const FfbInsRec* ins = a.ins + ib;
    const FfbLabelRec* lab = a.labels + lb;
    const uint32_t* cm = a.meta_arr ? a.meta_arr + ib : nullptr;        // compact meta stream
#define FFB_META(i) (cm ? cm[i] : ins[i].meta)
    const int64_t o1 = ib + 2 * k;                   // offset into the [N + 2K] arrays
    uint32_t* block_of = a.block_of + ib;
    uint32_t* block_start = a.block_start + o1;
    int32_t* succ0 = a.succ0 + o1;
    int32_t* succ1 = a.succ1 + o1;
    uint32_t* pred_ptr = a.pred_ptr + o1;
    uint32_t* pred_list = a.pred_list + 2 * o1;
    int32_t* rpo_num = a.rpo_num + o1;
    uint32_t* rpo_order = a.rpo_order + o1;
    int32_t* idom = a.idom + o1;
    uint32_t* mark = a.mark + o1;
    uint32_t* stack = a.stack + o1;
    double* weight = a.weight + o1;
    LabelTable lt;
    lt.key = a.lab_key + 4 * lb + 8 * k; lt.first = a.lab_first + 4 * lb + 8 * k; lt.last = a.lab_last + 4 * lb + 8 * k;
    lt.cap = 4; while (lt.cap < 2 * L + 2) lt.cap <<= 1;          // <= 4L + 8
    if (kPart == 1 && lt.cap <= (uint32_t)kLabSlots) {             // probed once per label, branch and loop: keep it on chip
      lt.key = s_lkey[wid]; lt.first = s_lfirst[wid]; lt.last = s_llast[wid];
    }
    CachedScales st;
    st.g.key = a.sc_key + 4 * ib + 8 * k; st.g.val = a.sc_val + 4 * ib + 8 * k;
    st.g.cap = 4; while (st.g.cap < 2 * n + 2) st.g.cap <<= 1;      // <= 4n + 8
    st.ckey = s_ckey[wid]; st.cval = s_cval[wid]; st.used = 0; st.spilled = false;

    if (kPart != 1) for (uint32_t i = lane; i < kMapSlots; i += 32) st.ckey[i] = 0;
    if (kPart != 2) {                                // ======== CFG, loops, trips, weights ========
    // ---- labels: last definition wins, dictionary order = first definition (ptx.py:234) ----
    for (uint32_t i = lane; i < lt.cap; i += 32) { lt.key[i] = 0; lt.first[i] = 0xffffffffu; lt.last[i] = 0; }
    // flow_kernel<1>, up to 32 * kLeadWords statements: the leader flags live in a shared-memory bit set and the
    // statements are visited once (meta word in, block number out) instead of a zero fill, two flag passes and a
    // read-back of block_of in HBM
    const bool lead_bits = kPart == 1 && n <= 32u * (uint32_t)kLeadWords;
    uint32_t* lbits = s_lead[wid];
    if (lead_bits) { for (uint32_t i = lane; i < (n + 31u) / 32u; i += 32) lbits[i] = 0; }
    else { for (uint32_t i = lane; i < n; i += 32) block_of[i] = 0; }
    __syncwarp();
    for (uint32_t i = lane; i < L; i += 32) {
      const uint64_t key = lab[i].hash + 1;
      uint32_t s = slot_of(lab[i].hash, lt.cap);
      for (;;) {
        const unsigned long long prev = atomicCAS((unsigned long long*)&lt.key[s], 0ull, (unsigned long long)key);
        if (prev == 0ull || prev == key) break;
        s = (s + 1) & (lt.cap - 1u);
      }
      atomicMin(&lt.first[s], i);
      atomicMax(&lt.last[s], i);
    }
    __syncwarp();
    // ---- leaders (cfg.py:63-70); block_of doubles as the flag array first ----
    for (uint32_t i = lane; i < L; i += 32) {
      const uint32_t s = lt.find(lab[i].hash);
      if (lt.last[s] == i && lab[i].index < n) {                               // effective definition only
        const uint32_t at = lab[i].index;
        if (lead_bits) atomicOr(&lbits[at >> 5], 1u << (at & 31u)); else block_of[at] = 1;
      }
    }
    if (!lead_bits) {
      for (uint32_t i = lane; i + 1 < n; i += 32) {
        const uint32_t m = FFB_META(i);
        const uint32_t base = ffb_meta_base(m);
        if (ffb_meta_cls(m) == FFB_CLS_BRANCH || base == FFB_BASE_RET || base == FFB_BASE_EXIT) block_of[i + 1] = 1;
      }
      if (lane == 0) block_of[0] = 1;
    }
    __syncwarp();
    nb = 0;
    if (lead_bits) {
      // four chunks of 32 statements per trip: the four meta loads are in flight together
      unsigned carry = 1u;                           // statement 0 is a leader; then: the previous chunk ended in a branch / ret / exit
      for (uint32_t c = 0; c < n; c += 128) {
        uint32_t m4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { const uint32_t i = c + 32u * u + lane; m4[u] = i < n ? FFB_META(i) : 0u; }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t cc = c + 32u * u;
          if (cc < n) {                              // warp-uniform
            const uint32_t i = cc + lane;
            const uint32_t m = m4[u], base = ffb_meta_base(m);
            const bool ends = i < n && (ffb_meta_cls(m) == FFB_CLS_BRANCH || base == FFB_BASE_RET || base == FFB_BASE_EXIT);
            const unsigned em = __ballot_sync(kAll, ends);
            unsigned lead = lbits[cc >> 5] | (em << 1) | carry;
            carry = em >> 31;
            if (n - cc < 32u) lead &= (1u << (n - cc)) - 1u;
            const uint32_t id = nb + __popc(lead & (0xffffffffu >> (31 - lane))) - 1;   // leaders at or before me
            if (i < n) block_of[i] = id;
            if ((lead >> lane) & 1u) block_start[id] = i;
            nb += __popc(lead);
          }
        }
      }
    } else
    for (uint32_t c = 0; c < n; c += 32) {
      const uint32_t i = c + lane;
      const bool f = i < n && block_of[i] != 0;
      const unsigned mask = __ballot_sync(kAll, f);
      const uint32_t id = nb + __popc(mask & (0xffffffffu >> (31 - lane))) - 1;   // leaders at or before me
      if (i < n) block_of[i] = id;
      if (f) block_start[id] = i;
      nb += __popc(mask);
    }
    if (lane == 0) block_start[nb] = n;
    for (uint32_t b = lane; b <= nb; b += 32) { pred_ptr[b] = 0; }
    __syncwarp();
    // ---- edges (cfg.py:80-92) and branch-target validation (ptx.py:277-284) ----
    bool bad_target = false;
    for (uint32_t b = lane; b < nb; b += 32) {
      const uint32_t li = block_start[b + 1] - 1;
      const uint32_t m = FFB_META(li);
      const uint32_t base = ffb_meta_base(m);
      int32_t t0 = -1, t1 = -1;
      if (ffb_meta_cls(m) == FFB_CLS_BRANCH) {
        const uint64_t tgt = ins[li].aux;
        const uint32_t s = tgt ? lt.find(ffb_op_hash(tgt)) : lt.cap;
        if (s == lt.cap) bad_target = true;
        else {
          const uint32_t tidx = lab[lt.last[s]].index;
          if (tidx < n) t0 = (int32_t)block_of[tidx];
          if (ffb_meta_has_pred(m) && b + 1 < nb) t1 = (int32_t)(b + 1);
        }
      } else if (base == FFB_BASE_RET || base == FFB_BASE_EXIT) {
      } else if (b + 1 < nb) {
        t1 = (int32_t)(b + 1);
      }
      succ0[b] = t0; succ1[b] = t1;
      if (t0 >= 0) atomicAdd(&pred_ptr[t0 + 1], 1u);
      if (t1 >= 0) atomicAdd(&pred_ptr[t1 + 1], 1u);
    }
    if (__any_sync(kAll, bad_target)) {
      if (lane == 0) {
        a.status[k] = FFB_E_MALFORMED_PTX; if (a.flow) a.flow[k] = fi;
        if (kPart == 1) { FlowMid md; md.status = FFB_E_MALFORMED_PTX; md.nb = md.n_edges = md.n_loops = 0; a.mid[k] = md; }
      }
      continue;
    }
    __syncwarp();
    n_edges = 0;
    {   // inclusive scan of pred_ptr[1..nb] in chunks of 32
      uint32_t carry = 0;
      for (uint32_t c = 1; c <= nb; c += 32) {
        const uint32_t i = c + lane;
        uint32_t v = i <= nb ? pred_ptr[i] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) { const uint32_t o = __shfl_up_sync(kAll, v, d); if (lane >= d) v += o; }
        if (i <= nb) pred_ptr[i] = v + carry;
        carry += __shfl_sync(kAll, v, 31);
      }
      n_edges = carry;
    }
    __syncwarp();
    for (uint32_t b = lane; b < nb; b += 32) mark[b] = pred_ptr[b];          // fill cursors
    __syncwarp();
    for (uint32_t b = lane; b < nb; b += 32) {
      if (succ0[b] >= 0) pred_list[atomicAdd(&mark[succ0[b]], 1u)] = b;
      if (succ1[b] >= 0) pred_list[atomicAdd(&mark[succ1[b]], 1u)] = b;
    }
    for (uint32_t b = lane; b < nb; b += 32) { rpo_num[b] = -1; idom[b] = -1; weight[b] = 1.0; }
    __syncwarp();
    for (uint32_t b = lane; b < nb; b += 32) mark[b] = 0;
    __syncwarp();
    // ---- lane 0: reverse post-order from block 0 and immediate dominators ----
    if (lane == 0) {
      uint32_t post = 0, sp = 0;
      stack[sp++] = 0; mark[0] = 1;          // mark: 0 unseen, 1 = next child is succ0, 2 = succ1, 3 = done
      while (sp) {
        const uint32_t b = stack[sp - 1];
        int32_t child = -1;
        while (mark[b] < 3 && child < 0) {
          const int32_t c = mark[b] == 1 ? succ0[b] : succ1[b];
          ++mark[b];
          if (c >= 0 && mark[c] == 0) child = c;
        }
        if (child >= 0) { mark[child] = 1; stack[sp++] = (uint32_t)child; }
        else { rpo_order[post++] = b; --sp; }
      }
      const uint32_t n_reach = post;
      for (uint32_t i = 0; i < n_reach; ++i) rpo_num[rpo_order[i]] = (int32_t)(n_reach - 1 - i);   // 0 = entry
      idom[0] = 0;
      for (bool changed = true; changed;) {
        changed = false;
        for (int32_t r = (int32_t)n_reach - 2; r >= 0; --r) {            // reverse post-order, entry skipped
          const uint32_t b = rpo_order[r];
          int32_t nd = -1;
          for (uint32_t p = pred_ptr[b]; p < pred_ptr[b + 1]; ++p) {
            const uint32_t q = pred_list[p];
            if (rpo_num[q] < 0 || idom[q] < 0) continue;
            if (nd < 0) { nd = (int32_t)q; continue; }
            int32_t x = (int32_t)q, y = nd;
            while (x != y) {
              while (rpo_num[x] > rpo_num[y]) x = idom[x];
              while (rpo_num[y] > rpo_num[x]) y = idom[y];
            }
            nd = x;
          }
          if (nd != idom[b]) { idom[b] = nd; changed = true; }
        }
      }
    }
    __syncwarp();
    for (uint32_t b = lane; b < nb; b += 32) mark[b] = 0;
    __syncwarp();
    // ---- natural loops, one per header in ascending header order (cfg.py:124-151) ----
    n_loops = 0;
    for (uint32_t h = 0; h < nb; ++h) {
      const uint32_t stamp = h + 1;
      int is_header = 0;
      if (lane == 0) {
        for (uint32_t p = pred_ptr[h]; p < pred_ptr[h + 1]; ++p) {
          const uint32_t u = pred_list[p];
          if (!dominates(idom, rpo_num, h, u)) continue;
          is_header = 1;
          mark[h] = stamp;                      // body = {h, u} + everything that reaches u without passing h
          mark[u] = stamp;
          uint32_t top = 0;
          stack[top++] = u;
          while (top) {
            const uint32_t x = stack[--top];
            if (x == h) continue;
            for (uint32_t q = pred_ptr[x]; q < pred_ptr[x + 1]; ++q) {
              const uint32_t y = pred_list[q];
              if (mark[y] != stamp) { mark[y] = stamp; stack[top++] = y; }
            }
          }
        }
      }
      is_header = __shfl_sync(kAll, is_header, 0);
      if (!is_header) continue;
      __syncwarp();
      const uint32_t h0 = block_start[h];
      // compact list of the body's blocks: the scans of the trip recogniser visit these only
      // (bodies with more than kBodyList blocks fall back to testing every block's mark)
      uint32_t* blist = s_blist[wid];
      uint32_t n_bl = 0;
      for (uint32_t b0 = 0; b0 < nb; b0 += 32) {
        const uint32_t b = b0 + lane;
        const bool in = b < nb && mark[b] == stamp;
        const unsigned msk = __ballot_sync(kAll, in);
        if (in) { const uint32_t at = n_bl + __popc(msk & ((1u << lane) - 1u)); if (at < (uint32_t)kBodyList) blist[at] = b; }
        n_bl += __popc(msk);
      }
      const bool bl_ok = n_bl <= (uint32_t)kBodyList;
      const uint32_t n_scan = bl_ok ? n_bl : nb;
      __syncwarp();
      // header label: the dictionary's last name that maps to the header's first instruction
      int64_t best = -1;                        // (first-definition order << 32) | record index
      for (uint32_t i = lane; i < L; i += 32) {
        const uint32_t s = lt.find(lab[i].hash);
        if (lt.last[s] != i || lab[i].index != h0) continue;       // only effective definitions
        const int64_t cand = ((int64_t)lt.first[s] << 32) | (int64_t)i;
        best = cand > best ? cand : best;
      }
      best = warp_max_i64(best);
      const bool hl_any = best >= 0;
      const uint64_t hl_hash = hl_any ? lab[(uint32_t)(best & 0xffffffff)].hash : 0;
      const uint32_t hl_off = hl_any ? lab[(uint32_t)(best >> 32)].off : 0;
      // ---- trip count ----
      double trip = -1.0;
      bool annotated = false;
      if (hl_any) {
        for (int q = 0; q < a.n_ann; ++q)
          if (a.ann_hash[q] == hl_hash) { trip = a.ann_trip[q]; annotated = true; if (a.ann_hit && lane == 0) a.ann_hit[q] = 1; }
      }
      if (!annotated) {
        // cfg.py:191-279; "last match in the body" = maximum index over the body's statements
        bool ok = true;
        int64_t latch = -1;
        for (uint32_t bi = 0; bi < n_scan; ++bi) {
          const uint32_t b = bl_ok ? blist[bi] : bi;
          if (!bl_ok && mark[b] != stamp) continue;
          for (uint32_t i = block_start[b] + lane; i < block_start[b + 1]; i += 32) {
            const uint32_t m = FFB_META(i);
            if (ffb_meta_cls(m) == FFB_CLS_BRANCH && ffb_meta_has_pred(m)) {
              const uint32_t s = lt.find(ffb_op_hash(ins[i].aux));
              if (lab[lt.last[s]].index == h0) latch = i;
            }
          }
        }
        latch = warp_max_i64(latch);
        int64_t cmp_i = -1;
        if (latch < 0) ok = false;
        if (ok) {
          const uint64_t preg = ins[latch].pred;
          for (uint32_t bi = 0; bi < n_scan; ++bi) {
            const uint32_t b = bl_ok ? blist[bi] : bi;
            if (!bl_ok && mark[b] != stamp) continue;
            for (uint32_t i = block_start[b] + lane; i < block_start[b + 1]; i += 32) {
              const uint32_t m = FFB_META(i);
              if (ffb_meta_base(m) == FFB_BASE_SETP && ffb_meta_nops(m) >= 1) {
                const uint64_t d0 = ins[i].op[0];
                if (ffb_op_kind(d0) != FFB_OPK_INT && ffb_op_hash(d0) == preg) cmp_i = i;
              }
            }
          }
          cmp_i = warp_max_i64(cmp_i);
          if (cmp_i < 0 || ffb_meta_nops(FFB_META(cmp_i)) < 3) ok = false;
        }
        uint64_t counter = 0; int64_t bound = 0; uint32_t rel = FFB_CMP_NONE;
        if (ok) {
          const FfbInsRec& c = ins[cmp_i];
          counter = c.op[1];
          if (!starts_with_percent(counter)) ok = false;
          if (ok && ffb_op_kind(c.op[2]) == FFB_OPK_BIGINT) { ok = false; status = FFB_E_CAPACITY; }
          if (ok && ffb_op_kind(c.op[2]) != FFB_OPK_INT) ok = false;
          if (ok) bound = ffb_op_int(c.op[2]);
          rel = ffb_meta_cmp(c.meta);
          if (rel == FFB_CMP_NONE) ok = false;
          if (ok && ffb_meta_pred_neg(ins[latch].meta)) {
            const uint32_t inv[7] = {0, FFB_CMP_GE, FFB_CMP_LT, FFB_CMP_GT, FFB_CMP_LE, FFB_CMP_NE, FFB_CMP_EQ};
            rel = inv[rel];
          }
        }
        int64_t stride = 0;
        if (ok) {
          // exactly one `add/sub counter, counter, <int literal>` in the body (cfg.py:229-240)
          const uint64_t ch = ffb_op_hash(counter);
          int n_upd = 0, n_bad = 0, n_big = 0;
          int64_t my_stride = 0;
          for (uint32_t bi = 0; bi < n_scan; ++bi) {
            const uint32_t b = bl_ok ? blist[bi] : bi;
            if (!bl_ok && mark[b] != stamp) continue;
            for (uint32_t i = block_start[b] + lane; i < block_start[b + 1]; i += 32) {
              const uint32_t m = FFB_META(i);
              const uint32_t base = ffb_meta_base(m);
              if ((base == FFB_BASE_ADD || base == FFB_BASE_SUB) && ffb_meta_nops(m) == 3 && ffb_meta_dst_reg(m)) {
                const FfbInsRec& r = ins[i];
                if (ffb_op_hash(r.op[0]) == ch && starts_with_percent(r.op[1]) && ffb_op_hash(r.op[1]) == ch) {
                  ++n_upd;
                  if (ffb_op_kind(r.op[2]) == FFB_OPK_BIGINT) ++n_big;
                  else if (ffb_op_kind(r.op[2]) != FFB_OPK_INT) ++n_bad;
                  else my_stride = base == FFB_BASE_SUB ? -ffb_op_int(r.op[2]) : ffb_op_int(r.op[2]);
                }
              }
            }
          }
          n_upd = warp_sum_i(n_upd); n_bad = warp_sum_i(n_bad); n_big = warp_sum_i(n_big);
          if (n_big) status = FFB_E_CAPACITY;
          if (n_upd != 1 || n_bad || n_big) ok = false;
          else {
            // the single matching lane holds the stride; others hold 0
            stride = my_stride;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) stride += __shfl_xor_sync(kAll, stride, d);
            if (stride == 0) ok = false;
          }
        }
        int64_t init = 0;
        if (ok) {
          // the LAST write to the counter before the header decides (cfg.py:246-254)
          const uint64_t ch = ffb_op_hash(counter);
          int64_t found = -1;
          for (int64_t hi = (int64_t)h0; hi > 0 && found < 0; hi -= 32) {
            const int64_t i = hi - 1 - lane;                     // lane 0 looks at the latest statement
            bool hit = false;
            if (i >= 0) {
              const uint32_t m = FFB_META(i);
              if (ffb_meta_nops(m) != 0 && ffb_meta_dst_reg(m)) hit = ffb_op_hash(ins[i].op[0]) == ch;
            }
            const unsigned mask = __ballot_sync(kAll, hit);
            if (mask) found = hi - 1 - (__ffs((int)mask) - 1);
          }
          bool have_init = false;
          if (found >= 0) {
            const FfbInsRec& r = ins[found];
            if (ffb_meta_base(r.meta) == FFB_BASE_MOV && ffb_meta_nops(r.meta) == 2) {
              if (ffb_op_kind(r.op[1]) == FFB_OPK_INT) { init = ffb_op_int(r.op[1]); have_init = true; }
              else if (ffb_op_kind(r.op[1]) == FFB_OPK_BIGINT) status = FFB_E_CAPACITY;
            }
          }
          if (!have_init) ok = false;
        }
        if (ok) {
          // cfg.py:259-279, Python int arithmetic: "/" is true division, then ceil / floor
          double trips = 0.0;
          const double span_up = (double)(bound - init), span_dn = (double)(init - bound);
          if (rel == FFB_CMP_LT && stride > 0) trips = ceil(span_up / (double)stride);
          else if (rel == FFB_CMP_LE && stride > 0) trips = floor(span_up / (double)stride) + 1.0;
          else if (rel == FFB_CMP_GT && stride < 0) trips = ceil(span_dn / (double)(-stride));
          else if (rel == FFB_CMP_GE && stride < 0) trips = floor(span_dn / (double)(-stride)) + 1.0;
          else if (rel == FFB_CMP_NE) {
            const int64_t span = bound - init;
            if (span % stride == 0 && span / stride > 0) trips = (double)(span / stride);
            else ok = false;
          } else ok = false;
          if (ok) trip = trips < 1.0 ? 1.0 : trips;
        }
        if (!ok) trip = a.default_trip;
      }
      if (!(trip > 1.0)) trip = 1.0;                                  // cfg.py:181 max(1.0, trip)
      int n_body = 0;
      for (uint32_t b = lane; b < nb; b += 32)
        if (mark[b] == stamp) { weight[b] *= trip; ++n_body; }       // cfg.py:52-53
      n_body = warp_sum_i(n_body);
      if (a.out_loops) {
        if (lane == 0) {
          FfbLoopRec lr;
          lr.header = h; lr.n_body = (uint32_t)n_body; lr.trip = trip; lr.label_hash = hl_any ? hl_hash : 0;
          lr.label_off = hl_off; lr.has_label = hl_any ? 1u : 0u;
          a.out_loops[o1 + n_loops] = lr;
        }
        if (a.out_loop_body && (int64_t)(n_loops + 1) * nb <= a.loop_body_cap)
          for (uint32_t b = lane; b < nb; b += 32) a.out_loop_body[(int64_t)n_loops * nb + b] = mark[b] == stamp ? 1 : 0;
      }
      ++n_loops;
      __syncwarp();
    }
    __syncwarp();
    }                                                // ======== end of the CFG part ========
    if (kPart == 1) {
      // trip errors are warp-uniform, but the OR costs nothing; the scratch writes of this warp are ordered
      // before the next launch by the kernel boundary
      uint32_t st_all = status;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) st_all |= __shfl_xor_sync(kAll, st_all, d);
      if (lane == 0) {
        FlowMid md; md.status = st_all; md.nb = nb; md.n_edges = n_edges; md.n_loops = n_loops; a.mid[k] = md;
        if (st_all != FFB_OK) { a.status[k] = st_all; if (a.flow) { fi.n_blocks = nb; fi.n_edges = n_edges; fi.n_loops = n_loops; a.flow[k] = fi; } }
      }
      continue;
    }
    // ---- one textual pass: affine scales, aligned fraction, dynamic counts ----
    // Parallel form: 32 statements per round, one per lane.  A chunk-local table maps every register
    // the chunk defines to the mask of defining lanes, so a source is either "before the chunk" (looked
    // up in the shared-memory map, all lanes at once) or "lane j of this chunk" (read after j has
    // published); dependent statements resolve in waves.  The last definer of each name updates the
    // map.  The sums are accumulated per lane and reduced at the end, which is bit-identical to the
    // reference's in-order sums whenever every partial sum is exactly representable (all weights on
    // a 1/64 grid and the totals below 2^44 - checked here); otherwise, or when the kernel names more
    // registers than the on-chip map holds, the pass continues sequentially on lane 0.
    Sums acc;
    acc.n_mem = acc.mem_bytes = acc.u_fp = acc.u_int = acc.u_sfu = acc.u_alu = acc.n_sync = acc.al_hit = acc.al_tot = 0.0;
    bool exact_sums = true;
    {
      double wmax = 0.0;
      for (uint32_t b = lane; b < nb; b += 32) {
        const double w = weight[b], w64 = w * 64.0;
        if (!(w64 == floor(w64))) exact_sums = false;
        wmax = w > wmax ? w : wmax;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) { const double o = __shfl_xor_sync(kAll, wmax, d); wmax = o > wmax ? o : wmax; }
      exact_sums = !__any_sync(kAll, !exact_sums) && wmax * (double)n * 64.0 < 17592186044416.0;     // 2^44
    }
    uint32_t c0 = 0;
    uint32_t used = 0;                               // names in the on-chip map (warp-uniform)
    uint64_t* ch_key = s_chkey[wid];
    uint32_t* ch_mask = s_chmask[wid];
    int64_t* ch_val = s_chval[wid];
    const unsigned lt_lanes = (1u << lane) - 1u;
    for (; a.parallel_pass && exact_sums && c0 < n && used + 32 <= kMapFill; c0 += 32) {
      const uint32_t cnt = n - c0 < 32 ? n - c0 : 32;
      const bool live = (uint32_t)lane < cnt;
      ch_key[lane] = 0; ch_key[lane + 32] = 0; ch_mask[lane] = 0; ch_mask[lane + 32] = 0;
      uint32_t m = 0;
      uint64_t op0 = 0, op1 = 0, op2 = 0, op3 = 0, aux = 0;
      double wgt = 0.0;
      if (live) {
        const uint4* src = reinterpret_cast<const uint4*>(ins + c0 + lane);
        const uint4 q0 = src[0], q1 = src[1], q2 = src[2], q3 = src[3];
        m = q0.x;
        aux = (uint64_t)q1.z | ((uint64_t)q1.w << 32);
        op0 = (uint64_t)q2.x | ((uint64_t)q2.y << 32); op1 = (uint64_t)q2.z | ((uint64_t)q2.w << 32);
        op2 = (uint64_t)q3.x | ((uint64_t)q3.y << 32); op3 = (uint64_t)q3.z | ((uint64_t)q3.w << 32);
        wgt = weight[block_of[c0 + lane]];
      }
      const uint32_t cls = ffb_meta_cls(m), nops = ffb_meta_nops(m);
      const bool is_mem = cls == FFB_CLS_MEMLOAD || cls == FFB_CLS_MEMSTORE;
      // does this statement define a name?  (alignment.py:84-95)
      bool defines = live && nops >= 1 && ffb_meta_dst_reg(m) && (is_mem ? cls == FFB_CLS_MEMLOAD : ffb_meta_base(m) != FFB_BASE_SETP);
      const uint64_t dh = ffb_op_hash(op0);
      __syncwarp();
      uint32_t my_slot = 0;
      if (defines) {
        uint32_t s = slot_of(dh, 64);
        for (;;) {
          const unsigned long long prev = atomicCAS((unsigned long long*)&ch_key[s], 0ull, (unsigned long long)(dh + 1));
          if (prev == 0ull || prev == dh + 1) break;
          s = (s + 1) & 63u;
        }
        atomicOr(&ch_mask[s], 1u << lane);
        my_slot = s;
      }
      __syncwarp();
      // sources: operands 1..3 and aux
      SrcScales sc;
      int p1 = -1, p2 = -1, p3 = -1, pa = -1;
      unsigned deps = 0;
#define FFB_RESOLVE(D, S, P)                                                                      \
      {                                                                                           \
        const uint64_t kd = ffb_op_kind(D);                                                       \
        S = kd == FFB_OPK_TIDX ? 1 : ((kd == FFB_OPK_UNKNOWN || kd == FFB_OPK_NONE || kd == FFB_OPK_REG) ? kNoneScale : 0); \
        if (live && kd == FFB_OPK_REG) {                                                          \
          const uint64_t h = ffb_op_hash(D);                                                      \
          uint32_t s = slot_of(h, 64);                                                            \
          unsigned defs = 0;                                                                      \
          for (;;) {                                                                              \
            const uint64_t k = ch_key[s];                                                         \
            if (k == h + 1) { defs = ch_mask[s] & lt_lanes; break; }                              \
            if (k == 0) break;                                                                    \
            s = (s + 1) & 63u;                                                                    \
          }                                                                                       \
          if (defs) { P = 31 - __clz((int)defs); deps |= 1u << P; }                               \
          else S = st.get(h);                                                                     \
        }                                                                                         \
      }
      // a memory statement reads one scale only - the address register of a global access (alignment.py:137-144);
      // what it defines does not depend on its operands (:84-88).  Everything else may read all four.
      const bool wants_addr = is_mem && ffb_meta_space(m) == FFB_SP_GLOBAL && ffb_meta_addr(m) == FFB_ADDR_REG;
      sc.s1 = sc.s2 = sc.s3 = sc.sa = kNoneScale;
      if (!is_mem && defines) {
        FFB_RESOLVE(op1, sc.s1, p1)
        FFB_RESOLVE(op2, sc.s2, p2)
        FFB_RESOLVE(op3, sc.s3, p3)
      }
      if (wants_addr || (!is_mem && defines)) FFB_RESOLVE(aux, sc.sa, pa)
#undef FFB_RESOLVE
      // statements whose contribution needs no scale are counted here, once, with all lanes together
      if (live && !wants_addr) count_statement(m, wgt, kNoneScale, acc);
      // waves: a statement runs once the lanes it depends on have published
      bool mine_done = !live;
      int64_t v = kNoneScale;
      unsigned done_mask = __ballot_sync(kAll, mine_done);
      while (done_mask != kAll) {
        if (!mine_done && (deps & ~done_mask) == 0) {
          if (p1 >= 0) sc.s1 = ch_val[p1];
          if (p2 >= 0) sc.s2 = ch_val[p2];
          if (p3 >= 0) sc.s3 = ch_val[p3];
          if (pa >= 0) sc.sa = ch_val[pa];
          if (is_mem) v = ffb_meta_space(m) == FFB_SP_PARAM ? 0 : kNoneScale;            // alignment.py:84-88
          else if (defines) defines = eval_def(m, op1, op2, op3, sc, &v, &status);
          if (defines) ch_val[lane] = v;
          if (wants_addr) count_statement(m, wgt, sc.sa, acc);
          mine_done = true;
        }
        __syncwarp();
        done_mask = __ballot_sync(kAll, mine_done);
      }
      // the last definer of each name updates the map
      bool fresh = false;
      if (defines && (ch_mask[my_slot] >> lane) == 1u) {
        uint32_t c = slot_of(dh, kMapSlots);
        for (;;) {
          const unsigned long long k = st.ckey[c];
          if (k == dh + 1) break;
          if (k == 0) {
            const unsigned long long prev = atomicCAS((unsigned long long*)&st.ckey[c], 0ull, (unsigned long long)(dh + 1));
            if (prev == 0ull) { fresh = true; break; }
            if (prev == dh + 1) break;
          }
          c = (c + 1) & (kMapSlots - 1);
        }
        st.cval[c] = v;
      }
      used += __popc(__ballot_sync(kAll, fresh));
      __syncwarp();
    }
    // totals of the parallel part (exact, so the order of the additions does not matter)
    double n_mem = warp_sum_d(acc.n_mem), mem_bytes = warp_sum_d(acc.mem_bytes), u_fp = warp_sum_d(acc.u_fp), u_int = warp_sum_d(acc.u_int),
           u_sfu = warp_sum_d(acc.u_sfu), u_alu = warp_sum_d(acc.u_alu), n_sync = warp_sum_d(acc.n_sync);
    double al_hit = warp_sum_d(acc.al_hit), al_tot = warp_sum_d(acc.al_tot);
    {
      unsigned sor = status;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) sor |= __shfl_xor_sync(kAll, sor, d);
      status = sor;
    }
    st.used = used;
    // sequential remainder (all of the kernel when the parallel form does not apply)
    for (; c0 < n; c0 += 32) {
      const uint32_t cnt = n - c0 < 32 ? n - c0 : 32;
      if (lane == 0) {                                 // (records straight from HBM: this form is the rare one)
        Sums sq;
        sq.n_mem = n_mem; sq.mem_bytes = mem_bytes; sq.u_fp = u_fp; sq.u_int = u_int; sq.u_sfu = u_sfu; sq.u_alu = u_alu;
        sq.n_sync = n_sync; sq.al_hit = al_hit; sq.al_tot = al_tot;
        for (uint32_t q0 = 0; q0 < cnt; ++q0) {
          const FfbInsRec r = ins[c0 + q0];
          const uint32_t m = r.meta, cls = ffb_meta_cls(m), nops = ffb_meta_nops(m);
          const double wgt = weight[block_of[c0 + q0]];
          const bool is_mem = cls == FFB_CLS_MEMLOAD || cls == FFB_CLS_MEMSTORE;
          if (is_mem) {
            const int64_t sa = (ffb_meta_space(m) == FFB_SP_GLOBAL && ffb_meta_addr(m) == FFB_ADDR_REG) ? st.get(ffb_op_hash(r.aux)) : kNoneScale;
            count_statement(m, wgt, sa, sq);
            if (cls == FFB_CLS_MEMLOAD && nops >= 1 && ffb_meta_dst_reg(m))                    // alignment.py:84-88
              st.put(ffb_op_hash(r.op[0]), ffb_meta_space(m) == FFB_SP_PARAM ? 0 : kNoneScale);
            continue;
          }
          count_statement(m, wgt, kNoneScale, sq);
          if (nops == 0 || !ffb_meta_dst_reg(m)) continue;                                      // alignment.py:91-95
          SrcScales sc;
          sc.s1 = operand_scale_c(r.op[1], st); sc.s2 = operand_scale_c(r.op[2], st);
          sc.s3 = operand_scale_c(r.op[3], st); sc.sa = operand_scale_c(r.aux, st);
          int64_t v;
          if (eval_def(m, r.op[1], r.op[2], r.op[3], sc, &v, &status)) st.put(ffb_op_hash(r.op[0]), v);
        }
        n_mem = sq.n_mem; mem_bytes = sq.mem_bytes; u_fp = sq.u_fp; u_int = sq.u_int; u_sfu = sq.u_sfu; u_alu = sq.u_alu;
        n_sync = sq.n_sync; al_hit = sq.al_hit; al_tot = sq.al_tot;
      }
      __syncwarp();
    }
    status = __shfl_sync(kAll, status, 0) | status;      // lane 0 owns the dataflow errors; trip errors are uniform
    if (lane == 0) {
      feat[FFB_F_N_MEM] = n_mem; feat[FFB_F_MEM_BYTES] = mem_bytes;
      feat[FFB_F_FP32] = u_fp; feat[FFB_F_INT] = u_int; feat[FFB_F_SFU] = u_sfu; feat[FFB_F_ALU] = u_alu;
      feat[FFB_F_N_SYNC] = n_sync;
      feat[FFB_F_ALIGNED] = al_tot == 0.0 ? 1.0 : al_hit / al_tot;                            // alignment.py:145-147
      feat[FFB_F_STATIC_SHARED] = (double)inf.static_shared;
      feat[FFB_F_REGS_DECLARED] = (double)inf.regs_declared;
      feat[FFB_F_N_INSTR] = (double)n;
      a.status[k] = status;
      fi.n_blocks = nb; fi.n_edges = n_edges; fi.n_loops = n_loops;
      if (a.flow) a.flow[k] = fi;
    }
    if (a.out_block_start) for (uint32_t b = lane; b <= nb; b += 32) a.out_block_start[o1 + b] = block_start[b];
    if (a.out_weights) for (uint32_t b = lane; b < nb; b += 32) a.out_weights[o1 + b] = weight[b];
    if (a.out_edges && lane == 0) {
      uint32_t e = 0;
      for (uint32_t b = 0; b < nb; ++b) {
        if (succ0[b] >= 0) { a.out_edges[2 * (2 * o1 + e)] = (int32_t)b; a.out_edges[2 * (2 * o1 + e) + 1] = succ0[b]; ++e; }
        if (succ1[b] >= 0) { a.out_edges[2 * (2 * o1 + e)] = (int32_t)b; a.out_edges[2 * (2 * o1 + e) + 1] = succ1[b]; ++e; }
      }
    }
    __syncwarp();
  }
}

}  // namespace

extern "C" int32_t ffb_kernel_features(FfbContext* ctx, const FfbFlowDesc* d, void* stream_) {
  if (!ctx || !d || d->n_segs < 0 || !d->d_info || !d->d_ins_base || !d->d_lab_base || !d->d_ins || !d->d_labels ||
      !d->d_feat || !d->d_status || d->n_ins_total < 0 || d->n_lab_total < 0)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_kernel_features: bad argument");
  if (d->n_segs == 0) return FFB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));
  const int64_t K = d->n_segs, N = d->n_ins_total, L = d->n_lab_total;
  const size_t n1 = (size_t)(N + 2 * K + 8);       // block-indexed arrays
  const size_t nL = (size_t)(4 * L + 8 * K + 16), nS = (size_t)(4 * N + 8 * K + 16);
  size_t bytes = 0;
  auto take = [&](size_t count, size_t elem) { size_t off = bytes; bytes += (count * elem + 15) & ~(size_t)15; return off; };
  const size_t o_block_of = take((size_t)N + 8, 4), o_bstart = take(n1, 4), o_s0 = take(n1, 4), o_s1 = take(n1, 4),
               o_pp = take(n1, 4), o_pl = take(2 * n1, 4), o_rn = take(n1, 4), o_ro = take(n1, 4), o_id = take(n1, 4),
               o_mk = take(n1, 4), o_sk = take(n1, 4), o_w = take(n1, 8), o_lk = take(nL, 8), o_lf = take(nL, 4),
               o_ll = take(nL, 4), o_sk2 = take(nS, 8), o_sv = take(nS, 8),
               o_ah = take((size_t)(d->n_ann > 0 ? d->n_ann : 1), 8), o_at = take((size_t)(d->n_ann > 0 ? d->n_ann : 1), 8),
               o_work = take(2, 8), o_mid = take((size_t)K, sizeof(FlowMid));
  int32_t rc = ffb_reserve(ctx, &ctx->d_flow, bytes);
  if (rc) return rc;
  char* base = (char*)ctx->d_flow.p;
  FlowArgs a = {};
  a.n_segs = K; a.info = d->d_info; a.ins_base = d->d_ins_base; a.lab_base = d->d_lab_base;
  a.ins = (const FfbInsRec*)d->d_ins; a.labels = (const FfbLabelRec*)d->d_labels; a.order = d->d_order;
  a.meta_arr = d->d_meta;
  a.default_trip = d->default_trip;
  a.parallel_pass = (d->flags & FFB_FLOW_SEQUENTIAL_PASS) ? 0 : 1;
  a.n_ann = d->n_ann > 0 ? d->n_ann : 0; a.ann_hit = d->d_ann_hit;
  a.feat = d->d_feat; a.status = d->d_status; a.flow = d->d_flow;
  a.block_of = (uint32_t*)(base + o_block_of); a.block_start = (uint32_t*)(base + o_bstart);
  a.succ0 = (int32_t*)(base + o_s0); a.succ1 = (int32_t*)(base + o_s1);
  a.pred_ptr = (uint32_t*)(base + o_pp); a.pred_list = (uint32_t*)(base + o_pl);
  a.rpo_num = (int32_t*)(base + o_rn); a.rpo_order = (uint32_t*)(base + o_ro); a.idom = (int32_t*)(base + o_id);
  a.mark = (uint32_t*)(base + o_mk); a.stack = (uint32_t*)(base + o_sk); a.weight = (double*)(base + o_w);
  a.lab_key = (uint64_t*)(base + o_lk); a.lab_first = (uint32_t*)(base + o_lf); a.lab_last = (uint32_t*)(base + o_ll);
  a.sc_key = (uint64_t*)(base + o_sk2); a.sc_val = (int64_t*)(base + o_sv);
  a.ann_hash = (const uint64_t*)(base + o_ah); a.ann_trip = (const double*)(base + o_at);
  a.work = (unsigned long long*)(base + o_work);
  a.mid = (FlowMid*)(base + o_mid);
  FFB_CUDA(ctx, cudaMemsetAsync(a.work, 0, 16, stream));
  if (a.n_ann > 0) {
    if (!d->h_ann_hash || !d->h_ann_trip) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_kernel_features: annotation arrays missing");
    rc = ffb_stage_reserve(ctx, (size_t)a.n_ann * 16);
    if (rc) return rc;
    memcpy(ctx->h_stage, d->h_ann_hash, (size_t)a.n_ann * 8);
    memcpy((char*)ctx->h_stage + (size_t)a.n_ann * 8, d->h_ann_trip, (size_t)a.n_ann * 8);
    FFB_CUDA(ctx, cudaMemcpyAsync(base + o_ah, ctx->h_stage, (size_t)a.n_ann * 8, cudaMemcpyHostToDevice, stream));
    FFB_CUDA(ctx, cudaMemcpyAsync(base + o_at, (char*)ctx->h_stage + (size_t)a.n_ann * 8, (size_t)a.n_ann * 8, cudaMemcpyHostToDevice, stream));
    FFB_CUDA(ctx, cudaEventRecord(ctx->stage_free, stream));
    ctx->stage_busy = true;
  }
  a.out_block_start = d->d_block_start; a.out_edges = d->d_edges; a.out_loops = d->d_loops;
  a.out_loop_body = d->d_loop_body; a.loop_body_cap = d->loop_body_cap; a.out_weights = d->d_weights;
  int64_t ctas = (K + kFlowWarps - 1) / kFlowWarps;
  const int64_t max_ctas = (int64_t)ctx->sm_count * 16;
  if (ctas > max_ctas) ctas = max_ctas;
  const bool detail = d->d_flow || d->d_block_start || d->d_edges || d->d_loops || d->d_loop_body || d->d_weights || a.n_ann > 0;
  if (detail || (d->flags & FFB_FLOW_ONE_KERNEL)) {
    FFB_LAUNCH(flow_kernel<0>, (unsigned)ctas, kFlowWarps * 32, 0, stream, a);
    return ffb_check_launch(ctx, "flow_kernel");
  }
  FFB_LAUNCH(flow_kernel<1>, (unsigned)ctas, kFlowWarps * 32, 0, stream, a);
  rc = ffb_check_launch(ctx, "flow_kernel<cfg>");
  if (rc) return rc;
  FFB_LAUNCH(flow_kernel<2>, (unsigned)ctas, kFlowWarps * 32, 0, stream, a);
  return ffb_check_launch(ctx, "flow_kernel<dataflow>");
}

// Name hash used for annotation keys (same function as the lexer's label hash).
extern "C" uint64_t ffb_name_hash(const uint8_t* name, int64_t len) {
  FfbHasher x;
  ffb_hash_init(x);
  for (int64_t i = 0; i < len; ++i) ffb_hash_byte(x, name[i]);
  return ffb_hash_done(x);
}
