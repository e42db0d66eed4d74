// K4: Pareto skyline in (energy, time).
//
// Reference rule restated (explorer.py:122-140, :209-212): after the throughput floor
// t <= t_peak / rho, a point is dropped iff another point has STRICTLY lower e and
// STRICTLY lower t; equal points and partial ties all stay; the front is reported in
// (e, t, tie) order where tie reproduces the reference's (block_x, block_y, p_cap) key.
//
// One CTA owns one group of candidates:
//   1. stream the group's (e, t) from HBM into shared memory (the only DRAM traffic:
//      16 B per candidate), reducing min t on the way;
//   2. floor, then a 256-bucket histogram of min-t over the e range and its exclusive
//      prefix-min: a point whose lower-e buckets already hold a smaller t is provably
//      dominated (buckets are monotone in e, so "lower bucket" implies "strictly lower e");
//   3. the few survivors (every true front member survives) are bitonic-sorted by the
//      reference key and filtered exactly with a prefix-min over strictly-lower-e groups,
//      evaluated with warp-shuffle scans — the sort-based skyline of north_star (4).
// Large single sets (BASELINE config 5) reuse the same kernel hierarchically: fronts of
// 4096-point chunks are appended to a compact buffer and reduced again until one group is
// left; exact because strict dominance is transitive.
#include "ffb_common.cuh"
#include <stdlib.h>

#include <math.h>
#include <string.h>
#include <type_traits>

namespace {

constexpr int kThreads = 512;
constexpr int kBuckets = 256;
constexpr uint32_t kPad = 0xffffffffu;

FFB_HD uint64_t ordered_bits(double v) {
  // monotone map double -> uint64 (total order on non-NaN values)
#if defined(__CUDA_ARCH__) || defined(FFB_SIMT_EMUL)
  uint64_t b = (uint64_t)__double_as_longlong(v);
#else
  uint64_t b; memcpy(&b, &v, 8);
#endif
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

struct SkyArgs {
  const double* e;
  const double* t;
  const uint64_t* id;       // optional per-point id (tie-break + compact output)
  const double* occ;        // optional third objective (higher is better): see step 6b
  double* out_occ;          // compact output of occ (hierarchical passes)
  const uint32_t* tie;      // optional [group_size] tie rank
  int64_t n_total;          // total points (last group may be short)
  int64_t group_size;
  double rho;               // <= 0: no floor
  int resident;             // points staged in shared memory
  int surv_cap;             // survivor capacity (entries of s_pm / s_gs)
  int sort_cap;             // power of two >= surv_cap (entries of s_idx)
  int surv_bytes;           // bytes of the survivor region: max(surv_cap * 12 for s_pm + s_gs, sort_cap * 8 for the sort keys)
  int tie_smem;             // tie ranks staged in shared memory as u16
  // per-group outputs (optional)
  uint32_t* front_idx;
  uint32_t* front_n;
  double* tpeak;
  int64_t cap_front;
  int64_t* front_off;       // optional: compact mode, offset of each group's run in front_idx
  unsigned long long* front_total;   // compact mode: running total (atomic)
  // compact outputs (optional): appended at an atomically reserved offset
  double* out_e;
  double* out_t;
  uint64_t* out_id;
  unsigned long long* out_count;
  int64_t out_cap;
  uint32_t* status;
};

template <typename T, typename Op>
FFB_D T warp_scan_incl(T v, Op op, T ident) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v = op(v, o);
  }
  (void)ident;
  return v;
}

// In-place inclusive scan of arr[0..n) by the whole CTA. part: kThreads scratch entries.
template <typename T, typename Op>
FFB_D void block_scan_incl(T* arr, int n, T* part, Op op, T ident) {
  const int tid = threadIdx.x;
  const int per = (n + kThreads - 1) / kThreads;
  const int lo = tid * per;
  const int hi = lo + per < n ? lo + per : n;
  T acc = ident;
  for (int i = lo; i < hi; ++i) { acc = op(acc, arr[i]); arr[i] = acc; }
  T incl = warp_scan_incl(acc, op, ident);
  const int lane = tid & 31, wid = tid >> 5;
  if (lane == 31) part[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    T w = lane < kThreads / 32 ? part[lane] : ident;
    w = warp_scan_incl(w, op, ident);
    if (lane < kThreads / 32) part[lane] = w;
  }
  __syncthreads();
  T excl_lane = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl_lane = ident;
  T prefix = op(wid > 0 ? part[wid - 1] : ident, excl_lane);
  for (int i = lo; i < hi; ++i) arr[i] = op(prefix, arr[i]);
  __syncthreads();
}

struct MinD { FFB_D double operator()(double a, double b) const { return b < a ? b : a; } };
struct MaxU { FFB_D uint32_t operator()(uint32_t a, uint32_t b) const { return b > a ? b : a; } };
struct AddU { FFB_D uint32_t operator()(uint32_t a, uint32_t b) const { return a + b; } };

FFB_D double block_reduce_min(double v, double* part) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { double o = __shfl_xor_sync(0xffffffffu, v, d); v = o < v ? o : v; }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) part[wid] = v;
  __syncthreads();
  double r = part[0];
  for (int w = 1; w < kThreads / 32; ++w) r = part[w] < r ? part[w] : r;
  return r;
}
FFB_D double block_reduce_max(double v, double* part) { return -block_reduce_min(-v, part); }

// IT: storage type of in-group indices (uint16_t when the group has at most 65535 points)
template <typename IT>
__global__ void __launch_bounds__(kThreads)
skyline_group_kernel(SkyArgs a) {
  constexpr uint32_t kPadI = (uint32_t)(IT)~(IT)0;
  FFB_DYN_SMEM(smem_raw);
  __shared__ double s_part[kThreads / 32 + 1];
  __shared__ unsigned long long s_bmin[kBuckets];
  __shared__ unsigned int s_count;
  __shared__ unsigned long long s_base;

  const int tid = threadIdx.x;
  const int64_t g = blockIdx.x;
  const int64_t p0 = g * a.group_size;
  int64_t rem = a.n_total - p0;
  const int G = (int)(rem < a.group_size ? rem : a.group_size);
  const int MC = a.surv_cap;

  // shared-memory carve-up: [resident e,t] [pm MC] [idx sort_cap] [gs MC]
  double* s_e = reinterpret_cast<double*>(smem_raw);
  double* s_t = s_e + (a.resident ? a.group_size : 0);
  double* s_pm = s_t + (a.resident ? a.group_size : 0);
  uint32_t* s_gs = reinterpret_cast<uint32_t*>(s_pm + MC);
  IT* s_idx = reinterpret_cast<IT*>(reinterpret_cast<unsigned char*>(s_pm) + a.surv_bytes);
  uint16_t* s_tie = reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(s_idx) + (size_t)a.sort_cap * 4);   // slots are 4 B wide
  // sort keys (ordered bits of e) live where s_pm / s_gs are built after the sort
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(s_pm);
  __shared__ int s_redo;

  const double* ge = a.e + p0;
  const double* gt = a.t + p0;
  const double* pe = a.resident ? s_e : ge;
  const double* pt = a.resident ? s_t : gt;

  // ---- 1. load + min t ----
  double tmin = INFINITY;
  for (int i = tid; i < G; i += kThreads) {
    const double tv = gt[i];
    if (a.resident) { s_e[i] = ge[i]; s_t[i] = tv; }
    if (a.tie_smem) s_tie[i] = (uint16_t)a.tie[i];          // general sort only
    tmin = tv < tmin ? tv : tmin;
  }
  const double t_peak = block_reduce_min(tmin, s_part);
  if (tid == 0) { s_count = 0; if (a.tpeak) a.tpeak[g] = t_peak; }
  const double thr = (a.rho > 0.0) ? t_peak / a.rho : INFINITY;       // explorer.py:210
  // ---- 2. e range over eligible points ----
  double emin = INFINITY, emax = -INFINITY;
  for (int i = tid; i < G; i += kThreads) {
    const double ev = pe[i], tv = pt[i];
    const bool ok = tv <= thr && ev < INFINITY && tv < INFINITY;
    if (ok) { emin = ev < emin ? ev : emin; emax = ev > emax ? ev : emax; }
  }
  emin = block_reduce_min(emin, s_part);
  emax = block_reduce_max(emax, s_part);
  for (int b = tid; b < kBuckets; b += kThreads) s_bmin[b] = ~0ull;
  __syncthreads();
  const double span = emax - emin;
  const double scale = (span > 0.0 && span < INFINITY) ? (double)(kBuckets - 1) / span : 0.0;
  // ---- 3. bucket min-t ----
  for (int i = tid; i < G; i += kThreads) {
    const double ev = pe[i], tv = pt[i];
    const bool ok = tv <= thr && ev < INFINITY && tv < INFINITY;
    if (ok) {
      int b = (int)((ev - emin) * scale);
      b = b < 0 ? 0 : (b > kBuckets - 1 ? kBuckets - 1 : b);
      atomicMin(&s_bmin[b], (unsigned long long)ordered_bits(tv));
    }
  }
  __syncthreads();
  // exclusive prefix-min over buckets (threads beyond kBuckets carry the identity)
  {
    unsigned long long v = tid < kBuckets ? s_bmin[tid] : ~0ull;
    unsigned long long incl = v;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      unsigned long long o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl = o < incl ? o : incl;
    }
    unsigned long long* wpart = reinterpret_cast<unsigned long long*>(s_part);
    __syncthreads();
    if (lane == 31) wpart[wid] = incl;
    __syncthreads();
    unsigned long long before = ~0ull;
    for (int w = 0; w < wid; ++w) before = wpart[w] < before ? wpart[w] : before;
    unsigned long long excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = ~0ull;
    excl = before < excl ? before : excl;
    __syncthreads();
    if (tid < kBuckets) s_bmin[tid] = excl;
  }
  __syncthreads();
  auto tie_of = [&](uint32_t i) -> uint64_t {
    if (a.tie_smem) return s_tie[i];
    if (a.tie) return a.tie[i];
    if (a.id) return a.id[p0 + i];
    return (uint64_t)i;
  };
  // packed sort slots: 64-bit key (ordered bits of e) + 32-bit (tie << 16 | index); needs 16-bit indices and ties
  const bool packed = sizeof(IT) == 2 && a.id == nullptr;
  uint32_t* s_lo = reinterpret_cast<uint32_t*>(s_idx);
  if (tid == 0) s_redo = 0;
  __syncthreads();
  // ---- 4. cull, collect survivors ----
  for (int i0 = 0; i0 < G; i0 += kThreads) {
    const int i = i0 + tid;
    bool keep = false;
    if (i < G) {
      const double ev = pe[i], tv = pt[i];
      const bool ok = tv <= thr && ev < INFINITY && tv < INFINITY;
      if (ok) {
        int b = (int)((ev - emin) * scale);
        b = b < 0 ? 0 : (b > kBuckets - 1 ? kBuckets - 1 : b);
        keep = a.occ != nullptr || !(s_bmin[b] < (unsigned long long)ordered_bits(tv));   // the min-t cull ignores occ
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int lane = tid & 31;
    unsigned base = 0;
    if (lane == 0 && m) base = atomicAdd(&s_count, (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
      const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
      if (pos < (unsigned)MC) {
        if (packed) {
          const uint64_t tv = tie_of((uint32_t)i);
          if (tv > 0xffffull) s_redo = 1;                          // tie rank does not fit: general sort
          s_lo[pos] = ((uint32_t)tv << 16) | (uint32_t)i;
          s_key[pos] = (unsigned long long)ordered_bits(pe[i] + 0.0);     // -0.0 == 0.0
        } else s_idx[pos] = (IT)i;
      }
    }
  }
  __syncthreads();
  const unsigned m_surv = s_count;
  if (m_surv > (unsigned)MC) {
    if (tid == 0) {
      if (a.front_n) a.front_n[g] = kPad;
      if (a.status) atomicOr(a.status, 1u << FFB_E_CAPACITY);
    }
    return;
  }
  int m2 = 1;
  while (m2 < (int)m_surv) m2 <<= 1;
  for (int i = m_surv + tid; i < m2; i += kThreads) {
    if (packed) { s_lo[i] = 0xffffffffu; s_key[i] = ~0ull; } else s_idx[i] = (IT)kPadI;
  }
  __syncthreads();

  // ---- 5. bitonic sort of survivors by (e, t, tie) ----
  auto less = [&](uint32_t x, uint32_t y) -> bool {
    if (x == kPadI) return false;
    if (y == kPadI) return true;
    const double ex = pe[x], ey = pe[y];
    if (ex != ey) return ex < ey;
    const double tx = pt[x], ty = pt[y];
    if (tx != ty) return tx < ty;
    return tie_of(x) < tie_of(y);
  };
  // Stages with partner distance >= 64 synchronise the CTA; the remaining ones (32..1) of a
  // level stay inside 64-element chunks, one warp per chunk, with warp-level barriers only.
  auto network = [&](auto cex) {
    const int lane = tid & 31, wid = tid >> 5;
    for (int k = 2; k <= m2; k <<= 1) {
      int j = k >> 1;
      for (; j >= 64; j >>= 1) {
        for (int p = tid; p < (m2 >> 1); p += kThreads) {      // one compare-exchange per pair
          const int i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
          cex(i, i | j, (i & k) == 0);
        }
        __syncthreads();
      }
      for (int c0 = wid * 64; c0 < m2; c0 += (kThreads / 32) * 64) {
        for (int j2 = j; j2 > 0; j2 >>= 1) {
          const int i = c0 + (((lane & ~(j2 - 1)) << 1) | (lane & (j2 - 1)));
          if ((i | j2) < m2) cex(i, i | j2, (i & k) == 0);
          __syncwarp();
        }
      }
      __syncthreads();
    }
  };
  auto cex_general = [&](int i, int ixj, bool asc) {
    const uint32_t x = s_idx[i], y = s_idx[ixj];
    if (less(y, x) == asc) { s_idx[i] = (IT)y; s_idx[ixj] = (IT)x; }
  };
  if (packed) {
    // Fast order: (ordered bits of e, tie, index) compared from the slots themselves, no look-ups.  In
    // the model's grids a tie in e is a tie in t as well (e is a function of t and the cap), so this IS
    // the (e, t, tie) order; the check below verifies that t never decreases inside a run of equal e
    // and the sort is redone with the full comparator if it does.
    auto cex_packed = [&](int i, int ixj, bool asc) {
      const unsigned long long kx = s_key[i], ky = s_key[ixj];
      const uint32_t lx = s_lo[i], ly = s_lo[ixj];
      const bool y_less = ky < kx || (ky == kx && ly < lx);
      if (y_less == asc && (ky != kx || ly != lx)) { s_key[i] = ky; s_key[ixj] = kx; s_lo[i] = ly; s_lo[ixj] = lx; }
    };
    if (!s_redo) network(cex_packed);
    // slots -> 16-bit indices, in place (every thread reads its slots before anyone writes)
    // (block by block: the 16-bit index of slot p lands inside slot p/2, which an earlier block owned)
    for (int base = 0; base < m2; base += kThreads) {
      const int p = base + tid;
      const uint32_t v = p < m2 ? s_lo[p] : 0u;
      __syncthreads();
      if (p < m2) s_idx[p] = (IT)(v & 0xffffu);
      __syncthreads();
    }
    bool bad = false;                                   // equal e, decreasing t: the (e, tie) order is not (e, t, tie)
    for (int p = 1 + tid; p < (int)m_surv; p += kThreads) {
      const uint32_t i = s_idx[p], q = s_idx[p - 1];
      if (pe[i] == pe[q] && pt[q] > pt[i]) bad = true;
    }
    if (bad) s_redo = 1;
    __syncthreads();
    if (s_redo) network(cex_general);
  } else {
    network(cex_general);
  }
  // ---- 6. exact filter: keep iff t <= min t over strictly lower e ----
  const int m = (int)m_surv;
  for (int p = tid; p < m; p += kThreads) {
    const uint32_t i = s_idx[p];
    s_pm[p] = pt[i];
    s_gs[p] = (p == 0 || pe[i] != pe[s_idx[p - 1]]) ? (uint32_t)p : 0u;
  }
  __syncthreads();
  if (a.occ == nullptr) block_scan_incl(s_pm, m, s_part, MinD(), (double)INFINITY);
  block_scan_incl(s_gs, m, reinterpret_cast<uint32_t*>(s_part), MaxU(), 0u);
  if (a.occ != nullptr) {
    // ---- 6b. three objectives (extension, no reference semantics) ----
    // drop i iff some j has e_j < e_i, t_j < t_i and occ_j >= occ_i.  Occupancy takes few distinct values
    // (resident warps / max warps), so the test is one prefix-min of t per occupancy level L over the points
    // with occ >= L, read at the end of the strictly-lower-e prefix.  More than 64 levels: FFB_E_CAPACITY.
    __shared__ unsigned long long s_lev[64];
    __shared__ int s_nlev, s_over;
    uint8_t* s_rank = reinterpret_cast<uint8_t*>(s_idx) + (size_t)a.sort_cap * 2;      // free half of the 4-byte sort slots
    uint8_t* s_keep = s_rank + a.sort_cap;
    if (tid < 64) s_lev[tid] = ~0ull;
    if (tid == 0) { s_nlev = 0; s_over = 0; }
    __syncthreads();
    const double* gocc = a.occ + p0;
    for (int p = tid; p < m; p += kThreads) {
      const unsigned long long ob = (unsigned long long)ordered_bits(gocc[s_idx[p]] + 0.0);
      uint32_t sl = (uint32_t)((ob * 0x9E3779B97F4A7C15ull) >> 58);
      int tries = 0;
      for (; tries < 64; ++tries) {
        const unsigned long long prev = atomicCAS(&s_lev[sl], ~0ull, ob);
        if (prev == ~0ull || prev == ob) break;
        sl = (sl + 1) & 63u;
      }
      if (tries == 64) s_over = 1;
      s_keep[p] = 1;
    }
    __syncthreads();
    if (s_over) {
      if (tid == 0) { if (a.front_n) a.front_n[g] = kPad; if (a.status) atomicOr(a.status, 1u << FFB_E_CAPACITY); }
      return;
    }
    if (tid < 32) {                                     // sort the (<= 64) levels ascending, empties last
      unsigned long long x = s_lev[tid], y = s_lev[tid + 32];
      for (int k = 2; k <= 64; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
          if (j == 32) { if (y < x) { const unsigned long long z = x; x = y; y = z; } }      // asc over the whole 64 (k == 64 only)
          else {
            const unsigned long long ox = __shfl_xor_sync(0xffffffffu, x, j), oy = __shfl_xor_sync(0xffffffffu, y, j);
            const bool lower = (tid & j) == 0;
            const bool ascx = (tid & k) == 0, ascy = ((tid + 32) & k) == 0;
            x = (lower == ascx) ? (ox < x ? ox : x) : (ox > x ? ox : x);
            y = (lower == ascy) ? (oy < y ? oy : y) : (oy > y ? oy : y);
          }
        }
      s_lev[tid] = x; s_lev[tid + 32] = y;
      const unsigned nx = __ballot_sync(0xffffffffu, x != ~0ull), ny = __ballot_sync(0xffffffffu, y != ~0ull);
      if (tid == 0) s_nlev = __popc(nx) + __popc(ny);
    }
    __syncthreads();
    const int n_lev = s_nlev;
    for (int p = tid; p < m; p += kThreads) {
      const unsigned long long ob = (unsigned long long)ordered_bits(gocc[s_idx[p]] + 0.0);
      int r = 0;
      while (s_lev[r] != ob) ++r;
      s_rank[p] = (uint8_t)r;
    }
    __syncthreads();
    for (int v = 0; v < n_lev; ++v) {
      for (int p = tid; p < m; p += kThreads) s_pm[p] = s_rank[p] >= v ? pt[s_idx[p]] : (double)INFINITY;
      __syncthreads();
      block_scan_incl(s_pm, m, s_part, MinD(), (double)INFINITY);
      for (int p = tid; p < m; p += kThreads) {
        if (s_rank[p] != v) continue;
        const uint32_t gs = s_gs[p];
        if (gs != 0u && s_pm[gs - 1] < pt[s_idx[p]]) s_keep[p] = 0;
      }
      __syncthreads();
    }
    for (int p = tid; p < m; p += kThreads) s_gs[p] = s_keep[p];
    __syncthreads();
  } else {
  // keep flags -> positions (reuse s_gs after reading the group start)
  for (int p0i = 0; p0i < m; p0i += kThreads) {
    const int p = p0i + tid;
    uint32_t keep = 0;
    if (p < m) {
      const uint32_t gs = s_gs[p];
      keep = (gs == 0u) ? 1u : (pt[s_idx[p]] <= s_pm[gs - 1] ? 1u : 0u);
    }
    __syncthreads();
    if (p < m) s_gs[p] = keep;
  }
  __syncthreads();
  }
  // s_pm no longer needed past this point for p beyond gs lookups: all reads done above
  block_scan_incl(s_gs, m, reinterpret_cast<uint32_t*>(s_part), AddU(), 0u);
  const uint32_t f = m > 0 ? s_gs[m - 1] : 0u;
  if (tid == 0) {
    if (a.front_n) a.front_n[g] = f;
    if (a.front_idx && !a.front_off && (int64_t)f > a.cap_front && a.status) atomicOr(a.status, 1u << FFB_E_CAPACITY);
    if (a.out_count) s_base = atomicAdd(a.out_count, (unsigned long long)f);
    if (a.front_off) {
      s_base = atomicAdd(a.front_total, (unsigned long long)f);
      a.front_off[g] = (int64_t)s_base;
      if (s_base + f > (unsigned long long)a.cap_front && a.status) atomicOr(a.status, 1u << FFB_E_CAPACITY);
    }
  }
  __syncthreads();
  const unsigned long long obase = (a.out_count || a.front_off) ? s_base : 0ull;
  if (a.out_count && obase + f > (unsigned long long)a.out_cap) {
    if (tid == 0 && a.status) atomicOr(a.status, 1u << FFB_E_CAPACITY);
  }
  for (int p = tid; p < m; p += kThreads) {
    const uint32_t incl = s_gs[p];
    const uint32_t prev = p > 0 ? s_gs[p - 1] : 0u;
    if (incl != prev) {
      const uint32_t rank = prev;
      const uint32_t i = s_idx[p];
      if (a.front_off) { if (obase + rank < (unsigned long long)a.cap_front) a.front_idx[obase + rank] = i; }
      else if (a.front_idx && (int64_t)rank < a.cap_front) a.front_idx[g * a.cap_front + rank] = i;
      if (a.out_count && obase + rank < (unsigned long long)a.out_cap) {
        a.out_e[obase + rank] = pe[i];
        a.out_t[obase + rank] = pt[i];
        a.out_id[obase + rank] = a.id ? a.id[p0 + i] : (uint64_t)(p0 + i);
        if (a.out_occ) a.out_occ[obase + rank] = a.occ[p0 + i];
      }
    }
  }
}

struct Plan { int resident; int surv_cap; int sort_cap; int surv_bytes; int tie_smem; size_t smem; };

// Survivor capacity = group size whenever shared memory allows, so a front made of ties
// (every candidate on it) is still exact; two CTAs per SM stay resident for the 3248-point
// groups of the headline workload (52 KB of points + 55 KB of survivor arrays).
Plan plan_groups(const FfbContext* ctx, int64_t group_size, bool has_tie, bool has_id) {
  Plan p;
  const size_t limit = ctx->smem_optin ? ctx->smem_optin - 4096 : 96 * 1024;
  const int64_t idx_bytes = group_size <= 65535 ? 2 : 4;
  auto need = [idx_bytes](int64_t mc, bool resident, int64_t g) {
    int64_t sc = 64; while (sc < mc) sc <<= 1;
    const int64_t region = ((mc * 12 > sc * 8 ? mc * 12 : sc * 8) + 15) / 16 * 16;
    return (size_t)(region + sc * 4 + (resident ? g * 16 : 0) + 64);      // 4 B per sort slot: u32 (tie << 16 | index) or IT
  };
  int64_t mc = group_size < 32 ? 32 : group_size;
  p.resident = need(mc, true, group_size) <= limit ? 1 : 0;
  if (!p.resident) { while (mc > 1024 && need(mc, false, group_size) > limit) mc = mc / 2; }
  int64_t sc = 64; while (sc < mc) sc <<= 1;
  p.surv_cap = (int)mc; p.sort_cap = (int)sc;
  p.surv_bytes = (int)(((mc * 12 > sc * 8 ? mc * 12 : sc * 8) + 15) / 16 * 16);
  p.smem = need(mc, p.resident != 0, group_size);
  p.tie_smem = 0;
  // the packed sort reads every survivor's tie exactly once (into its slot): staging the ties would only cost occupancy
  const bool packed = group_size <= 65535 && !has_id;
  if (has_tie && !packed && p.resident && group_size <= 65535 && p.smem + (size_t)group_size * 2 + 16 <= limit) {
    p.tie_smem = 1;
    p.smem += (size_t)group_size * 2 + 16;
  }
  return p;
}

// ---- streaming pre-filter of one huge candidate set (two objectives) --------------------------------
// Two coalesced passes over (e, t) (the first one over a 1/16 sample when the set is large) take the set from n to
// roughly n / kPreBuckets + the neighbourhood of the front before any sorting starts: pass 1 leaves min t per e-bucket (any monotone bucketing of e is valid, the
// range comes from a sample and out-of-range values clamp to the edge buckets), an exclusive prefix-min over
// the buckets follows, pass 2 keeps a candidate unless a STRICTLY lower bucket holds a strictly smaller t -
// i.e. unless it is provably dominated (explorer.py:122-140: drop iff some j has e_j < e_i and t_j < t_i).
// NaNs neither dominate nor get dropped.  Survivors are compacted with their ids.
constexpr int kPreBuckets = 4096;                             // table entries: e-buckets x occupancy levels
constexpr int kPreThreads = 512;
constexpr int kPreRun = 4096;                                 // candidates per sampled run of pass 1
constexpr int kPreLevels = 64;                                // distinct occupancy values the three-objective filter handles
// Three objectives (drop i iff some j has e_j < e_i, t_j < t_i and occ_j >= occ_i): the table gets one column per
// DISTINCT occupancy value (pass 0 collects them, at most kPreLevels; more: no pre-filter), min t per (e-bucket,
// level); after the exclusive prefix-min over the buckets a suffix-min over the levels makes entry (b, l) the
// smallest t among strictly lower e-buckets and occupancy >= level l.
struct PreArgs {
  const double* e; const double* t; const double* occ; const uint64_t* id;
  int64_t n;
  int64_t sample;                   // pass 1 reads every sample-th run of kPreRun candidates (1: all)
  double* range;                    // {lo, scale}
  unsigned long long* gmin;         // [kPreBuckets] min t per (bucket, level), later the prefix / suffix minima
  unsigned long long* lv_set;       // [2 * kPreLevels] hash set of ordered occupancy bits + 1 (pass 0)
  double* lv;                       // [kPreLevels] the distinct occupancy values, ascending
  int* n_lv;                        // their number (0: more than kPreLevels)
  int levels, lshift;               // columns of the table (power of two >= *n_lv, fixed by the host after pass 0); log2
  double* out_e; double* out_t; double* out_occ; uint64_t* out_id;
  int64_t out_cap;
  unsigned long long* out_count;
  uint32_t* overflow;
};
FFB_D int pre_bucket(double ev, double lo, double scale, int n_buckets) {
  const double x = (ev - lo) * scale;
  if (!(x > 0.0)) return 0;                                   // below the sampled range, or NaN
  return x >= (double)(n_buckets - 1) ? n_buckets - 1 : (int)x;
}
FFB_D int pre_level(double ov, const double* s_lv, int n_lv) {           // rank of ov among the distinct values (exact match exists)
  int lo = 0, hi = n_lv - 1;
  while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_lv[mid] < ov) lo = mid + 1; else hi = mid; }
  return lo;
}
__global__ void __launch_bounds__(kPreThreads) pre_levels_kernel(PreArgs a) {
  // pass 0 (three objectives): the distinct occupancy values, through a per-CTA set first
  __shared__ unsigned long long s_set[2 * kPreLevels];
  __shared__ int s_over;
  for (int i = threadIdx.x; i < 2 * kPreLevels; i += kPreThreads) s_set[i] = 0ull;
  if (threadIdx.x == 0) s_over = 0;
  __syncthreads();
  unsigned long long last = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * kPreThreads + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * kPreThreads) {
    const double ov = a.occ[i] + 0.0;
    const unsigned long long key = (unsigned long long)ordered_bits(ov) + 1ull;
    if (key == last || ov != ov) continue;
    last = key;
    uint32_t s = (uint32_t)((key * 0x9e3779b97f4a7c15ull) >> 57);
    for (int pr = 0; pr < 2 * kPreLevels; ++pr) {
      const unsigned long long prev = atomicCAS(&s_set[s], 0ull, key);
      if (prev == 0ull || prev == key) break;
      s = (s + 1) & (2 * kPreLevels - 1);
      if (pr == 2 * kPreLevels - 1) s_over = 1;
    }
  }
  __syncthreads();
  if (s_over) { *a.overflow = 1u; return; }
  for (int i = threadIdx.x; i < 2 * kPreLevels; i += kPreThreads) {
    const unsigned long long key = s_set[i];
    if (!key) continue;
    uint32_t s = (uint32_t)((key * 0x9e3779b97f4a7c15ull) >> 57);
    for (int pr = 0; pr < 2 * kPreLevels; ++pr) {
      const unsigned long long prev = atomicCAS(&a.lv_set[s], 0ull, key);
      if (prev == 0ull || prev == key) break;
      s = (s + 1) & (2 * kPreLevels - 1);
      if (pr == 2 * kPreLevels - 1) *a.overflow = 1u;
    }
  }
}
__global__ void pre_levels_sort_kernel(PreArgs a) {            // one warp: <= 128 slots -> ascending distinct values
  if (threadIdx.x != 0) return;
  int n = 0;
  double v[2 * kPreLevels];
  for (int i = 0; i < 2 * kPreLevels; ++i) {
    const unsigned long long key = a.lv_set[i];
    if (!key) continue;
    const unsigned long long ob = key - 1ull;
    const unsigned long long bits = (ob & 0x8000000000000000ull) ? (ob & 0x7fffffffffffffffull) : ~ob;
    v[n++] = __longlong_as_double((long long)bits);
  }
  if (n > kPreLevels || *a.overflow) { *a.n_lv = 0; return; }
  for (int i = 1; i < n; ++i) { const double x = v[i]; int j = i - 1; while (j >= 0 && v[j] > x) { v[j + 1] = v[j]; --j; } v[j + 1] = x; }
  for (int i = 0; i < n; ++i) a.lv[i] = v[i];
  *a.n_lv = n;
}
__global__ void __launch_bounds__(1024) pre_range_kernel(PreArgs a) {
  __shared__ double s_lo[32], s_hi[32];
  const int n_buckets = kPreBuckets >> a.lshift;
  const int64_t m = a.n < 65536 ? a.n : 65536;
  const int64_t stride = a.n / m;                             // sample spread over the whole set
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = a.e[i * stride];
    if (v > -INFINITY && v < INFINITY) { lo = v < lo ? v : lo; hi = v > hi ? v : hi; }
  }
  for (int d = 16; d > 0; d >>= 1) {
    const double ol = __shfl_xor_sync(0xffffffffu, lo, d), oh = __shfl_xor_sync(0xffffffffu, hi, d);
    lo = ol < lo ? ol : lo; hi = oh > hi ? oh : hi;
  }
  if ((threadIdx.x & 31) == 0) { s_lo[threadIdx.x >> 5] = lo; s_hi[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = s_lo[w] < lo ? s_lo[w] : lo; hi = s_hi[w] > hi ? s_hi[w] : hi; }
    const double span = hi - lo;
    a.range[0] = lo < INFINITY ? lo : 0.0;
    a.range[1] = (span > 0.0 && span < INFINITY) ? (double)n_buckets / span : 0.0;
  }
  for (int b = threadIdx.x; b < kPreBuckets; b += blockDim.x) a.gmin[b] = ~0ull;
}
__global__ void __launch_bounds__(kPreThreads) pre_min_kernel(PreArgs a) {
  __shared__ unsigned long long s_min[kPreBuckets];
  __shared__ double s_lv[kPreLevels];
  const int n_buckets = kPreBuckets >> a.lshift, n_lv = a.occ ? *a.n_lv : 1;
  for (int b = threadIdx.x; b < kPreBuckets; b += kPreThreads) s_min[b] = ~0ull;
  if (a.occ && threadIdx.x < n_lv) s_lv[threadIdx.x] = a.lv[threadIdx.x];
  __syncthreads();
  const double lo = a.range[0], scale = a.range[1];
  // every `sample`-th run of kPreRun candidates: a minimum over a SUBSET is still a valid certificate (the pass-2
  // test names an existing dominator), so large sets pay one full pass instead of two
  const int64_t n_s = a.sample > 1 ? (a.n / ((int64_t)kPreRun * a.sample)) * kPreRun : a.n;
  for (int64_t j = (int64_t)blockIdx.x * kPreThreads + threadIdx.x; j < n_s; j += (int64_t)gridDim.x * kPreThreads) {
    const int64_t i = a.sample > 1 ? (j / kPreRun) * ((int64_t)kPreRun * a.sample) + (j % kPreRun) : j;
    const double ev = a.e[i], tv = a.t[i];
    if (ev != ev || tv != tv) continue;
    int slot = pre_bucket(ev, lo, scale, n_buckets);
    if (a.occ) {
      const double ov = a.occ[i] + 0.0;
      if (ov != ov) continue;
      slot = (slot << a.lshift) | pre_level(ov, s_lv, n_lv);
    }
    const unsigned long long tb = (unsigned long long)ordered_bits(tv);
    if (tb < s_min[slot]) atomicMin(&s_min[slot], tb);        // the plain read only spares atomics that cannot win
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kPreBuckets; b += kPreThreads)
    if (s_min[b] != ~0ull) atomicMin(&a.gmin[b], s_min[b]);
}
__global__ void __launch_bounds__(1024) pre_prefix_kernel(PreArgs a) {
  __shared__ unsigned long long s_tab[kPreBuckets];
  __shared__ unsigned long long s_w[32];
  const int tid = threadIdx.x;
  if (a.lshift == 0) {
    // two objectives: exclusive prefix-min over kPreBuckets values, 4 per thread, warp scan, scan of the warp totals
    unsigned long long v[4], run = ~0ull;
    for (int k = 0; k < 4; ++k) { v[k] = a.gmin[4 * tid + k]; }
    unsigned long long tot = v[0] < v[1] ? v[0] : v[1];
    tot = v[2] < tot ? v[2] : tot; tot = v[3] < tot ? v[3] : tot;
    unsigned long long incl = tot;
    for (int d = 1; d < 32; d <<= 1) { const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, d); if ((tid & 31) >= d && o < incl) incl = o; }
    if ((tid & 31) == 31) s_w[tid >> 5] = incl;
    __syncthreads();
    if (tid < 32) {
      unsigned long long w = s_w[tid], wi = w;
      for (int d = 1; d < 32; d <<= 1) { const unsigned long long o = __shfl_up_sync(0xffffffffu, wi, d); if (tid >= d && o < wi) wi = o; }
      const unsigned long long ex = __shfl_up_sync(0xffffffffu, wi, 1);
      s_w[tid] = tid == 0 ? ~0ull : ex;
    }
    __syncthreads();
    unsigned long long before = __shfl_up_sync(0xffffffffu, incl, 1);
    if ((tid & 31) == 0) before = ~0ull;
    run = before < s_w[tid >> 5] ? before : s_w[tid >> 5];
    for (int k = 0; k < 4; ++k) { a.gmin[4 * tid + k] = run; run = v[k] < run ? v[k] : run; }
    return;
  }
  // three objectives, in shared memory: per level an exclusive prefix-min over the e-buckets (thread l walks column
  // l), then per bucket a suffix-min over the levels (occupancy >= level)
  const int levels = 1 << a.lshift, n_buckets = kPreBuckets >> a.lshift;
  for (int i = tid; i < kPreBuckets; i += blockDim.x) s_tab[i] = a.gmin[i];
  __syncthreads();
  if (tid < levels) {
    unsigned long long run = ~0ull;
    for (int b = 0; b < n_buckets; ++b) {
      const int at = (b << a.lshift) | tid;
      const unsigned long long v = s_tab[at];
      s_tab[at] = run;
      run = v < run ? v : run;
    }
  }
  __syncthreads();
  for (int b = tid; b < n_buckets; b += blockDim.x) {
    unsigned long long run = ~0ull;
    for (int l = levels - 1; l >= 0; --l) {
      const int at = (b << a.lshift) | l;
      const unsigned long long v = s_tab[at];
      run = v < run ? v : run;
      s_tab[at] = run;
    }
  }
  __syncthreads();
  for (int i = tid; i < kPreBuckets; i += blockDim.x) a.gmin[i] = s_tab[i];
}
__global__ void __launch_bounds__(kPreThreads) pre_filter_kernel(PreArgs a) {
  __shared__ unsigned long long s_pm[kPreBuckets];
  __shared__ double s_lv[kPreLevels];
  const int n_buckets = kPreBuckets >> a.lshift, n_lv = a.occ ? *a.n_lv : 1;
  for (int b = threadIdx.x; b < kPreBuckets; b += kPreThreads) s_pm[b] = a.gmin[b];
  if (a.occ && threadIdx.x < n_lv) s_lv[threadIdx.x] = a.lv[threadIdx.x];
  __syncthreads();
  const double lo = a.range[0], scale = a.range[1];
  const int lane = threadIdx.x & 31;
  const int64_t step = (int64_t)gridDim.x * kPreThreads;
  const int64_t n_round = (a.n + step - 1) / step * step;     // whole warps take part in every ballot
  for (int64_t i = (int64_t)blockIdx.x * kPreThreads + threadIdx.x; i < n_round; i += step) {
    bool keep = false;
    double ev = 0.0, tv = 0.0, ov = 0.0;
    if (i < a.n) {
      ev = a.e[i]; tv = a.t[i];
      if (a.occ) ov = a.occ[i];
      keep = ev != ev || tv != tv || ov != ov;
      if (!keep) {
        int slot = pre_bucket(ev, lo, scale, n_buckets);
        if (a.occ) slot = (slot << a.lshift) | pre_level(ov + 0.0, s_lv, n_lv);
        keep = !(s_pm[slot] < (unsigned long long)ordered_bits(tv));
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(a.out_count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
      const int64_t at = (int64_t)base + __popc(m & ((1u << lane) - 1u));
      if (at < a.out_cap) {
        a.out_e[at] = ev; a.out_t[at] = tv; a.out_id[at] = a.id ? a.id[i] : (uint64_t)i;
        if (a.occ) a.out_occ[at] = ov;
      }
      else *a.overflow = 1u;
    }
  }
}

int32_t launch_groups(FfbContext* ctx, SkyArgs a, int64_t n_groups, cudaStream_t stream) {
  Plan p = plan_groups(ctx, a.group_size, a.tie != nullptr, a.id != nullptr);
  a.resident = p.resident;
  a.surv_cap = p.surv_cap;
  a.sort_cap = p.sort_cap;
  a.surv_bytes = p.surv_bytes;
  a.tie_smem = p.tie_smem;
  if (n_groups > 0x7fffffffLL) return ffb_fail(ctx, FFB_E_CAPACITY, "skyline: too many groups for one launch");
  if (a.group_size <= 65535) {
    FFB_CUDA(ctx, cudaFuncSetAttribute(skyline_group_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    FFB_LAUNCH(skyline_group_kernel<uint16_t>, (unsigned)n_groups, kThreads, p.smem, stream, a);
  } else {
    FFB_CUDA(ctx, cudaFuncSetAttribute(skyline_group_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    FFB_LAUNCH(skyline_group_kernel<uint32_t>, (unsigned)n_groups, kThreads, p.smem, stream, a);
  }
  return ffb_check_launch(ctx, "skyline_group_kernel");
}

}  // namespace

extern "C" int32_t ffb_skyline_groups(FfbContext* ctx, const double* d_e, const double* d_t,
                                      int64_t n_groups, int64_t group_size, const uint32_t* d_tie,
                                      double rho, uint32_t* d_front_idx, uint32_t* d_front_n,
                                      double* d_tpeak, int64_t cap_front, int64_t* d_front_off,
                                      uint32_t* d_status, void* stream) {
  return ffb_skyline_groups3(ctx, d_e, d_t, nullptr, n_groups, group_size, d_tie, rho, d_front_idx, d_front_n, d_tpeak,
                             cap_front, d_front_off, d_status, stream);
}

extern "C" int32_t ffb_skyline_groups3(FfbContext* ctx, const double* d_e, const double* d_t, const double* d_occ,
                                       int64_t n_groups, int64_t group_size, const uint32_t* d_tie,
                                       double rho, uint32_t* d_front_idx, uint32_t* d_front_n,
                                       double* d_tpeak, int64_t cap_front, int64_t* d_front_off,
                                       uint32_t* d_status, void* stream) {
  if (!ctx || !d_e || !d_t || n_groups < 0 || group_size <= 0 || group_size > 0x7fffffffLL || cap_front < 0)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_skyline_groups: bad argument");
  if (d_occ && group_size > 65535)
    return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_skyline_groups3: three-objective groups hold at most 65535 candidates");
  if (!(rho <= 1.0)) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_skyline_groups: rho must be <= 1");
  if (n_groups == 0) return FFB_OK;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));
  SkyArgs a = {};
  a.e = d_e; a.t = d_t; a.occ = d_occ; a.id = nullptr; a.tie = d_tie;
  a.n_total = n_groups * group_size; a.group_size = group_size; a.rho = rho;
  a.front_idx = d_front_idx; a.front_n = d_front_n; a.tpeak = d_tpeak; a.cap_front = cap_front;
  a.status = d_status;
  if (d_front_off) {
    int32_t rc = ffb_reserve(ctx, &ctx->d_sky, 256);
    if (rc) return rc;
    a.front_off = d_front_off;
    a.front_total = (unsigned long long*)ctx->d_sky.p;
    FFB_CUDA(ctx, cudaMemsetAsync(a.front_total, 0, 8, (cudaStream_t)stream));
  }
  return launch_groups(ctx, a, n_groups, (cudaStream_t)stream);
}

extern "C" int32_t ffb_skyline(FfbContext* ctx, const double* d_e, const double* d_t, const double* d_occ,
                               const uint64_t* d_id, int64_t n, double rho, uint64_t* d_front_id,
                               double* d_front_e, double* d_front_t, int64_t cap_front,
                               int64_t* h_front_n, double* h_tpeak, void* stream_) {
  if (!ctx || !d_e || !d_t || n < 0 || !h_front_n || cap_front <= 0 || !d_front_id)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_skyline: bad argument");
  if (!(rho <= 1.0)) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_skyline: rho must be <= 1");
  cudaStream_t stream = (cudaStream_t)stream_;
  *h_front_n = 0;
  if (h_tpeak) *h_tpeak = INFINITY;
  if (n == 0) return FFB_OK;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));

  // Level structure: chunk fronts -> compact buffer -> ... -> one group.  The floor is
  // applied on the last level only: front(floor(X)) == floor(front(X)) because a dominator
  // has strictly smaller t and is therefore itself eligible.
  const int64_t chunk = 4096;
  int64_t work_cap = n / 8 + 4 * chunk;
  if (work_cap < cap_front) work_cap = cap_front;
  // scratch: two ping-pong triples + counters/status
  const size_t tri = (size_t)work_cap * (d_occ ? 32 : 24);
  int32_t rc = ffb_reserve(ctx, &ctx->d_sky, 2 * tri + 256 + (size_t)kPreBuckets * 8 + 64 + (size_t)3 * kPreLevels * 8 + 64);
  if (rc) return rc;
  char* base = (char*)ctx->d_sky.p;
  double* buf_e[2] = {(double*)base, (double*)(base + tri)};
  double* buf_t[2] = {buf_e[0] + work_cap, buf_e[1] + work_cap};
  uint64_t* buf_id[2] = {(uint64_t*)(buf_t[0] + work_cap), (uint64_t*)(buf_t[1] + work_cap)};
  double* buf_occ[2] = {(double*)(buf_id[0] + work_cap), (double*)(buf_id[1] + work_cap)};       // only with d_occ
  const double* cur_occ = d_occ;
  unsigned long long* d_count = (unsigned long long*)(base + 2 * tri);
  uint32_t* d_status = (uint32_t*)(d_count + 4);
  double* d_tp = (double*)(d_count + 8);

  const double* cur_e = d_e; const double* cur_t = d_t; const uint64_t* cur_id = d_id;
  int64_t cur_n = n;
  int which = 0;
  bool stalled = false;
  FFB_CUDA(ctx, cudaMemsetAsync(d_count, 0, 128, stream));
  int64_t pre_min = (int64_t)1 << 20;
  if (const char* ev = getenv("FFB_SKYLINE_PREFILTER_MIN")) pre_min = atoll(ev);      // test hook: small sets through the pre-filter
  if (n >= pre_min) {
    // large sets: the streaming pre-filter first (see above); when its survivors do not fit the work buffer (a set
    // that is mostly front), or a three-objective set has more than kPreLevels distinct occupancy values, the levels
    // below start from the whole set as before
    PreArgs pa = {};
    pa.e = d_e; pa.t = d_t; pa.occ = d_occ; pa.id = d_id; pa.n = n;
    pa.sample = n >= ((int64_t)1 << 26) ? 16 : 1;
    char* pbase = base + 2 * tri + 256;
    pa.gmin = (unsigned long long*)pbase; pa.range = (double*)(pbase + (size_t)kPreBuckets * 8);
    pa.lv_set = (unsigned long long*)(pbase + (size_t)kPreBuckets * 8 + 64);
    pa.lv = (double*)(pa.lv_set + 2 * kPreLevels);
    pa.n_lv = (int*)(pa.lv + kPreLevels);
    pa.out_e = buf_e[0]; pa.out_t = buf_t[0]; pa.out_id = buf_id[0]; pa.out_occ = d_occ ? buf_occ[0] : nullptr; pa.out_cap = work_cap;
    pa.out_count = d_count + 3; pa.overflow = d_status + 1;
    unsigned ctas = (unsigned)ctx->sm_count * 4;
    if ((int64_t)ctas * kPreThreads > n) ctas = (unsigned)((n + kPreThreads - 1) / kPreThreads);
    bool usable = true;
    if (d_occ) {
      FFB_CUDA(ctx, cudaMemsetAsync(pa.lv_set, 0, (size_t)2 * kPreLevels * 8 + (size_t)kPreLevels * 8 + 16, stream));
      FFB_LAUNCH(pre_levels_kernel, ctas, kPreThreads, 0, stream, pa);
      FFB_LAUNCH(pre_levels_sort_kernel, 1, 32, 0, stream, pa);
      int h_lv = 0;
      FFB_CUDA(ctx, cudaMemcpyAsync(&h_lv, pa.n_lv, sizeof(int), cudaMemcpyDeviceToHost, stream));
      FFB_CUDA(ctx, cudaStreamSynchronize(stream));
      usable = h_lv > 0;
      while ((1 << pa.lshift) < h_lv) ++pa.lshift;
      pa.levels = 1 << pa.lshift;
      FFB_CUDA(ctx, cudaMemsetAsync(d_count, 0, 128, stream));       // the overflow flag of pass 0 shares the status word
    }
    if (usable) {
      FFB_LAUNCH(pre_range_kernel, 1, 1024, 0, stream, pa);
      FFB_LAUNCH(pre_min_kernel, ctas, kPreThreads, 0, stream, pa);
      FFB_LAUNCH(pre_prefix_kernel, 1, 1024, 0, stream, pa);
      FFB_LAUNCH(pre_filter_kernel, ctas, kPreThreads, 0, stream, pa);
      rc = ffb_check_launch(ctx, "skyline pre-filter");
      if (rc) return rc;
      unsigned long long h_kept = 0; uint32_t h_over = 0;
      FFB_CUDA(ctx, cudaMemcpyAsync(&h_kept, pa.out_count, sizeof(h_kept), cudaMemcpyDeviceToHost, stream));
      FFB_CUDA(ctx, cudaMemcpyAsync(&h_over, pa.overflow, sizeof(h_over), cudaMemcpyDeviceToHost, stream));
      FFB_CUDA(ctx, cudaStreamSynchronize(stream));
      if (!h_over && (int64_t)h_kept <= work_cap) {
        cur_e = buf_e[0]; cur_t = buf_t[0]; cur_id = buf_id[0]; cur_n = (int64_t)h_kept; which = 1;
        if (d_occ) cur_occ = buf_occ[0];
      }
    }
    FFB_CUDA(ctx, cudaMemsetAsync(d_count, 0, 128, stream));
  }
  for (int level = 0; level < 64; ++level) {
    // normally the last level is one resident chunk; a set that stopped shrinking (its front is
    // larger than a chunk, e.g. heavy ties) is finished by one CTA streaming from L2 with the
    // largest survivor capacity shared memory allows
    const bool last = cur_n <= chunk || stalled;
    const int64_t n_groups = (cur_n + chunk - 1) / chunk;
    SkyArgs a = {};
    a.e = cur_e; a.t = cur_t; a.id = cur_id; a.tie = nullptr;
    a.occ = cur_occ;
    if (d_occ && (last ? cur_n : chunk) > 65535)
      return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_skyline: the three-objective front does not reduce to one 65535-point group (%lld left)", (long long)cur_n);
    a.n_total = cur_n; a.group_size = last ? cur_n : chunk;
    a.rho = last ? rho : 0.0;
    a.status = d_status;
    a.out_count = d_count + (level & 3);
    if (last) {
      a.out_e = d_front_e ? d_front_e : buf_e[which]; a.out_t = d_front_t ? d_front_t : buf_t[which];
      a.out_id = d_front_id; a.out_cap = d_front_e && d_front_t ? cap_front : (cap_front < work_cap ? cap_front : work_cap);
      a.tpeak = d_tp;
    } else {
      a.out_e = buf_e[which]; a.out_t = buf_t[which]; a.out_id = buf_id[which]; a.out_cap = work_cap;
      if (d_occ) a.out_occ = buf_occ[which];
    }
    FFB_CUDA(ctx, cudaMemsetAsync(a.out_count, 0, sizeof(unsigned long long), stream));
    rc = launch_groups(ctx, a, last ? 1 : n_groups, stream);
    if (rc) return rc;
    unsigned long long h_count = 0; uint32_t h_status = 0;
    FFB_CUDA(ctx, cudaMemcpyAsync(&h_count, a.out_count, sizeof(h_count), cudaMemcpyDeviceToHost, stream));
    FFB_CUDA(ctx, cudaMemcpyAsync(&h_status, d_status, sizeof(h_status), cudaMemcpyDeviceToHost, stream));
    FFB_CUDA(ctx, cudaStreamSynchronize(stream));
    if (h_status & (1u << FFB_E_CAPACITY)) {
      // the chunk fronts (or the final group's front) outgrew their buffer: a set that is mostly front.  Two
      // objectives finish with the device-wide sort over what this level STARTED from (ffb_bigfront.cu).
      if (!d_occ && cur_n < ((int64_t)1 << 32))
        return ffb_big_front(ctx, cur_e, cur_t, cur_id, cur_n, rho, d_front_id, d_front_e, d_front_t, cap_front, h_front_n, h_tpeak, stream);
      return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_skyline: front exceeds capacity at level %d (%llu candidates kept of %lld)",
                      level, h_count, (long long)cur_n);
    }
    if (last) {
      *h_front_n = (int64_t)h_count;
      if (h_tpeak) {
        // t_peak of the whole set = min t = min over the final group (the min-t point is
        // never dominated, so it reaches the last level)
        FFB_CUDA(ctx, cudaMemcpyAsync(h_tpeak, d_tp, sizeof(double), cudaMemcpyDeviceToHost, stream));
        FFB_CUDA(ctx, cudaStreamSynchronize(stream));
      }
      return FFB_OK;
    }
    if ((int64_t)h_count * 4 > cur_n * 3) {
      // the set stopped shrinking: its front is larger than a chunk (ties).  Small ones are finished by one CTA
      // streaming from L2; larger ones by the device-wide sort (two objectives)
      if ((int64_t)h_count > 8192) {
        if (d_occ || (int64_t)h_count >= ((int64_t)1 << 32))
          return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_skyline: candidate set does not reduce (%llu of %lld on chunk fronts)",
                          h_count, (long long)cur_n);
        return ffb_big_front(ctx, buf_e[which], buf_t[which], buf_id[which], (int64_t)h_count, rho, d_front_id, d_front_e, d_front_t,
                             cap_front, h_front_n, h_tpeak, stream);
      }
      stalled = true;
    }
    cur_e = buf_e[which]; cur_t = buf_t[which]; cur_id = buf_id[which];
    if (d_occ) cur_occ = buf_occ[which];
    cur_n = (int64_t)h_count;
    which ^= 1;
  }
  return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_skyline: level limit reached");
}
