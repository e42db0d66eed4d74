// K2 + K3 + K4 fused, fronts only: the whole of pareto_explore (explorer.py:186-212 =
// generate_valid_configs -> evaluate_configs -> throughput floor -> pareto_front) for every
// (kernel, spec) group in ONE kernel.  A caller that wants fronts never sees the [K,S,J,C] grid:
// the 16 B per point that ffb_predict_grid writes and ffb_skyline_groups reads back stay in
// shared memory (the two-kernel route moves 4 GB through HBM per 1.25e8 points for nothing).
//
// One CTA per group (kernel k, spec s), J shapes x C caps candidates:
//   1. one thread per shape evaluates the cap-independent chain (ffb_model.cuh, the SAME device
//      functions the grid kernel uses, -fmad=false) and walks the cap axis; e goes to shared
//      memory, t is one value per shape (the time model has no cap term, time_model.py:98-129);
//   2. t_peak = min t, floor t <= t_peak / rho (explorer.py:209-210);
//   3. exact ties are merged first: a hash table in shared memory (open addressing, atomicCAS) maps every
//      eligible candidate to the representative of its (e, t) class and counts the class.  Model grids are
//      full of exact ties - shapes that share (threads, min(bx, 32), |ln(bx/by)|) give the same t and the
//      same p_dyn, cap-limited candidates of one t share e = t * cap + e_overhead - and the reference keeps
//      them all (explorer.py:137: t <= best_t), which is why 47% of a 3248-point group sits on its front;
//   4. the UNIQUE keys are ordered by value-bucket counting sort: bucket = floor((e - emin) * scale) is
//      monotone in e, so a lower bucket means strictly lower e; counts -> exclusive scan -> scatter; a key's
//      rank is its bucket's start plus the number of bucket mates with a smaller (e, t).  The same mate loop
//      applies the reference's filter (explorer.py:132-139): a class is dropped iff some candidate has
//      strictly lower e AND strictly lower t, i.e. iff min(prefix-min of t over lower buckets, t of mates
//      with lower e) < t.  This replaces the 66-stage bitonic network of skyline_group_kernel (65% of that
//      kernel, ncu r1z) by linear passes;
//   5. kept classes are numbered in key order; the candidates, taken in (bx, by, cap) order (a host-built
//      permutation, explorer.py:113-119), are then STABLY radix-sorted by their class number (6 bits per
//      pass, 1-3 passes): every warp ranks a contiguous run of the sequence with __match_any_sync and
//      per-warp digit counters, one block scan over (digit, warp) turns the counters into offsets.  The
//      first pass drops everything that is not on the front, so it also compacts.  Stable + tie order in =
//      (e, t, bx, by, cap) order out, in linear time however large the tie classes are.
// Output: in-group indices j * C + c, dense or compact like ffb_skyline_groups, optionally with (e, t).
#include "ffb_model.cuh"

#include <string.h>
#include <algorithm>
#include <numeric>
#include <vector>

using namespace ffbm;

namespace {

constexpr int kXThreads = 512;
constexpr int kXWarps = kXThreads / 32;
constexpr int kDigits = 64;                    // radix of the final stable sort (6 bits per pass)
constexpr unsigned kXAll = 0xffffffffu;
constexpr int kMaxClassA = 96;                 // (threads, regs) classes kept on chip; shape tables with more fall back to eval_unit

struct ExploreArgs {
  const double* feat;
  const int64_t* res;
  Tables tb;
  int64_t n_groups;
  int n_specs, n_shapes, n_caps;
  uint32_t div_c;              // ceil(2^32 / C): i / C == (i * div_c) >> 32 for i < 2^16 * ... (checked on the host)
  const uint16_t* by_tie;      // [G] candidate indices in (block_x, block_y, block_z, regs, cap) order (explorer.py:113-119)
  double rho;
  int nb;                      // value buckets (power of two, multiple of kXThreads)
  int n_slots;                 // hash slots (power of two >= 2 G)
  uint32_t* front_idx;
  uint32_t* front_n;
  double* tpeak;
  int64_t cap_front;
  int64_t* front_off;
  unsigned long long* front_total;
  double* front_e;
  double* front_t;
  uint32_t* status;
};

// i / C for candidate indices (i < 2^15, C <= 4096): one multiply-high; div_c == 0 stands for C == 1
FFB_D int div_c_of(unsigned i, uint32_t div_c) { return div_c ? (int)__umulhi(i, div_c) : (int)i; }

FFB_D unsigned long long ord_bits(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

FFB_D double block_min_d(double v, double* part) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { const double o = __shfl_xor_sync(kXAll, v, d); v = o < v ? o : v; }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) part[wid] = v;
  __syncthreads();
  double r = part[0];
#pragma unroll
  for (int w = 1; w < kXThreads / 32; ++w) r = part[w] < r ? part[w] : r;
  return r;
}

// exclusive scan (sum of u32 / min of u64) over nb entries, each thread owning nb / kXThreads consecutive ones
FFB_D void scan_buckets(uint32_t* cnt, unsigned long long* bmin, int nb, uint32_t* part_c, unsigned long long* part_m) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = nb / kXThreads;              // nb is a multiple of kXThreads (host)
  const int lo = tid * per;
  uint32_t sum = 0;
  unsigned long long mn = ~0ull;
  for (int i = 0; i < per; ++i) { sum += cnt[lo + i]; const unsigned long long v = bmin[lo + i]; mn = v < mn ? v : mn; }
  uint32_t isum = sum;
  unsigned long long imn = mn;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t os = __shfl_up_sync(kXAll, isum, d);
    const unsigned long long om = __shfl_up_sync(kXAll, imn, d);
    if (lane >= d) { isum += os; imn = om < imn ? om : imn; }
  }
  if (lane == 31) { part_c[wid] = isum; part_m[wid] = imn; }
  __syncthreads();
  uint32_t base = 0;
  unsigned long long bm = ~0ull;
  for (int w = 0; w < wid; ++w) { base += part_c[w]; bm = part_m[w] < bm ? part_m[w] : bm; }
  uint32_t ex = __shfl_up_sync(kXAll, isum, 1);
  unsigned long long em = __shfl_up_sync(kXAll, imn, 1);
  if (lane == 0) { ex = 0; em = ~0ull; }
  uint32_t run = base + ex;
  unsigned long long rm = bm < em ? bm : em;
  for (int i = 0; i < per; ++i) {
    const uint32_t c = cnt[lo + i];
    const unsigned long long v = bmin[lo + i];
    cnt[lo + i] = run; bmin[lo + i] = rm;
    run += c; rm = v < rm ? v : rm;
  }
  __syncthreads();
}

// One stable pass of the class-number radix sort.  kFirst: the source is the tie-ordered permutation in
// global memory and candidates that are not on the front are dropped.  Returns the number of items written.
template <bool kFirst>
FFB_D int radix_pass(const uint16_t* src, uint16_t* dst, int n, int shift, const uint16_t* s_cls, const uint16_t* s_krank,
                     uint32_t* s_wcnt, uint16_t* s_lrank, uint32_t* s_pc) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int chunk = ((n + kXWarps * 32 - 1) / (kXWarps * 32)) * 32;      // contiguous run per warp, whole rounds
  const int wbeg = wid * chunk, wend = wbeg + chunk < n ? wbeg + chunk : n;
  for (int q = tid; q < kDigits * kXWarps; q += kXThreads) s_wcnt[q] = 0;
  __syncthreads();
  for (int r0 = wbeg; r0 < wend; r0 += 32) {
    const int idx = r0 + lane;
    uint32_t d = kDigits + (uint32_t)lane;                               // idle lanes: a digit of their own
    if (idx < wend) {
      const uint32_t item = src[idx];
      const uint32_t c16 = s_cls[item];
      const uint32_t kr = c16 == 0xffffu ? 0xffffu : s_krank[c16];
      if (!kFirst || kr != 0xffffu) d = (kr >> shift) & (kDigits - 1);
    }
    const unsigned peers = __match_any_sync(kXAll, d);
    uint32_t pre = 0;
    if (d < (uint32_t)kDigits) pre = s_wcnt[d * kXWarps + wid];
    __syncwarp();
    if (d < (uint32_t)kDigits) {
      if ((peers & lt_mask) == 0u) s_wcnt[d * kXWarps + wid] = pre + (uint32_t)__popc(peers);
      s_lrank[idx] = (uint16_t)(pre + (uint32_t)__popc(peers & lt_mask));
    } else if (idx < wend) s_lrank[idx] = 0xffffu;
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan over (digit, warp): kDigits * kXWarps = 2 entries per thread
  constexpr int kPer = kDigits * kXWarps / kXThreads;
  uint32_t v[kPer], sum = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) { v[q] = s_wcnt[tid * kPer + q]; sum += v[q]; }
  uint32_t incl = sum;
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) { const uint32_t o = __shfl_up_sync(kXAll, incl, dd); if (lane >= dd) incl += o; }
  if (lane == 31) s_pc[wid] = incl;
  __syncthreads();
  uint32_t before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kXWarps; ++w) { if (w < wid) before += s_pc[w]; total += s_pc[w]; }
  uint32_t run = before + incl - sum;
#pragma unroll
  for (int q = 0; q < kPer; ++q) { s_wcnt[tid * kPer + q] = run; run += v[q]; }
  __syncthreads();
  for (int r0 = wbeg; r0 < wend; r0 += 32) {
    const int idx = r0 + lane;
    if (idx < wend) {
      const uint32_t lr = s_lrank[idx];
      if (lr != 0xffffu) {
        const uint32_t item = src[idx];
        const uint32_t kr = s_krank[s_cls[item]];
        dst[s_wcnt[((kr >> shift) & (kDigits - 1)) * kXWarps + wid] + lr] = (uint16_t)item;
      }
    }
  }
  __syncthreads();
  return (int)total;
}

__global__ void __launch_bounds__(kXThreads, 2)
explore_groups_kernel(ExploreArgs a) {
  FFB_DYN_SMEM(smem_raw);
  __shared__ double s_kr[kKsWidth];
  __shared__ double s_ca[kMaxClassA * kClassAWidth];     // factored model: rows per (threads, regs) class ...
  __shared__ double s_cb[33 * kClassBWidth];             // ... and per clipped block_x
  __shared__ double s_part[kXThreads / 32 + 1];
  __shared__ uint32_t s_pc[kXThreads / 32];
  __shared__ unsigned long long s_pm[kXThreads / 32];
  __shared__ unsigned int s_nuniq;
  __shared__ unsigned long long s_base;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int J = a.n_shapes, C = a.n_caps, G = J * C, NB = a.nb;
  const int64_t g = blockIdx.x;
  const int64_t k = g / a.n_specs;
  const int s = (int)(g - k * a.n_specs);

  // shared-memory carve-up
  double* s_e = reinterpret_cast<double*>(smem_raw);                              // [G]
  double* s_t = s_e + G;                                                          // [J]
  uint32_t* s_slots = reinterpret_cast<uint32_t*>(s_t + J);                       // [n_slots] hash table: representative candidate, or kEmpty
  //   ... the bucket arrays reuse the table once the classes are known
  unsigned long long* s_bmin = reinterpret_cast<unsigned long long*>(s_slots);    // [NB] min t per bucket -> exclusive prefix-min
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_bmin + NB);                     // [NB] counts -> starts -> ends
  //   ... and the radix counters / local ranks reuse it after that
  uint32_t* s_wcnt = s_slots;                                                     // [kDigits * kXWarps]
  uint16_t* s_lrank = reinterpret_cast<uint16_t*>(s_wcnt + kDigits * kXWarps);    // [G]
  uint16_t* s_cls = reinterpret_cast<uint16_t*>(s_slots + a.n_slots);             // [G] candidate -> representative
  uint16_t* s_krank = s_cls + G;                                                  // [G] per representative: class number in key order, 0xffff = dropped
  uint16_t* s_list = s_krank + G;                                                 // [G] representatives grouped by bucket; later a sort buffer
  uint16_t* s_sorted = s_list + G;                                                // [G] representative | keep << 15, in key order; later a sort buffer
  constexpr uint32_t kEmpty = 0xffffffffu;

  const double* f = a.feat + k * FFB_FEAT_WIDTH;
  const double* sp = a.tb.spec + (size_t)s * FFB_SPEC_WIDTH;
  const double* sd = a.tb.sd + (size_t)s * kSdWidth;
  const int64_t shared_dyn = a.res[2 * k + 0], total_blocks = a.res[2 * k + 1];
  if (tid == 0) {
    eval_kernel_spec(f, shared_dyn, total_blocks, sp, sd, a.tb.psm + (size_t)s * a.tb.psm_n, s_kr);
    s_nuniq = 0;
  }
  for (int b = tid; b < a.n_slots; b += kXThreads) s_slots[b] = kEmpty;
  __syncthreads();

  // ---- 1. the model: one thread per shape, cap axis innermost ----
  double tmin = INFINITY;
  const double2* ct = reinterpret_cast<const double2*>(a.tb.cap_tab + (size_t)s * C * 4);
  // the class rows first (32 + 32 for the reference's 464 shapes), then two divides per shape; kernels whose row
  // carries override columns, and shape tables with too many classes, evaluate every shape in full
  const bool classes = a.tb.n_a > 0 && a.tb.n_a <= kMaxClassA && f[FFB_F_OVR] == 0.0;
  if (classes) {
    for (int i = tid; i < a.tb.n_a + a.tb.n_b; i += kXThreads) {
      if (i < a.tb.n_a) eval_class_a(f, sp, sd, s_kr, a.tb.a_rep[2 * i], a.tb.a_rep[2 * i + 1], shared_dyn, total_blocks, s_ca + i * kClassAWidth);
      else eval_class_b(f, sp, sd, a.tb.b_rep[i - a.tb.n_a], s_cb + (i - a.tb.n_a) * kClassBWidth);
    }
    __syncthreads();
  }
  const double p_static = sp[FFB_S_P_STATIC], e_over = sp[FFB_S_E_OVERHEAD];
  for (int j = tid; j < J; j += kXThreads) {
    double t_exec, p_pre;
    bool valid;
    if (classes) {
      const int32_t cls = a.tb.shape_cls[j];
      const double* ca = s_ca + (cls & 0xffff) * kClassAWidth;
      eval_shape(sp, s_kr, ca, s_cb + (cls >> 16) * kClassBWidth, a.tb.shape_log[j], &t_exec, &p_pre);
      valid = ca[CA_VALID] != 0.0;
    } else {
      Unit u;
      eval_unit(f, sp, sd, s_kr, a.tb.shape + 4 * j, a.tb.shape_log[j], shared_dyn, total_blocks, 0, u);
      t_exec = u.t_exec; p_pre = u.p_pre; valid = u.valid;
    }
    bool any_ok = false;
    for (int c = 0; c < C; ++c) {
      const double2 sc_cap = ct[2 * c], room_ok = ct[2 * c + 1];
      double p_dyn;
      bool limited;
      const double e = eval_cap(t_exec, p_pre, p_static, e_over, sc_cap.x, sc_cap.y, room_ok.x, &p_dyn, &limited);
      const bool ok = valid && room_ok.y != 0.0;
      s_e[j * C + c] = ok ? e + 0.0 : INFINITY;            // (+ 0.0: -0.0 and 0.0 are one key)
      any_ok = any_ok || ok;
    }
    const double tj = any_ok ? t_exec + 0.0 : INFINITY;
    s_t[j] = tj;
    tmin = tj < tmin ? tj : tmin;
  }
  // ---- 2. t_peak and the floor (explorer.py:209-210) ----
  const double t_peak = block_min_d(tmin, s_part);
  const double thr = (a.rho > 0.0) ? t_peak / a.rho : INFINITY;
  // ---- 3. classes of equal (e, t) ----
  double emin = INFINITY, emax = -INFINITY;
  const uint32_t smask = (uint32_t)a.n_slots - 1u;
  for (int i = tid; i < G; i += kXThreads) {
    const int j = div_c_of((unsigned)i, a.div_c);
    const double ev = s_e[i], tv = s_t[j];
    uint32_t rep = kEmpty;
    if (tv <= thr && ev < INFINITY && tv < INFINITY) {
      emin = ev < emin ? ev : emin; emax = ev > emax ? ev : emax;
      unsigned long long h = ((unsigned long long)__double_as_longlong(ev) ^ ((unsigned long long)__double_as_longlong(tv) * 0x9e3779b97f4a7c15ull)) * 0xbf58476d1ce4e5b9ull;
      uint32_t p = (uint32_t)(h >> 40) & smask;
      for (;;) {
        uint32_t v = reinterpret_cast<volatile uint32_t*>(s_slots)[p];
        if (v == kEmpty) {
          v = atomicCAS(&s_slots[p], kEmpty, (uint32_t)i);
          if (v == kEmpty) { rep = (uint32_t)i; break; }
        }
        if (s_e[v] == ev && s_t[div_c_of(v, a.div_c)] == tv) { rep = v; break; }
        p = (p + 1) & smask;
      }
    }
    s_cls[i] = (uint16_t)rep;                              // 0xffff: not eligible
  }
  emin = block_min_d(emin, s_part);
  emax = -block_min_d(-emax, s_part);                      // (the barriers inside also close the table phase)
  const double span = emax - emin;
  const double scale = (span > 0.0 && span < INFINITY) ? (double)(NB - 1) / span : 0.0;
  auto bucket_of = [&](double ev) -> int {
    int b = (int)((ev - emin) * scale);
    return b < 0 ? 0 : (b > NB - 1 ? NB - 1 : b);
  };
  for (int b = tid; b < NB; b += kXThreads) { s_cnt[b] = 0; s_bmin[b] = ~0ull; }      // the table is dead: its space holds the buckets
  __syncthreads();
  // ---- 4a. bucket counts and per-bucket min t over the representatives ----
  unsigned n_mine = 0;
  for (int i = tid; i < G; i += kXThreads) {
    if (s_cls[i] != (uint16_t)i) continue;
    const int b = bucket_of(s_e[i]);
    atomicAdd(&s_cnt[b], 1u);
    atomicMin(&s_bmin[b], ord_bits(s_t[div_c_of((unsigned)i, a.div_c)]));
    ++n_mine;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) n_mine += __shfl_xor_sync(kXAll, n_mine, d);
  if (lane == 0 && n_mine) atomicAdd(&s_nuniq, n_mine);
  __syncthreads();
  // ---- 4b. bucket starts, exclusive prefix-min of t ----
  scan_buckets(s_cnt, s_bmin, NB, s_pc, s_pm);
  const int n_uniq = (int)s_nuniq;
  // ---- 4c. scatter (s_cnt[b] ends as the END of bucket b) ----
  for (int i = tid; i < G; i += kXThreads)
    if (s_cls[i] == (uint16_t)i) s_list[atomicAdd(&s_cnt[bucket_of(s_e[i])], 1u)] = (uint16_t)i;
  __syncthreads();
  // ---- 4d. rank inside the bucket + the dominance filter (keys are unique: no tie-break needed) ----
  for (int q = tid; q < n_uniq; q += kXThreads) {
    const int i = s_list[q];
    const double ev = s_e[i], tv = s_t[div_c_of((unsigned)i, a.div_c)];
    const int b = bucket_of(ev);
    const int lo = b ? (int)s_cnt[b - 1] : 0, hi = (int)s_cnt[b];
    int rank = lo;
    bool dominated = s_bmin[b] < ord_bits(tv);          // some candidate in a lower bucket (strictly lower e) has lower t
    for (int m = lo; m < hi; ++m) {
      const int i2 = s_list[m];
      const double e2 = s_e[i2], t2 = s_t[div_c_of((unsigned)i2, a.div_c)];
      if (e2 < ev) { ++rank; dominated = dominated || t2 < tv; }
      else if (e2 == ev && t2 < tv) ++rank;
    }
    s_sorted[rank] = (uint16_t)(i | (dominated ? 0 : 0x8000));
  }
  __syncthreads();
  // ---- 5a. number the kept classes in key order ----
  const int per = (n_uniq + kXThreads - 1) / kXThreads;
  const int lo = tid * per < n_uniq ? tid * per : n_uniq, hi = lo + per < n_uniq ? lo + per : n_uniq;
  uint32_t mine = 0;
  for (int p = lo; p < hi; ++p) mine += s_sorted[p] >> 15;
  uint32_t incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) { const uint32_t o = __shfl_up_sync(kXAll, incl, d); if (lane >= d) incl += o; }
  if (lane == 31) s_pc[wid] = incl;
  __syncthreads();
  uint32_t before = 0, n_kept = 0;
#pragma unroll
  for (int w = 0; w < kXWarps; ++w) { if (w < wid) before += s_pc[w]; n_kept += s_pc[w]; }
  uint32_t at = before + incl - mine;
  for (int p = lo; p < hi; ++p) {
    const uint32_t v = s_sorted[p];
    s_krank[v & 0x7fffu] = (v >> 15) ? (uint16_t)at++ : (uint16_t)0xffffu;
  }
  __syncthreads();
  // ---- 5b. stable radix sort of the candidates (tie order in) by class number ----
  int bits = 0;
  while ((1u << bits) < n_kept) ++bits;
  uint16_t* bufs[2] = {s_list, s_sorted};
  int total = radix_pass<true>(a.by_tie, bufs[0], G, 0, s_cls, s_krank, s_wcnt, s_lrank, s_pc);
  int cur = 0;
  for (int shift = 6; shift < bits; shift += 6) {
    radix_pass<false>(bufs[cur], bufs[cur ^ 1], total, shift, s_cls, s_krank, s_wcnt, s_lrank, s_pc);
    cur ^= 1;
  }
  const uint16_t* front = bufs[cur];
  if (tid == 0) {
    if (a.front_n) a.front_n[g] = (uint32_t)total;
    if (a.tpeak) a.tpeak[g] = t_peak;
    unsigned long long base = 0;
    if (a.front_off) {
      base = atomicAdd(a.front_total, (unsigned long long)total);
      a.front_off[g] = (int64_t)base;
      if (base + total > (unsigned long long)a.cap_front && a.status) atomicOr(a.status, 1u << FFB_E_CAPACITY);
    } else if ((int64_t)total > a.cap_front && a.status) atomicOr(a.status, 1u << FFB_E_CAPACITY);
    s_base = base;
  }
  __syncthreads();
  const unsigned long long obase = a.front_off ? s_base : (unsigned long long)g * (unsigned long long)a.cap_front;
  const unsigned long long olimit = a.front_off ? (unsigned long long)a.cap_front : obase + (unsigned long long)a.cap_front;
  for (int r = tid; r < total; r += kXThreads) {
    const uint32_t i = front[r];
    const unsigned long long o = obase + (unsigned)r;
    if (o < olimit) {
      if (a.front_idx) a.front_idx[o] = i;
      if (a.front_e) a.front_e[o] = s_e[i];
      if (a.front_t) a.front_t[o] = s_t[div_c_of(i, a.div_c)];
    }
  }
}

}  // namespace

extern "C" int32_t ffb_explore_groups(FfbContext* ctx, const FfbExploreDesc* d, void* stream_) {
  if (!ctx || !d) return FFB_E_BAD_ARGUMENT;
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t K = d->n_kernels, S = d->n_specs, J = d->n_shapes, C = d->n_caps;
  if (K < 0 || S <= 0 || J < 0 || C <= 0 || S > (1 << 20) || C > 4096 || d->cap_front < 0)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_explore_groups: bad extents K=%lld S=%lld J=%lld C=%lld",
                    (long long)K, (long long)S, (long long)J, (long long)C);
  if (!d->d_feat || !d->d_res || !d->h_spec || !d->h_shape || !d->h_cap || !d->d_front_n)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_explore_groups: null input");
  if (!(d->rho <= 1.0)) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_explore_groups: rho must be <= 1");
  if (K == 0) return FFB_OK;
  const int64_t G = J * C;
  if (G > 32767 || K * S > 0x7fffffffLL)
    return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_explore_groups: %lld candidates per group (limit 32767); use ffb_predict_grid + ffb_skyline_groups",
                    (long long)G);
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));
  if (J == 0) {
    FFB_CUDA(ctx, cudaMemsetAsync(d->d_front_n, 0, (size_t)(K * S) * 4, stream));
    return FFB_OK;
  }
  int nb = kXThreads;
  while (nb < G && nb < 2048) nb <<= 1;                       // ~1 unique key per bucket
  int n_slots = 64;
  while (n_slots < 2 * G) n_slots <<= 1;
  if ((size_t)n_slots * 4 < (size_t)nb * 12) n_slots = nb * 4;             // the bucket arrays reuse the table's space ...
  while ((size_t)n_slots * 4 < (size_t)kDigits * kXWarps * 4 + (size_t)G * 2 + 16) n_slots <<= 1;      // ... and so do the radix counters
  const size_t smem = (size_t)G * 8 + (size_t)J * 8 + (size_t)n_slots * 4 + (size_t)G * 8 + 64;
  const size_t limit = ctx->smem_optin ? ctx->smem_optin - 2048 : 96 * 1024;
  if (smem > limit)
    return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_explore_groups: a group of %lld candidates needs %zu B of shared memory; "
                    "use ffb_predict_grid + ffb_skyline_groups", (long long)G, smem);
  Tables tb;
  uint32_t host_err = 0;
  int32_t rc = ffb_build_tables(ctx, d->h_spec, d->h_shape, d->h_cap, FfbTableDims{S, J, C}, 0, stream, &tb, &host_err);
  if (rc) return rc;
  // candidates in tie order: (bx, by, bz, regs, j) over the shapes, then (cap, c) over the caps (explorer.py:113-119)
  std::vector<int> js(J), cs(C);
  std::iota(js.begin(), js.end(), 0);
  std::iota(cs.begin(), cs.end(), 0);
  const int32_t* hs = d->h_shape;
  std::sort(js.begin(), js.end(), [hs](int x, int y) {
    for (int q = 0; q < 4; ++q) if (hs[4 * x + q] != hs[4 * y + q]) return hs[4 * x + q] < hs[4 * y + q];
    return x < y; });
  const double* hc = d->h_cap;
  std::sort(cs.begin(), cs.end(), [hc](int x, int y) { return hc[x] != hc[y] ? hc[x] < hc[y] : x < y; });
  const size_t tie_bytes = ((size_t)G * 2 + 15) & ~(size_t)15;
  rc = ffb_reserve(ctx, &ctx->d_explore, tie_bytes + 64);
  if (rc) return rc;
  std::vector<uint16_t> by_tie((size_t)G);
  for (int64_t r = 0; r < J; ++r)
    for (int64_t q = 0; q < C; ++q) by_tie[(size_t)(r * C + q)] = (uint16_t)(js[r] * C + cs[q]);
  if (ctx->explore_shadow != by_tie || ctx->explore_shadow_dev != ctx->d_explore.p) {   // same shapes / caps as the last call: nothing to upload
    FFB_CUDA(ctx, cudaStreamSynchronize(stream));              // (the previous launch may still read the old table)
    FFB_CUDA(ctx, cudaMemcpyAsync(ctx->d_explore.p, by_tie.data(), by_tie.size() * 2, cudaMemcpyHostToDevice, stream));
    FFB_CUDA(ctx, cudaStreamSynchronize(stream));              // pageable source: keep it alive until the copy is done
    ctx->explore_shadow = by_tie;
    ctx->explore_shadow_dev = ctx->d_explore.p;
  }
  ExploreArgs a = {};
  a.feat = d->d_feat; a.res = d->d_res; a.tb = tb; a.n_groups = K * S;
  a.n_specs = (int)S; a.n_shapes = (int)J; a.n_caps = (int)C;
  a.div_c = C == 1 ? 0u : (uint32_t)((0x100000000ull + (uint64_t)C - 1) / (uint64_t)C);   // exact for i * (C - 1) < 2^32
  a.by_tie = (const uint16_t*)ctx->d_explore.p;
  a.rho = d->rho; a.nb = nb; a.n_slots = n_slots;
  a.front_idx = d->d_front_idx; a.front_n = d->d_front_n; a.tpeak = d->d_tpeak; a.cap_front = d->cap_front;
  a.front_off = d->d_front_off; a.front_e = d->d_front_e; a.front_t = d->d_front_t; a.status = d->d_status;
  if (d->d_front_off) {
    a.front_total = (unsigned long long*)((char*)ctx->d_explore.p + tie_bytes);
    FFB_CUDA(ctx, cudaMemsetAsync(a.front_total, 0, 8, stream));
  }
  FFB_CUDA(ctx, cudaFuncSetAttribute(explore_groups_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  FFB_LAUNCH(explore_groups_kernel, (unsigned)(K * S), kXThreads, smem, stream, a);
  rc = ffb_check_launch(ctx, "explore_groups_kernel");
  if (rc) return rc;
  if (host_err)
    for (int code = 1; code < 32; ++code)
      if (host_err & (1u << code)) return ffb_fail(ctx, code, "ffb_explore_groups: spec/cap check failed (status %d)", code);
  return FFB_OK;
}
