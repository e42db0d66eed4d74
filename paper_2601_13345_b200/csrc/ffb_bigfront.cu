// K4, large fronts: exact Pareto front of a candidate set whose front does not fit one CTA
// (tie-heavy sets such as pkg/tests/test_acceptance.py:114-115 at 10^8..10^9 candidates keep a
// constant FRACTION of the set: every point with the lowest e or the lowest t is on the front).
//
// explorer.py:111-140 restated with device-wide primitives:
//   _sorted_entries   stable LSD radix sort of a permutation by (e, t, id): 8-bit digits, one
//                     histogram + scan + stable scatter per digit, digits that are constant over
//                     the set are skipped;
//   pareto_front      over the sorted order, `best_t` = min t over STRICTLY lower e is the inclusive
//                     prefix-min of t read just in front of the candidate's equal-e run; a candidate
//                     stays iff not (best_t < t) and t <= t_peak / rho (explorer.py:209-211);
//   output            compaction in sorted order.
// Called by ffb_skyline when its chunk fronts stop shrinking (ffb_skyline.cu).  Two objectives.
#include "ffb_common.cuh"

#include <math.h>
#include <string.h>

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;                         // per thread: tiles of 4096
constexpr int kTileN = kThreads * kItems;
constexpr unsigned kAll = 0xffffffffu;

FFB_HD uint64_t ordered_bits(double v) {
#if defined(__CUDA_ARCH__) || defined(FFB_SIMT_EMUL)
  uint64_t b = (uint64_t)__double_as_longlong(v);
#else
  uint64_t b; memcpy(&b, &v, 8);
#endif
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// ---- block-wide helpers (kThreads threads) ----------------------------------------------------
FFB_D uint32_t block_excl_sum(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) { const uint32_t o = __shfl_up_sync(kAll, x, d); if (lane >= d) x += o; }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t y = lane < kThreads / 32 ? s_warp[lane] : 0u, z = y;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) { const uint32_t o = __shfl_up_sync(kAll, z, d); if (lane >= d) z += o; }
    if (lane < kThreads / 32) s_warp[lane] = z - y;
    if (lane == 31) s_warp[32] = z;
  }
  __syncthreads();
  const uint32_t r = s_warp[w] + x - v;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

// ---- generic three-kernel exclusive scan of u32 sums (digit tables, keep flags) -----------------
__global__ void __launch_bounds__(kThreads) sum_reduce_kernel(const uint32_t* v, int64_t n, uint32_t* part) {
  __shared__ uint32_t s_warp[33];
  const int64_t base = (int64_t)blockIdx.x * kTileN;
  uint32_t acc = 0;
  for (int k = 0; k < kItems; ++k) { const int64_t i = base + (int64_t)k * kThreads + threadIdx.x; if (i < n) acc += v[i]; }
  uint32_t tot;
  block_excl_sum(acc, s_warp, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(kThreads) sum_scan_parts_kernel(uint32_t* part, int64_t n_part, unsigned long long* grand) {
  __shared__ uint32_t s_warp[33];
  uint32_t carry = 0;
  for (int64_t b0 = 0; b0 < n_part; b0 += kThreads) {
    const int64_t i = b0 + threadIdx.x;
    const uint32_t v = i < n_part ? part[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_sum(v, s_warp, &tot);
    if (i < n_part) part[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && grand) *grand = carry;
}
__global__ void __launch_bounds__(kThreads) sum_apply_kernel(uint32_t* v, int64_t n, const uint32_t* part) {
  // exclusive scan inside the tile, thread-contiguous items so that the scan follows the index order
  __shared__ uint32_t s_warp[33];
  const int64_t base = (int64_t)blockIdx.x * kTileN + (int64_t)threadIdx.x * kItems;
  uint32_t loc[kItems], acc = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) { const int64_t i = base + k; loc[k] = i < n ? v[i] : 0u; acc += loc[k]; }
  uint32_t tot;
  uint32_t run = part[blockIdx.x] + block_excl_sum(acc, s_warp, &tot);
#pragma unroll
  for (int k = 0; k < kItems; ++k) { const int64_t i = base + k; if (i < n) v[i] = run; run += loc[k]; }
}

// ---- radix sort of (key, perm) pairs by one 8-bit digit -------------------------------------------
struct SortArgs {
  const uint64_t* key_in; const uint32_t* perm_in;
  uint64_t* key_out; uint32_t* perm_out;
  int64_t n;
  int shift;
  uint32_t* table;                  // [256 * n_tiles], digit-major
  int64_t n_tiles;
};
__global__ void __launch_bounds__(kThreads) digit_hist_kernel(SortArgs a) {
  __shared__ uint32_t s_cnt[256];
  s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTileN;
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
    if (i < a.n) atomicAdd(&s_cnt[(uint32_t)(a.key_in[i] >> a.shift) & 255u], 1u);
  }
  __syncthreads();
  a.table[(int64_t)threadIdx.x * a.n_tiles + blockIdx.x] = s_cnt[threadIdx.x];
}
__global__ void __launch_bounds__(kThreads) digit_scatter_kernel(SortArgs a) {
  __shared__ uint32_t s_off[256];                      // next output slot per digit for this tile
  __shared__ uint32_t s_wcnt[kThreads / 32][256];      // per-warp digit counts of the round
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s_off[threadIdx.x] = a.table[(int64_t)threadIdx.x * a.n_tiles + blockIdx.x];
  const int64_t base = (int64_t)blockIdx.x * kTileN;
  for (int k = 0; k < kItems; ++k) {
    for (int q = 0; q < kThreads / 32; ++q) s_wcnt[q][threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
    const bool live = i < a.n;
    uint64_t key = 0; uint32_t pv = 0, d = 256u + (uint32_t)lane;      // dead lanes match nobody
    if (live) { key = a.key_in[i]; pv = a.perm_in[i]; d = (uint32_t)(key >> a.shift) & 255u; }
    const unsigned peers = __match_any_sync(kAll, d);
    const uint32_t rank = (uint32_t)__popc(peers & ((1u << lane) - 1u));
    if (live && rank == 0) s_wcnt[w][d] = (uint32_t)__popc(peers);
    __syncthreads();
    uint32_t before = 0;
    if (live) for (int q = 0; q < w; ++q) before += s_wcnt[q][d];
    if (live) {
      const uint32_t at = s_off[d] + before + rank;
      a.key_out[at] = key; a.perm_out[at] = pv;
    }
    __syncthreads();
    uint32_t tot = 0;
    for (int q = 0; q < kThreads / 32; ++q) tot += s_wcnt[q][threadIdx.x];
    s_off[threadIdx.x] += tot;
    __syncthreads();
  }
}
// or / and of all keys: digits whose bits are the same in every key need no pass
__global__ void __launch_bounds__(kThreads) key_bits_kernel(const uint64_t* key, int64_t n, unsigned long long* acc) {
  unsigned long long o = 0, an = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) { o |= key[i]; an &= key[i]; }
  for (int d = 16; d > 0; d >>= 1) { o |= __shfl_xor_sync(kAll, o, d); an &= __shfl_xor_sync(kAll, an, d); }
  if ((threadIdx.x & 31) == 0) { atomicOr(&acc[0], o); atomicAnd(&acc[1], an); }
}

// ---- keys, gathers, the front rule ------------------------------------------------------------------
struct BigArgs {
  const double* e; const double* t; const uint64_t* id;
  int64_t n;
  uint64_t* key; uint32_t* perm;
  uint64_t* pmin;                  // inclusive prefix-min of t (ordered bits) over the sorted order
  uint32_t* keep;                  // keep flags, then output positions
  uint32_t* part;                  // per-tile partials
  unsigned long long* scal;        // [0] or-bits [1] and-bits [2] min t bits [3] count
  double rho;
  uint64_t* out_id; double* out_e; double* out_t; int64_t out_cap;
  uint32_t* overflow;
};
__global__ void __launch_bounds__(kThreads) iota_min_kernel(BigArgs a) {
  unsigned long long mn = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * kThreads) {
    a.perm[i] = (uint32_t)i;
    const double tv = a.t[i];
    if (tv == tv) { const unsigned long long b = (unsigned long long)ordered_bits(tv); mn = b < mn ? b : mn; }
  }
  for (int d = 16; d > 0; d >>= 1) { const unsigned long long o = __shfl_xor_sync(kAll, mn, d); mn = o < mn ? o : mn; }
  if ((threadIdx.x & 31) == 0) atomicMin(&a.scal[2], mn);
}
// which: 0 id, 1 t, 2 e
__global__ void __launch_bounds__(kThreads) gather_key_kernel(BigArgs a, int which) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * kThreads) {
    const uint32_t p = a.perm[i];
    uint64_t k;
    if (which == 0) k = a.id ? a.id[p] : (uint64_t)p;
    else k = ordered_bits((which == 1 ? a.t[p] : a.e[p]) + 0.0);          // -0.0 sorts with 0.0
    a.key[i] = k;
  }
}
// inclusive prefix-min of t over the sorted order, three kernels like the sum scan
__global__ void __launch_bounds__(kThreads) min_reduce_kernel(BigArgs a) {
  __shared__ unsigned long long s_w[kThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kTileN;
  unsigned long long mn = ~0ull;
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
    if (i < a.n) { const double tv = a.t[a.perm[i]]; const unsigned long long b = tv == tv ? (unsigned long long)ordered_bits(tv) : ~0ull; mn = b < mn ? b : mn; }
  }
  for (int d = 16; d > 0; d >>= 1) { const unsigned long long o = __shfl_xor_sync(kAll, mn, d); mn = o < mn ? o : mn; }
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < kThreads / 32; ++q) mn = s_w[q] < mn ? s_w[q] : mn;
    reinterpret_cast<unsigned long long*>(a.pmin)[a.n + blockIdx.x] = mn;      // tile minima live behind the n prefix values
  }
}
__global__ void min_scan_parts_kernel(BigArgs a, int64_t n_tiles) {               // one lane: n_tiles <= n / 4096
  if (threadIdx.x != 0) return;
  unsigned long long* part = reinterpret_cast<unsigned long long*>(a.pmin) + a.n;
  unsigned long long run = ~0ull;
  for (int64_t b = 0; b < n_tiles; ++b) { const unsigned long long v = part[b]; part[b] = run; run = v < run ? v : run; }
}
__global__ void __launch_bounds__(kThreads) min_apply_kernel(BigArgs a) {
  __shared__ unsigned long long s_w[kThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kTileN + (int64_t)threadIdx.x * kItems;
  unsigned long long loc[kItems], mn = ~0ull;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t i = base + k;
    loc[k] = ~0ull;
    if (i < a.n) { const double tv = a.t[a.perm[i]]; if (tv == tv) loc[k] = (unsigned long long)ordered_bits(tv); }
    mn = loc[k] < mn ? loc[k] : mn;
  }
  unsigned long long incl = mn;
  for (int d = 1; d < 32; d <<= 1) { const unsigned long long o = __shfl_up_sync(kAll, incl, d); if (lane >= d && o < incl) incl = o; }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  unsigned long long run = reinterpret_cast<const unsigned long long*>(a.pmin)[a.n + blockIdx.x];      // everything in front of the tile
  for (int q = 0; q < w; ++q) run = s_w[q] < run ? s_w[q] : run;
  const unsigned long long prev = __shfl_up_sync(kAll, incl, 1);
  if (lane > 0) run = prev < run ? prev : run;
#pragma unroll
  for (int k = 0; k < kItems; ++k) { const int64_t i = base + k; run = loc[k] < run ? loc[k] : run; if (i < a.n) a.pmin[i] = run; }
}
// keep flag of sorted position i: its equal-e run starts at s (found by walking back over equal e: runs of ties can
// be long, so the walk uses the fact that t ascends inside a run - a binary search over [0, i] on the sorted e keys)
__global__ void __launch_bounds__(kThreads) keep_kernel(BigArgs a) {
  const unsigned long long tmin = a.scal[2];
  double thr = INFINITY;
  if (a.rho > 0.0 && tmin != ~0ull) {
    const unsigned long long b = (tmin & 0x8000000000000000ull) ? (tmin & 0x7fffffffffffffffull) : ~tmin;
    thr = __longlong_as_double((long long)b) / a.rho;                               // explorer.py:209-211
  }
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * kThreads) {
    const uint64_t ke = a.key[i];                        // sorted e keys (last sort key)
    int64_t lo = 0, hi = i;                              // first position with this e: gallop back, then bisect
    for (int64_t step = 1; step <= i; step <<= 1) {
      if (a.key[i - step] < ke) { lo = i - step + 1; break; }
      hi = i - step;
    }
    while (lo < hi) { const int64_t mid = (lo + hi) >> 1; if (a.key[mid] < ke) lo = mid + 1; else hi = mid; }
    const double tv = a.t[a.perm[i]];
    bool keep = tv <= thr || !(a.rho > 0.0);
    if (a.rho > 0.0 && !(tv <= thr)) keep = false;
    if (keep && lo > 0 && tv == tv) keep = !(a.pmin[lo - 1] < (unsigned long long)ordered_bits(tv));
    a.keep[i] = keep ? 1u : 0u;
  }
}
__global__ void __launch_bounds__(kThreads) emit_kernel(BigArgs a, const uint32_t* flags) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * kThreads) {
    if (!flags[i]) continue;
    const int64_t at = a.keep[i];
    if (at >= a.out_cap) { *a.overflow = 1u; continue; }
    const uint32_t p = a.perm[i];
    a.out_id[at] = a.id ? a.id[p] : (uint64_t)p;
    if (a.out_e) a.out_e[at] = a.e[p];
    if (a.out_t) a.out_t[at] = a.t[p];
  }
}

}  // namespace

// Front of (e, t, id)[0, n), n < 2^32, in reference order.  Device scratch: ctx->d_bigfront (the inputs may live in
// ctx->d_sky).  Synchronises (the count is returned).
int32_t ffb_big_front(FfbContext* ctx, const double* d_e, const double* d_t, const uint64_t* d_id, int64_t n, double rho,
                      uint64_t* d_front_id, double* d_front_e, double* d_front_t, int64_t cap_front,
                      int64_t* h_front_n, double* h_tpeak, cudaStream_t stream) {
  if (n <= 0 || n >= ((int64_t)1 << 32)) return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_skyline: %lld candidates left for the sort-based finish (limit 2^32)", (long long)n);
  const int64_t n_tiles = (n + kTileN - 1) / kTileN;
  size_t bytes = 0;
  auto take = [&](size_t count, size_t elem) { size_t off = bytes; bytes += (count * elem + 255) & ~(size_t)255; return off; };
  const size_t o_key0 = take((size_t)n, 8), o_key1 = take((size_t)n, 8), o_perm0 = take((size_t)n, 4), o_perm1 = take((size_t)n, 4),
               o_pmin = take((size_t)(n + n_tiles + 8), 8), o_keep = take((size_t)n, 4), o_flag = take((size_t)n, 4),
               o_table = take((size_t)(256 * n_tiles), 4), o_part = take((size_t)((256 * n_tiles + kTileN - 1) / kTileN + n_tiles + 8), 4),
               o_scal = take(8, 8);
  int32_t rc = ffb_reserve(ctx, &ctx->d_bigfront, bytes);
  if (rc) return rc;
  char* base = (char*)ctx->d_bigfront.p;
  uint64_t* key[2] = {(uint64_t*)(base + o_key0), (uint64_t*)(base + o_key1)};
  uint32_t* perm[2] = {(uint32_t*)(base + o_perm0), (uint32_t*)(base + o_perm1)};
  BigArgs a = {};
  a.e = d_e; a.t = d_t; a.id = d_id; a.n = n; a.rho = rho;
  a.pmin = (uint64_t*)(base + o_pmin); a.keep = (uint32_t*)(base + o_keep); a.part = (uint32_t*)(base + o_part);
  a.scal = (unsigned long long*)(base + o_scal);
  a.out_id = d_front_id; a.out_e = d_front_e; a.out_t = d_front_t; a.out_cap = cap_front;
  a.overflow = (uint32_t*)(a.scal + 4);
  uint32_t* flags = (uint32_t*)(base + o_flag);
  uint32_t* table = (uint32_t*)(base + o_table);
  int64_t g64 = (n + kThreads - 1) / kThreads;
  const unsigned grid = (unsigned)(g64 < (int64_t)ctx->sm_count * 8 ? g64 : (int64_t)ctx->sm_count * 8);
  const unsigned long long init[8] = {0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  FFB_CUDA(ctx, cudaMemcpyAsync(a.scal, init, sizeof(init), cudaMemcpyHostToDevice, stream));
  int cur = 0;
  a.perm = perm[cur]; a.key = key[cur];
  FFB_LAUNCH(iota_min_kernel, grid, kThreads, 0, stream, a);
  for (int which = 0; which < 3; ++which) {                  // least significant key first: id, t, e
    a.perm = perm[cur]; a.key = key[cur];
    FFB_LAUNCH(gather_key_kernel, grid, kThreads, 0, stream, a, which);
    const unsigned long long reset[2] = {0ull, ~0ull};
    unsigned long long bits[2];
    FFB_CUDA(ctx, cudaMemcpyAsync(a.scal, reset, sizeof(reset), cudaMemcpyHostToDevice, stream));
    FFB_LAUNCH(key_bits_kernel, grid, kThreads, 0, stream, key[cur], n, a.scal);
    FFB_CUDA(ctx, cudaMemcpyAsync(bits, a.scal, sizeof(bits), cudaMemcpyDeviceToHost, stream));
    FFB_CUDA(ctx, cudaStreamSynchronize(stream));
    const unsigned long long varying = bits[0] ^ bits[1];     // bits that differ somewhere
    for (int shift = 0; shift < 64; shift += 8) {
      if (!((varying >> shift) & 255ull)) continue;
      SortArgs s = {};
      s.key_in = key[cur]; s.perm_in = perm[cur]; s.key_out = key[cur ^ 1]; s.perm_out = perm[cur ^ 1];
      s.n = n; s.shift = shift; s.table = table; s.n_tiles = n_tiles;
      FFB_LAUNCH(digit_hist_kernel, (unsigned)n_tiles, kThreads, 0, stream, s);
      const int64_t m = 256 * n_tiles, m_tiles = (m + kTileN - 1) / kTileN;
      FFB_LAUNCH(sum_reduce_kernel, (unsigned)m_tiles, kThreads, 0, stream, table, m, a.part);
      FFB_LAUNCH(sum_scan_parts_kernel, 1, kThreads, 0, stream, a.part, m_tiles, (unsigned long long*)nullptr);
      FFB_LAUNCH(sum_apply_kernel, (unsigned)m_tiles, kThreads, 0, stream, table, m, a.part);
      FFB_LAUNCH(digit_scatter_kernel, (unsigned)n_tiles, kThreads, 0, stream, s);
      cur ^= 1;
    }
  }
  // key[cur] holds the sorted e keys, perm[cur] the order
  a.perm = perm[cur]; a.key = key[cur];
  FFB_LAUNCH(min_reduce_kernel, (unsigned)n_tiles, kThreads, 0, stream, a);
  FFB_LAUNCH(min_scan_parts_kernel, 1, 32, 0, stream, a, n_tiles);
  FFB_LAUNCH(min_apply_kernel, (unsigned)n_tiles, kThreads, 0, stream, a);
  FFB_LAUNCH(keep_kernel, grid, kThreads, 0, stream, a);
  FFB_CUDA(ctx, cudaMemcpyAsync(flags, a.keep, (size_t)n * 4, cudaMemcpyDeviceToDevice, stream));
  FFB_LAUNCH(sum_reduce_kernel, (unsigned)n_tiles, kThreads, 0, stream, a.keep, n, a.part);
  FFB_LAUNCH(sum_scan_parts_kernel, 1, kThreads, 0, stream, a.part, n_tiles, a.scal + 3);
  FFB_LAUNCH(sum_apply_kernel, (unsigned)n_tiles, kThreads, 0, stream, a.keep, n, a.part);
  FFB_LAUNCH(emit_kernel, grid, kThreads, 0, stream, a, (const uint32_t*)flags);
  rc = ffb_check_launch(ctx, "big front");
  if (rc) return rc;
  unsigned long long h[5];
  FFB_CUDA(ctx, cudaMemcpyAsync(h, a.scal, sizeof(h), cudaMemcpyDeviceToHost, stream));
  FFB_CUDA(ctx, cudaStreamSynchronize(stream));
  if ((int64_t)h[3] > cap_front || (uint32_t)h[4])
    return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_skyline: front of %llu points exceeds the output capacity %lld", h[3], (long long)cap_front);
  *h_front_n = (int64_t)h[3];
  if (h_tpeak) {
    double tp = INFINITY;
    if (h[2] != ~0ull) { const unsigned long long b = (h[2] & 0x8000000000000000ull) ? (h[2] & 0x7fffffffffffffffull) : ~h[2]; memcpy(&tp, &b, 8); }
    *h_tpeak = tp;
  }
  return FFB_OK;
}
