// TEST-ONLY SIMT emulation shim.
//
// Compiles the repo's .cu kernels as plain C++ (g++ -x c++ -DFFB_SIMT_EMUL) so that the
// kernel LOGIC can be exercised by the CPU test-suite in a container without a GPU.
// One OS thread per CUDA thread, CTAs run one after another, __syncthreads/__syncwarp are
// pthread barriers, warp collectives exchange through a per-warp mailbox.
//
// This is test infrastructure, like oracle/: nothing under paper_2601_13345_b200/ loads
// the emulated library, bench.py never touches it, and the product path raises
// NativeLibraryMissing when libffb.so (the real nvcc build) or a CUDA device is absent.
#pragma once
#ifndef FFB_SIMT_EMUL
#error "simt_emul.h is only for the FFB_SIMT_EMUL host build"
#endif

#include <pthread.h>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>
#include <algorithm>

#define __global__
#define __device__
#define __host__
#define __forceinline__ inline
#define __noinline__
#define __restrict__
#define __launch_bounds__(...)
#define __align__(n) alignas(n)
#define __shared__ static
#define __constant__ static

struct uint3_ { unsigned x, y, z; };
struct dim3 {
  unsigned x, y, z;
  dim3(unsigned x_ = 1, unsigned y_ = 1, unsigned z_ = 1) : x(x_), y(y_), z(z_) {}
};
struct uint4 { unsigned x, y, z, w; };
struct uint2 { unsigned x, y; };
inline uint4 make_uint4(unsigned x, unsigned y, unsigned z, unsigned w) { uint4 r; r.x = x; r.y = y; r.z = z; r.w = w; return r; }
struct double2 { double x, y; };
struct alignas(16) int4 { int x, y, z, w; };

namespace simt {
struct WarpBox {
  pthread_barrier_t bar;
  unsigned long long slot[32];
};
struct Cta {
  pthread_barrier_t bar;
  std::vector<WarpBox*> warps;
  unsigned nthreads;
  int vote = 0;
};
extern thread_local uint3_ t_threadIdx, t_blockIdx;
extern thread_local dim3 t_blockDim, t_gridDim;
extern thread_local WarpBox* t_warp;
extern thread_local Cta* t_cta;
extern unsigned char* dyn_smem;
void launch(dim3 grid, dim3 block, size_t smem, const std::function<void()>& body);
}  // namespace simt

#define threadIdx (simt::t_threadIdx)
#define blockIdx (simt::t_blockIdx)
#define blockDim (simt::t_blockDim)
#define gridDim (simt::t_gridDim)
static const int warpSize = 32;

inline void __syncthreads() { pthread_barrier_wait(&simt::t_cta->bar); }
inline int __syncthreads_or(int p) {
  simt::Cta* c = simt::t_cta;
  if (p) __atomic_store_n(&c->vote, 1, __ATOMIC_SEQ_CST);
  pthread_barrier_wait(&c->bar);
  const int r = __atomic_load_n(&c->vote, __ATOMIC_SEQ_CST);
  pthread_barrier_wait(&c->bar);
  if (threadIdx.x == 0) __atomic_store_n(&c->vote, 0, __ATOMIC_SEQ_CST);
  pthread_barrier_wait(&c->bar);
  return r;
}
inline void __syncwarp(unsigned = 0xffffffffu) { pthread_barrier_wait(&simt::t_warp->bar); }
inline void __threadfence() { std::atomic_thread_fence(std::memory_order_seq_cst); }
inline void __threadfence_block() { std::atomic_thread_fence(std::memory_order_seq_cst); }

inline int simt_lane() { return (int)(threadIdx.x & 31u); }

template <typename T>
inline T simt_xchg(T v, int src) {
  static_assert(sizeof(T) <= 8, "shuffle payload");
  simt::WarpBox* w = simt::t_warp;
  unsigned long long raw = 0;
  memcpy(&raw, &v, sizeof(T));
  w->slot[simt_lane()] = raw;
  pthread_barrier_wait(&w->bar);
  unsigned long long got = w->slot[src & 31];
  pthread_barrier_wait(&w->bar);
  T out;
  memcpy(&out, &got, sizeof(T));
  return out;
}
template <typename T> inline T __shfl_sync(unsigned, T v, int src, int = 32) { return simt_xchg(v, src); }
template <typename T> inline T __shfl_up_sync(unsigned, T v, unsigned d, int = 32) {
  int l = simt_lane(); int s = l - (int)d; T o = simt_xchg(v, s < 0 ? l : s); return s < 0 ? v : o;
}
template <typename T> inline T __shfl_down_sync(unsigned, T v, unsigned d, int = 32) {
  int l = simt_lane(); int s = l + (int)d; T o = simt_xchg(v, s > 31 ? l : s); return s > 31 ? v : o;
}
template <typename T> inline T __shfl_xor_sync(unsigned, T v, int m, int = 32) { return simt_xchg(v, simt_lane() ^ m); }
inline unsigned __ballot_sync(unsigned, int pred) {
  simt::WarpBox* w = simt::t_warp;
  w->slot[simt_lane()] = pred ? 1ull : 0ull;
  pthread_barrier_wait(&w->bar);
  unsigned m = 0;
  for (int i = 0; i < 32; ++i) m |= (unsigned)(w->slot[i] & 1ull) << i;
  pthread_barrier_wait(&w->bar);
  return m;
}
template <typename T> inline unsigned __match_any_sync(unsigned, T v) {
  simt::WarpBox* w = simt::t_warp;
  unsigned long long raw = 0;
  memcpy(&raw, &v, sizeof(T));
  w->slot[simt_lane()] = raw;
  pthread_barrier_wait(&w->bar);
  unsigned m = 0;
  for (int i = 0; i < 32; ++i) m |= (unsigned)(w->slot[i] == raw) << i;
  pthread_barrier_wait(&w->bar);
  return m;
}
inline int __any_sync(unsigned m, int p) { return __ballot_sync(m, p) != 0; }
inline int __all_sync(unsigned m, int p) { return __ballot_sync(m, p) == 0xffffffffu; }

inline int __popc(unsigned v) { return __builtin_popcount(v); }
inline int __popcll(unsigned long long v) { return __builtin_popcountll(v); }
inline int __ffs(int v) { return __builtin_ffs(v); }
inline int __ffsll(long long v) { return __builtin_ffsll(v); }
inline int __clz(int v) { return v ? __builtin_clz((unsigned)v) : 32; }
inline int __clzll(long long v) { return v ? __builtin_clzll((unsigned long long)v) : 64; }
inline unsigned __brev(unsigned v) {
  unsigned r = 0; for (int i = 0; i < 32; ++i) r |= ((v >> i) & 1u) << (31 - i); return r;
}
inline long long __double_as_longlong(double d) { long long r; memcpy(&r, &d, 8); return r; }
inline double __longlong_as_double(long long v) { double r; memcpy(&r, &v, 8); return r; }
inline unsigned __vcmpeq4(unsigned a, unsigned b) {
  unsigned r = 0;
  for (int i = 0; i < 4; ++i) if (((a >> (8 * i)) & 0xffu) == ((b >> (8 * i)) & 0xffu)) r |= 0xffu << (8 * i);
  return r;
}
inline unsigned __funnelshift_r(unsigned lo, unsigned hi, unsigned sh) {
  const unsigned long long v = ((unsigned long long)hi << 32) | lo; return (unsigned)(v >> (sh & 31u));
}
inline int __popcll_(unsigned long long v) { return __builtin_popcountll(v); }
inline unsigned __byte_perm(unsigned a, unsigned b, unsigned s) {
  unsigned long long v = ((unsigned long long)b << 32) | a; unsigned r = 0;
  for (int i = 0; i < 4; ++i) { unsigned sel = (s >> (4 * i)) & 7u; r |= (unsigned)((v >> (8 * sel)) & 0xffu) << (8 * i); }
  return r;
}
template <typename T> inline T __ldg(const T* p) { return *p; }
inline double __dadd_rn(double a, double b) { return a + b; }
inline double __dmul_rn(double a, double b) { return a * b; }
inline double __ddiv_rn(double a, double b) { return a / b; }
inline unsigned __umulhi(unsigned a, unsigned b) { return (unsigned)(((unsigned long long)a * b) >> 32); }
inline unsigned long long __umul64hi(unsigned long long a, unsigned long long b) {
  return (unsigned long long)(((unsigned __int128)a * b) >> 64);
}

template <typename T> inline T atomicAdd(T* p, T v) { return __atomic_fetch_add(p, v, __ATOMIC_SEQ_CST); }
inline double atomicAdd(double* p, double v) {
  unsigned long long* q = (unsigned long long*)p; unsigned long long old = __atomic_load_n(q, __ATOMIC_SEQ_CST);
  for (;;) { double nv = __longlong_as_double((long long)old) + v; unsigned long long nb; memcpy(&nb, &nv, 8);
    if (__atomic_compare_exchange_n(q, &old, nb, false, __ATOMIC_SEQ_CST, __ATOMIC_SEQ_CST)) return __longlong_as_double((long long)old); }
}
template <typename T> inline T atomicOr(T* p, T v) { return __atomic_fetch_or(p, v, __ATOMIC_SEQ_CST); }
template <typename T> inline T atomicAnd(T* p, T v) { return __atomic_fetch_and(p, v, __ATOMIC_SEQ_CST); }
template <typename T> inline T atomicExch(T* p, T v) { return __atomic_exchange_n(p, v, __ATOMIC_SEQ_CST); }
template <typename T> inline T atomicCAS(T* p, T cmp, T v) {
  __atomic_compare_exchange_n(p, &cmp, v, false, __ATOMIC_SEQ_CST, __ATOMIC_SEQ_CST); return cmp;
}
template <typename T> inline T atomicMin(T* p, T v) {
  T old = __atomic_load_n(p, __ATOMIC_SEQ_CST);
  while (v < old && !__atomic_compare_exchange_n(p, &old, v, false, __ATOMIC_SEQ_CST, __ATOMIC_SEQ_CST)) {}
  return old;
}
template <typename T> inline T atomicMax(T* p, T v) {
  T old = __atomic_load_n(p, __ATOMIC_SEQ_CST);
  while (v > old && !__atomic_compare_exchange_n(p, &old, v, false, __ATOMIC_SEQ_CST, __ATOMIC_SEQ_CST)) {}
  return old;
}
using std::min;
using std::max;

// ---- a sliver of the CUDA runtime, enough for the host side of csrc/ ----
typedef int cudaError_t;
typedef void* cudaStream_t;
typedef void* cudaEvent_t;
enum { cudaSuccess = 0 };
enum cudaMemcpyKind { cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice, cudaMemcpyDefault };
inline const char* cudaGetErrorString(cudaError_t) { return "emul"; }
inline cudaError_t cudaGetLastError() { return 0; }
inline cudaError_t cudaPeekAtLastError() { return 0; }
inline cudaError_t cudaSetDevice(int) { return 0; }
inline cudaError_t cudaGetDevice(int* d) { *d = 0; return 0; }
inline cudaError_t cudaGetDeviceCount(int* n) { *n = 1; return 0; }
inline cudaError_t cudaMalloc(void** p, size_t n) { *p = calloc(1, n ? n : 1); return *p ? 0 : 2; }
inline cudaError_t cudaFree(void* p) { free(p); return 0; }
inline cudaError_t cudaMallocHost(void** p, size_t n) { *p = calloc(1, n ? n : 1); return *p ? 0 : 2; }
inline cudaError_t cudaFreeHost(void* p) { free(p); return 0; }
inline cudaError_t cudaMemcpyAsync(void* d, const void* s, size_t n, cudaMemcpyKind, cudaStream_t) { memmove(d, s, n); return 0; }
inline cudaError_t cudaMemcpy(void* d, const void* s, size_t n, cudaMemcpyKind) { memmove(d, s, n); return 0; }
inline cudaError_t cudaMemsetAsync(void* d, int v, size_t n, cudaStream_t) { memset(d, v, n); return 0; }
inline cudaError_t cudaStreamSynchronize(cudaStream_t) { return 0; }
inline cudaError_t cudaDeviceSynchronize() { return 0; }
inline cudaError_t cudaEventCreateWithFlags(cudaEvent_t* e, unsigned) { *e = nullptr; return 0; }
inline cudaError_t cudaEventCreate(cudaEvent_t* e) { *e = nullptr; return 0; }
inline cudaError_t cudaEventDestroy(cudaEvent_t) { return 0; }
inline cudaError_t cudaEventRecord(cudaEvent_t, cudaStream_t) { return 0; }
inline cudaError_t cudaEventSynchronize(cudaEvent_t) { return 0; }
inline cudaError_t cudaEventElapsedTime(float* ms, cudaEvent_t, cudaEvent_t) { *ms = 0.f; return 0; }
enum { cudaEventDisableTiming = 2 };
struct cudaDeviceProp { int multiProcessorCount; size_t sharedMemPerBlockOptin; int major, minor; char name[64]; };
inline cudaError_t cudaGetDeviceProperties(cudaDeviceProp* p, int) {
  memset(p, 0, sizeof(*p)); p->multiProcessorCount = 2; p->sharedMemPerBlockOptin = 227 * 1024; p->major = 10; strcpy(p->name, "simt-emul"); return 0;
}
enum cudaFuncAttribute { cudaFuncAttributeMaxDynamicSharedMemorySize };
template <typename F> inline cudaError_t cudaFuncSetAttribute(F, cudaFuncAttribute, int) { return 0; }

#define FFB_LAUNCH(kern, grid, block, smem, stream, ...) \
  simt::launch(dim3(grid), dim3(block), (size_t)(smem), [&]() { kern(__VA_ARGS__); })
#define FFB_DYN_SMEM(name) unsigned char* name = simt::dyn_smem
