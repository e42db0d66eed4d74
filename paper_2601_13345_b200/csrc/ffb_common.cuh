// Shared host/device plumbing for libffb (sm_100a).  Not part of the public ABI.
#pragma once

#ifdef FFB_SIMT_EMUL
#include "simt_emul.h"
#else
#include <cuda_runtime.h>
#define FFB_LAUNCH(kern, grid, block, smem, stream, ...) \
  kern<<<(grid), (block), (smem), (cudaStream_t)(stream)>>>(__VA_ARGS__)
#define FFB_DYN_SMEM(name) extern __shared__ __align__(16) unsigned char name[]
#endif

#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/ffb.h"

#define FFB_HD __host__ __device__ __forceinline__
#define FFB_D __device__ __forceinline__

// Python's min/max return the FIRST argument on ties and never reorder NaNs; the reference's
// arithmetic goes through them (features.py:59,114  time_model.py:37,44,78,81,106
// power_model.py:124,157), so the device code uses the same selection rule instead of fmin/fmax.
FFB_HD double py_min(double a, double b) { return (b < a) ? b : a; }
FFB_HD double py_max(double a, double b) { return (b > a) ? b : a; }

struct FfbBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct FfbContext {
  int device = 0;
  int sm_count = 148;
  size_t smem_optin = 0;
  std::string err;
  int64_t launches = 0;
  // growable device scratch, one per purpose so that calls on one stream can chain safely
  FfbBuf d_tables;     // predict: spec / shape / cap / pow tables
  FfbBuf d_kstab;      // predict: per (kernel, spec) hoisted values
  FfbBuf d_sky;        // skyline scratch
  FfbBuf d_lex;        // lexer scratch
  FfbBuf d_flow;       // dataflow scratch
  FfbBuf d_explore;    // fused explore: tie ranks + counter
  FfbBuf d_bigfront;   // sort-based finish of large fronts (ffb_bigfront.cu)
  std::vector<uint16_t> explore_shadow;   // host copy of the tie-order table d_explore holds
  void* explore_shadow_dev = nullptr;
  void* h_stage = nullptr;   // pinned staging for table uploads
  size_t h_stage_cap = 0;
  cudaEvent_t stage_free = nullptr;  // recorded after the last async copy out of h_stage
  bool stage_busy = false;
  // predict: host copy of the tables that d_tables currently holds (identical inputs skip the upload and its wait)
  std::vector<unsigned char> tables_shadow;
  void* tables_shadow_dev = nullptr;
  void* tables_shadow_stream = nullptr;   // the upload is only known to be ordered before work on this stream
};

int32_t ffb_fail(FfbContext* ctx, int32_t code, const char* fmt, ...);
int32_t ffb_reserve(FfbContext* ctx, FfbBuf* b, size_t bytes);
int32_t ffb_stage_reserve(FfbContext* ctx, size_t bytes);   // waits until earlier uploads drained
int32_t ffb_check_launch(FfbContext* ctx, const char* what);
// ffb_bigfront.cu: exact front of a set whose front does not fit one CTA (device-wide sort); synchronises
int32_t ffb_big_front(FfbContext* ctx, const double* d_e, const double* d_t, const uint64_t* d_id, int64_t n, double rho,
                      uint64_t* d_front_id, double* d_front_e, double* d_front_t, int64_t cap_front,
                      int64_t* h_front_n, double* h_tpeak, cudaStream_t stream);

#define FFB_CUDA(ctx, expr)                                                        \
  do {                                                                             \
    cudaError_t e__ = (expr);                                                      \
    if (e__ != cudaSuccess)                                                        \
      return ffb_fail((ctx), FFB_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e__)); \
  } while (0)
