// Context lifetime, scratch management and error reporting for libffb.
#include "ffb_common.cuh"

#include <stdarg.h>
#include <stdio.h>

int32_t ffb_fail(FfbContext* ctx, int32_t code, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return code;
}

int32_t ffb_reserve(FfbContext* ctx, FfbBuf* b, size_t bytes) {
  if (bytes <= b->cap) return FFB_OK;
  // growth frees the old block; callers only grow between dependent launches on one stream,
  // so drain the device first (rare: sizes settle after the first call of a given shape)
  if (b->p) {
    FFB_CUDA(ctx, cudaDeviceSynchronize());
    FFB_CUDA(ctx, cudaFree(b->p));
    b->p = nullptr;
    b->cap = 0;
  }
  size_t want = bytes + bytes / 4 + 4096;
  FFB_CUDA(ctx, cudaMalloc(&b->p, want));
  b->cap = want;
  return FFB_OK;
}

int32_t ffb_stage_reserve(FfbContext* ctx, size_t bytes) {
  if (ctx->stage_busy) {
    FFB_CUDA(ctx, cudaEventSynchronize(ctx->stage_free));
    ctx->stage_busy = false;
  }
  if (bytes > ctx->h_stage_cap) {
    if (ctx->h_stage) FFB_CUDA(ctx, cudaFreeHost(ctx->h_stage));
    ctx->h_stage = nullptr;
    size_t want = bytes + bytes / 2 + 4096;
    FFB_CUDA(ctx, cudaMallocHost(&ctx->h_stage, want));
    ctx->h_stage_cap = want;
  }
  return FFB_OK;
}

int32_t ffb_check_launch(FfbContext* ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ffb_fail(ctx, FFB_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  ctx->launches += 1;
  return FFB_OK;
}

extern "C" {

int32_t ffb_abi_version(void) { return FFB_ABI_VERSION; }

int32_t ffb_create(int32_t device, FfbContext** out) {
  if (!out) return FFB_E_BAD_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0 || device < 0 || device >= n) return FFB_E_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return FFB_E_CUDA;
  FfbContext* ctx = new FfbContext();
  ctx->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) {
    ctx->sm_count = prop.multiProcessorCount;
    ctx->smem_optin = prop.sharedMemPerBlockOptin;
  }
  if (cudaEventCreateWithFlags(&ctx->stage_free, cudaEventDisableTiming) != cudaSuccess) {
    delete ctx;
    return FFB_E_CUDA;
  }
  *out = ctx;
  return FFB_OK;
}

int32_t ffb_destroy(FfbContext* ctx) {
  if (!ctx) return FFB_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  FfbBuf* bufs[] = {&ctx->d_tables, &ctx->d_kstab, &ctx->d_sky, &ctx->d_lex, &ctx->d_flow, &ctx->d_explore, &ctx->d_bigfront};
  for (FfbBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->stage_free) cudaEventDestroy(ctx->stage_free);
  delete ctx;
  return FFB_OK;
}

const char* ffb_last_error(const FfbContext* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int64_t ffb_launch_count(const FfbContext* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
