// TEST-ONLY: runtime of the SIMT emulation shim (see simt_emul.h).
#include "simt_emul.h"

#include <thread>
#include <mutex>
#include <condition_variable>

namespace simt {
thread_local uint3_ t_threadIdx, t_blockIdx;
thread_local dim3 t_blockDim, t_gridDim;
thread_local WarpBox* t_warp = nullptr;
thread_local Cta* t_cta = nullptr;
unsigned char* dyn_smem = nullptr;

namespace {
struct Pool {
  std::vector<std::thread> threads;
  std::mutex mu;
  std::condition_variable cv_go, cv_done;
  unsigned long long epoch = 0;
  unsigned active = 0, remaining = 0;
  bool quit = false;
  // current CTA
  const std::function<void()>* body = nullptr;
  Cta* cta = nullptr;
  dim3 grid, block;
  uint3_ bidx{0, 0, 0};

  void worker(unsigned tid) {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_go.wait(lk, [&] { return quit || (epoch != seen && tid < active); });
        if (quit) return;
        seen = epoch;
      }
      t_blockDim = block; t_gridDim = grid; t_blockIdx = bidx;
      t_threadIdx.x = tid % block.x;
      t_threadIdx.y = (tid / block.x) % block.y;
      t_threadIdx.z = tid / (block.x * block.y);
      t_cta = cta;
      t_warp = cta->warps[tid / 32];
      (*body)();
      {
        std::unique_lock<std::mutex> lk(mu);
        if (--remaining == 0) cv_done.notify_all();
      }
    }
  }
  void ensure(unsigned n) {
    while (threads.size() < n) {
      unsigned tid = (unsigned)threads.size();
      threads.emplace_back([this, tid] { worker(tid); });
    }
  }
  ~Pool() {
    { std::unique_lock<std::mutex> lk(mu); quit = true; }
    cv_go.notify_all();
    for (auto& t : threads) t.join();
  }
};
Pool& pool() { static Pool p; return p; }
std::mutex g_launch_mu;
}  // namespace

void launch(dim3 grid, dim3 block, size_t smem, const std::function<void()>& body) {
  std::lock_guard<std::mutex> guard(g_launch_mu);
  unsigned nthreads = block.x * block.y * block.z;
  if (nthreads == 0 || nthreads > 1024) { fprintf(stderr, "simt: bad block size %u\n", nthreads); abort(); }
  if (nthreads % 32 != 0) { fprintf(stderr, "simt: block size %u not a warp multiple\n", nthreads); abort(); }
  Pool& p = pool();
  p.ensure(nthreads);
  std::vector<unsigned char> smem_buf(smem + 16);
  dyn_smem = (unsigned char*)(((uintptr_t)smem_buf.data() + 15) & ~(uintptr_t)15);
  Cta cta;
  cta.nthreads = nthreads;
  pthread_barrier_init(&cta.bar, nullptr, nthreads);
  for (unsigned w = 0; w < nthreads / 32; ++w) {
    WarpBox* wb = new WarpBox();
    pthread_barrier_init(&wb->bar, nullptr, 32);
    cta.warps.push_back(wb);
  }
  for (unsigned bz = 0; bz < grid.z; ++bz)
    for (unsigned by = 0; by < grid.y; ++by)
      for (unsigned bx = 0; bx < grid.x; ++bx) {
        {
          std::unique_lock<std::mutex> lk(p.mu);
          p.body = &body; p.cta = &cta; p.grid = grid; p.block = block;
          p.bidx = uint3_{bx, by, bz};
          p.active = nthreads; p.remaining = nthreads;
          ++p.epoch;
        }
        p.cv_go.notify_all();
        {
          std::unique_lock<std::mutex> lk(p.mu);
          p.cv_done.wait(lk, [&] { return p.remaining == 0; });
          p.active = 0;
        }
      }
  for (auto* wb : cta.warps) { pthread_barrier_destroy(&wb->bar); delete wb; }
  pthread_barrier_destroy(&cta.bar);
  dyn_smem = nullptr;
}
}  // namespace simt
