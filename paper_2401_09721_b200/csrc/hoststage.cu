// Host->device copies of PAGEABLE arrays (what load_ply / add_gaussian_noise
// hand to denoise): the driver copies pageable memory through a small bounce
// buffer on the calling thread (~15 GB/s here).  Instead, a per-context pool
// of host threads copies 2 MB chunks into pinned staging in parallel, and the
// calling thread issues each chunk's DMA as soon as it has landed, so the
// memcpy, the PCIe transfer and the other chunks overlap.
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "fgbd_internal.cuh"

namespace fgbd {

constexpr size_t kStageChunk = 2u << 20;

struct HostStager {
  std::vector<std::thread> threads;
  std::mutex m;
  std::condition_variable cv;
  bool quit = false;
  unsigned long long job = 0;  // generation of the current job
  // current job
  const char* src = nullptr;
  char* dst = nullptr;
  size_t bytes = 0, chunk = 0;
  int nchunks = 0;
  std::atomic<int> next{0};
  std::vector<std::atomic<int>> done;  // per chunk: 1 when staged
  // pinned staging, two regions (coordinates, colours)
  char* pinned[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};

  explicit HostStager(int n) : done(kMaxChunks) {
    for (int t = 0; t < n; ++t) threads.emplace_back([this] { loop(); });
  }
  ~HostStager() {
    {
      std::lock_guard<std::mutex> lk(m);
      quit = true;
    }
    cv.notify_all();
    for (auto& t : threads) t.join();
    for (auto* p : pinned)
      if (p) cudaFreeHost(p);
  }
  static constexpr int kMaxChunks = 4096;

  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return quit || job != seen; });
        if (quit) return;
        seen = job;
      }
      for (int k; (k = next.fetch_add(1)) < nchunks;) {
        const size_t off = (size_t)k * chunk;
        std::memcpy(dst + off, src + off, std::min(chunk, bytes - off));
        done[k].store(1, std::memory_order_release);
      }
    }
  }
};

void destroy_stager(fgbd_ctx* ctx) {
  delete ctx->stager;
  ctx->stager = nullptr;
}

static bool is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Start staging `bytes` of src into pinned region `region` on the pool
// (the calling thread joins in through stage_step).
static char* stage_begin(fgbd_ctx* ctx, const void* src, size_t bytes, int region, int* nchunks) {
  HostStager& h = *ctx->stager;
  if (h.cap[region] < bytes) {
    // a previous frame's DMA from this region has completed: every frame
    // synchronises its streams before returning
    if (h.pinned[region]) cudaFreeHost(h.pinned[region]);
    h.pinned[region] = nullptr;
    h.cap[region] = 0;
    if (cudaMallocHost(&h.pinned[region], bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    h.cap[region] = bytes;
  }
  *nchunks = (int)((bytes + kStageChunk - 1) / kStageChunk);
  char* stage = h.pinned[region];
  {
    std::lock_guard<std::mutex> lk(h.m);
    h.src = static_cast<const char*>(src);
    h.dst = stage;
    h.bytes = bytes;
    h.chunk = kStageChunk;
    h.nchunks = *nchunks;
    for (int k = 0; k < *nchunks; ++k) h.done[k].store(0, std::memory_order_relaxed);
    h.next.store(0);
    ++h.job;
  }
  h.cv.notify_all();
  return stage;
}

// the calling thread copies one more chunk, if any is left; false when none
static bool stage_step(HostStager& h) {
  const int k = h.next.fetch_add(1);
  if (k >= h.nchunks) return false;
  const size_t off = (size_t)k * h.chunk;
  std::memcpy(h.dst + off, h.src + off, std::min(h.chunk, h.bytes - off));
  h.done[k].store(1, std::memory_order_release);
  return true;
}

static bool stage_wanted(fgbd_ctx* ctx, const void* src, size_t bytes) {
  if (ctx->host_threads <= 0 || bytes < 2 * kStageChunk ||
      (bytes + kStageChunk - 1) / kStageChunk > (size_t)HostStager::kMaxChunks || !is_pageable(src))
    return false;
  if (!ctx->stager) ctx->stager = new HostStager(ctx->host_threads);
  return true;
}

int host_to_device(fgbd_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s,
                   int region) {
  if (bytes == 0) return FGBD_OK;
  int nchunks = 0;
  char* stage = stage_wanted(ctx, src, bytes) ? stage_begin(ctx, src, bytes, region, &nchunks)
                                              : nullptr;
  if (!stage) {
    FGBD_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return FGBD_OK;
  }
  HostStager& h = *ctx->stager;
  // copy along, and issue each chunk's DMA in order as soon as it has landed
  int issued = 0;
  while (issued < nchunks) {
    const bool worked = stage_step(h);
    while (issued < nchunks && h.done[issued].load(std::memory_order_acquire)) {
      const size_t off = (size_t)issued * kStageChunk;
      FGBD_CUDA(ctx, cudaMemcpyAsync(static_cast<char*>(dst) + off, stage + off,
                                     std::min(kStageChunk, bytes - off), cudaMemcpyHostToDevice, s));
      ++issued;
    }
    if (!worked && issued < nchunks) std::this_thread::yield();
  }
  return FGBD_OK;
}

bool host_stageable(fgbd_ctx* ctx, const void* src, size_t bytes) {
  return bytes && stage_wanted(ctx, src, bytes);
}

}  // namespace fgbd
