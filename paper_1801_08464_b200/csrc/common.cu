// Context-level helpers: stream-ordered allocation, copies, CUB scans.
#include "common.cuh"
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>

namespace mg {

thread_local Ctx *g_ctx = nullptr;

// Caching allocator: best-fit free list of cudaMalloc blocks, never returned
// to the driver until the context is destroyed (or an allocation fails).  All
// work is ordered on the context's single stream, so a freed block can be
// reused by the next allocation immediately.  This keeps setup / solve times
// free of driver allocation stalls (the stream-ordered pool showed 2-3x
// step-to-step variance from physical-memory remapping).
static size_t round_size(size_t b) {
  if (b <= ((size_t)1 << 20)) return (b + 511) & ~(size_t)511;
  return (b + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);
}

void alloc_release_cache(Ctx *c) {
  cudaStreamSynchronize(c->stream);
  for (auto &kv : c->free_blocks) cudaFree(kv.second);
  c->cached_bytes = 0;
  c->free_blocks.clear();
}

void *dmalloc(size_t bytes) {
  if (!bytes) return nullptr;
  Ctx *c = g_ctx;
  size_t rb = round_size(bytes);
  auto it = c->free_blocks.lower_bound(rb);
  if (it != c->free_blocks.end() && it->first <= rb * 2 + ((size_t)4 << 20)) {
    void *p = it->second;
    size_t sz = it->first;
    c->free_blocks.erase(it);
    c->cached_bytes -= sz;
    c->block_size[p] = sz;
    c->dev_bytes += (int64_t)sz;
    return p;
  }
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, rb);
  if (e != cudaSuccess) {
    cudaGetLastError();
    alloc_release_cache(c);
    e = cudaMalloc(&p, rb);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw MgError(MG_ERR_CUDA, std::string("device allocation of ") + std::to_string(bytes) +
                                   " bytes failed: " + cudaGetErrorString(e));
  }
  c->block_size[p] = rb;
  c->dev_bytes += (int64_t)rb;
  return p;
}

void dfree(void *p, size_t bytes) {
  (void)bytes;
  if (!p) return;
  Ctx *c = g_ctx;
  auto it = c->block_size.find(p);
  if (it == c->block_size.end()) return;
  size_t sz = it->second;
  c->block_size.erase(it);
  c->dev_bytes -= (int64_t)sz;
  c->free_blocks.emplace(sz, p);
  c->cached_bytes += sz;
}

void sync() { MG_CUDA(cudaStreamSynchronize(g_ctx->stream)); }

void trace(const char *what) {
  static int on = -1;
  static std::chrono::steady_clock::time_point last;
  if (on < 0) {
    const char *e = getenv("MG_TRACE");
    on = e && *e && *e != '0';
    last = std::chrono::steady_clock::now();
  }
  if (!on) return;
  sync();
  auto now = std::chrono::steady_clock::now();
  double ms = std::chrono::duration<double, std::milli>(now - last).count();
  fprintf(stderr, "[mg] %-40s %9.3f ms  (dev mem %.2f GiB)\n", what, ms, g_ctx->dev_bytes / 1073741824.0);
  last = std::chrono::steady_clock::now();
}

void h2d(void *dst, const void *src, size_t bytes) {
  if (!bytes) return;
  MG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g_ctx->stream));
  sync();
}
void d2h(void *dst, const void *src, size_t bytes) {
  if (!bytes) return;
  MG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g_ctx->stream));
  sync();
}
void dzero(void *dst, size_t bytes) {
  if (!bytes) return;
  MG_CUDA(cudaMemsetAsync(dst, 0, bytes, g_ctx->stream));
}
void d2d(void *dst, const void *src, size_t bytes) {
  if (!bytes) return;
  MG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, g_ctx->stream));
}

void *cub_scratch(size_t bytes) {
  Ctx *c = g_ctx;
  if (bytes > c->cub_cap) {
    if (c->cub_tmp) dfree(c->cub_tmp, c->cub_cap);
    size_t cap = bytes + bytes / 2 + 4096;
    c->cub_tmp = dmalloc(cap);
    c->cub_cap = cap;
  }
  return c->cub_tmp;
}

double *red_scratch(size_t n) {
  Ctx *c = g_ctx;
  if (n > c->red_cap) {
    if (c->red) dfree(c->red, c->red_cap * sizeof(double));
    size_t cap = n + 1024;
    c->red = (double *)dmalloc(cap * sizeof(double));
    c->red_cap = cap;
  }
  return c->red;
}

double *host_scratch(size_t n) {
  Ctx *c = g_ctx;
  if (n > c->hbuf_cap) {
    if (c->hbuf) cudaFreeHost(c->hbuf);
    size_t cap = n + 1024;
    MG_CUDA(cudaMallocHost(&c->hbuf, cap * sizeof(double)));
    c->hbuf_cap = cap;
  }
  return c->hbuf;
}

namespace {
struct SumI64 {
  __host__ __device__ int64_t operator()(int64_t a, int64_t b) const { return a + b; }
};
struct ToI64 {
  __host__ __device__ int64_t operator()(int a) const { return (int64_t)a; }
};
struct U8ToI64 {
  __host__ __device__ int64_t operator()(uint8_t a) const { return (int64_t)(a != 0); }
};
}  // namespace

__global__ void k_narrow(const int64_t *a, int *b, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (int)a[i];
}

int64_t exclusive_scan_i32_to_i32(const int *in, int *out, int n) {
  // out has n+1 entries; scanned in int64 to detect overflow, then narrowed
  DBuf<int64_t> tmp((size_t)n + 1);
  int64_t total = exclusive_scan_i32_to_i64(in, tmp.p, n);
  if (total > 2147483647LL)
    throw MgError(MG_ERR_UNSUPPORTED, "sparse matrix exceeds 2^31-1 stored entries");
  k_narrow<<<grid_for(n + 1, 256), 256, 0, stream()>>>(tmp.p, out, n + 1);
  check_launch("narrow");
  return total;
}

__global__ void k_set_last(int64_t *out, int n, const int64_t *scan_last, const int *in) {
  out[n] = scan_last[0] + (int64_t)in[n - 1];
}

int64_t exclusive_scan_i32_to_i64(const int *in, int64_t *out, int n) {
  if (n == 0) {
    int64_t z = 0;
    h2d(out, &z, sizeof(z));
    return 0;
  }
  cub::TransformInputIterator<int64_t, ToI64, const int *> it(in, ToI64());
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, out, n, stream());
  void *tmp = cub_scratch(bytes);
  MG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, it, out, n, stream()));
  count_launch();
  k_set_last<<<1, 1, 0, stream()>>>(out, n, out + (n - 1), in);
  check_launch("scan_last");
  int64_t total = 0;
  d2h(&total, out + n, sizeof(total));
  return total;
}

int64_t reduce_sum_i32(const int *in, int n) {
  if (n == 0) return 0;
  cub::TransformInputIterator<int64_t, ToI64, const int *> it(in, ToI64());
  DBuf<int64_t> o(1);
  size_t bytes = 0;
  cub::DeviceReduce::Sum(nullptr, bytes, it, o.p, n, stream());
  void *tmp = cub_scratch(bytes);
  MG_CUDA(cub::DeviceReduce::Sum(tmp, bytes, it, o.p, n, stream()));
  count_launch();
  int64_t t = 0;
  d2h(&t, o.p, sizeof(t));
  return t;
}

int64_t count_u8(const uint8_t *in, int n) {
  if (n == 0) return 0;
  cub::TransformInputIterator<int64_t, U8ToI64, const uint8_t *> it(in, U8ToI64());
  DBuf<int64_t> o(1);
  size_t bytes = 0;
  cub::DeviceReduce::Sum(nullptr, bytes, it, o.p, n, stream());
  void *tmp = cub_scratch(bytes);
  MG_CUDA(cub::DeviceReduce::Sum(tmp, bytes, it, o.p, n, stream()));
  count_launch();
  int64_t t = 0;
  d2h(&t, o.p, sizeof(t));
  return t;
}

}  // namespace mg
