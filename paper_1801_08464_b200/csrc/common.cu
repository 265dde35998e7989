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

static Ctx *alloc_owner() { return g_ctx->owner ? g_ctx->owner : g_ctx; }

static const size_t SLAB = (size_t)256 << 20;

bool alloc_in_slab(const Ctx *c, const void *p) {
  for (char *s : c->slabs)
    if ((const char *)p >= s && (const char *)p < s + SLAB) return true;
  return false;
}

void alloc_release_cache(Ctx *c) {
  // caller holds c->amu (or no worker is running); slab-carved blocks stay pooled
  cudaDeviceSynchronize();
  for (auto &pool : c->pools)
    for (auto it = pool.begin(); it != pool.end();) {
      if (alloc_in_slab(c, it->second.p)) { ++it; continue; }
      cudaFree(it->second.p);
      c->cached_bytes -= it->first;
      it = pool.erase(it);
    }
}

void alloc_release_slabs(Ctx *c) {
  for (char *s : c->slabs) cudaFree(s);
  c->slabs.clear();
  c->slab_cur = nullptr;
  c->slab_left = 0;
}

// MG_POOL=off (sanitizer runs): every buffer is its own exact-size cudaMalloc and
// is cudaFree'd on release, so memcheck sees accesses past a buffer's end that
// the caching allocator's rounded blocks and slabs would absorb
static bool pool_off() {
  static const bool off = [] {
    const char *e = getenv("MG_POOL");
    return e && std::string(e) == "off";
  }();
  return off;
}

void *dmalloc(size_t bytes) {
  if (!bytes) return nullptr;
  Ctx *c = alloc_owner();
  Ctx *me = g_ctx;
  cudaStream_t s = me->stream;
  std::lock_guard<std::mutex> lk(c->amu);
  if (pool_off()) {
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw MgError(MG_ERR_CUDA, std::string("device allocation of ") + std::to_string(bytes) +
                                     " bytes failed: " + cudaGetErrorString(e));
    }
    c->block_size[p] = Ctx::BlkInfo{bytes, me->pool_id};
    c->dev_bytes += (int64_t)bytes;
    return p;
  }
  size_t rb = round_size(bytes);
  const size_t limit = rb * 2 + ((size_t)4 << 20);
  const bool worker = me->owner != nullptr;
  if ((size_t)me->pool_id >= c->pools.size()) c->pools.resize(me->pool_id + 1);
  auto &pool = c->pools[me->pool_id];
  for (auto it = pool.lower_bound(rb); it != pool.end() && it->first <= limit; ++it) {
    const Ctx::FreeBlk &fb = it->second;
    bool ok = !fb.freer || fb.freer == s || (worker && fb.freer == c->stream && fb.epoch <= me->fork_epoch);
    if (!ok) continue;
    void *p = fb.p;
    size_t sz = it->first;
    pool.erase(it);
    c->cached_bytes -= sz;
    c->block_size[p] = Ctx::BlkInfo{sz, me->pool_id};
    c->dev_bytes += (int64_t)sz;
    return p;
  }
  // No block usable as is: take one freed on another stream and order this
  // stream after everything that stream has enqueued so far (its last use of
  // the block included).  A cross-stream wait is far cheaper than cudaMalloc,
  // which can stall for tens of ms behind queued work.
  for (auto it = pool.lower_bound(rb); it != pool.end() && it->first <= limit; ++it) {
    const Ctx::FreeBlk &fb = it->second;
    if (fb.freer && fb.freer != s) {
      cudaEvent_t ev;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) break;
      cudaEventRecord(ev, fb.freer);
      cudaStreamWaitEvent(s, ev, 0);
      cudaEventDestroy(ev);
    }
    void *p = fb.p;
    size_t sz = it->first;
    pool.erase(it);
    c->cached_bytes -= sz;
    c->block_size[p] = Ctx::BlkInfo{sz, me->pool_id};
    c->dev_bytes += (int64_t)sz;
    return p;
  }
  if (rb <= SLAB / 4) {
    if (rb > c->slab_left) {
      char *sl = nullptr;
      if (cudaMalloc(&sl, SLAB) == cudaSuccess) {
        c->slabs.push_back(sl);
        c->slab_cur = sl;
        c->slab_left = SLAB;
      } else {
        cudaGetLastError();
      }
    }
    if (rb <= c->slab_left) {
      void *p = c->slab_cur;
      c->slab_cur += rb;
      c->slab_left -= rb;
      c->block_size[p] = Ctx::BlkInfo{rb, me->pool_id};
      c->dev_bytes += (int64_t)rb;
      return p;
    }
  }
  void *p = nullptr;
  static const bool alloc_log = getenv("MG_ALLOC_LOG") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMalloc(&p, rb);
  if (alloc_log)
    fprintf(stderr, "[mg] cudaMalloc %zu bytes (pool %d): %.3f ms\n", rb, me->pool_id,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
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
  c->block_size[p] = Ctx::BlkInfo{rb, me->pool_id};
  c->dev_bytes += (int64_t)rb;
  return p;
}

void dfree(void *p, size_t bytes) {
  (void)bytes;
  if (!p) return;
  Ctx *c = alloc_owner();
  std::lock_guard<std::mutex> lk(c->amu);
  auto it = c->block_size.find(p);
  if (it == c->block_size.end()) return;
  Ctx::BlkInfo bi = it->second;
  c->block_size.erase(it);
  c->dev_bytes -= (int64_t)bi.size;
  if (pool_off()) {
    cudaFree(p);  // synchronises the device: no stream can still be using it
    return;
  }
  if ((size_t)bi.home >= c->pools.size()) c->pools.resize(bi.home + 1);
  c->pools[bi.home].emplace(bi.size, Ctx::FreeBlk{p, g_ctx->stream, c->epoch});
  c->cached_bytes += bi.size;
}

// after a join (no worker running, their streams idle) every cached block is
// safe on every stream: later workers fork behind the parent's work
static void neutralise_all(Ctx *c) {
  std::lock_guard<std::mutex> lk(c->amu);
  for (auto &pool : c->pools)
    for (auto &kv : pool) kv.second.freer = nullptr;
}

Ctx::~Ctx() {
  if (parked_exec) cudaGraphExecDestroy(parked_exec);
  for (auto &w : workers) {
    if (!w) continue;
    cudaStreamSynchronize(w->stream);
    if (w->hbuf) cudaFreeHost(w->hbuf);
    cudaStreamDestroy(w->stream);
  }
}

TaskGroup::TaskGroup() : parent_(g_ctx) {
  Ctx *root = parent_->owner ? parent_->owner : parent_;
  std::lock_guard<std::mutex> lk(root->amu);
  slot_ = parent_->open_groups++;
}

TaskGroup::~TaskGroup() {
  if (!joined_) {
    try { join(); } catch (...) {}
  }
  Ctx *root = parent_->owner ? parent_->owner : parent_;
  std::lock_guard<std::mutex> lk(root->amu);
  parent_->open_groups--;
}

static bool concurrent_setup() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_CONCURRENT_SETUP");
    on = !(e && *e == '0');
    return on;
  }();
  return on;
}

void TaskGroup::run(std::function<void()> fn) {
  if (!concurrent_setup() || trace_on()) {
    // inline: same error semantics as a worker (recorded, reported at the join)
    std::exception_ptr e = nullptr;
    try {
      fn();
    } catch (...) {
      e = std::current_exception();
    }
    err_.push_back(e);
    return;
  }
  // Workers belong to the root (API) context: groups may nest (a task that
  // starts its own group) and several groups of one root may be open at once
  // (the MGR level tasks and the coarse AMG's).  Task k of the group opened as
  // the slot-th open group of parent context P always runs on the worker keyed
  // (P, slot, k): the same code path gets the same workers every setup, so each
  // worker's home pool settles on its own needs (no pool misses in steady state).
  Ctx *p = parent_;
  Ctx *root = p->owner ? p->owner : p;
  Ctx *w = nullptr;
  {
    std::lock_guard<std::mutex> lk(root->amu);
    const std::array<int, 3> key{p->pool_id, slot_, (int)used_.size()};
    auto it = root->worker_of.find(key);
    if (it != root->worker_of.end()) w = it->second;
    if (!w) {
      auto nw = std::make_unique<Ctx>();
      nw->device = root->device;
      nw->num_sms = root->num_sms;
      nw->owner = root;
      nw->pool_id = (int)root->workers.size() + 1;
      // worker streams at the lowest priority: the parent's stream carries the
      // setup's critical path (MGR RAP, coarse AMG); worker blocks fill the gaps
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      const char *pe = getenv("MG_WORKER_PRIORITY");
      int prio = (pe && *pe == '0') ? 0 : lo;
      MG_CUDA(cudaStreamCreateWithPriority(&nw->stream, cudaStreamNonBlocking, prio));
      w = nw.get();
      root->worker_of[key] = w;
      root->workers.push_back(std::move(nw));
    }
    if (w->busy) throw MgError(MG_ERR_CUDA, "internal: setup worker already running");
    w->busy = true;
    // root-stream frees up to this epoch are ordered before the worker: for a
    // nested fork, those ordered before the parent worker's own fork
    const int64_t e = root->epoch++;
    w->fork_epoch = p == root ? e : p->fork_epoch;
  }
  w->launches = 0;
  w->syncs = 0;
  // the worker's stream starts after everything the parent enqueued so far,
  // so blocks the parent freed before this point are safe on both streams
  cudaEvent_t ev;
  MG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  MG_CUDA(cudaEventRecord(ev, p->stream));
  MG_CUDA(cudaStreamWaitEvent(w->stream, ev, 0));
  cudaEventDestroy(ev);
  used_.push_back(w);
  err_.push_back(nullptr);
  joined_ = false;
  size_t slot = err_.size() - 1;
  int dev = p->device;
  th_.emplace_back([this, w, fn, slot, dev]() {
    cudaSetDevice(dev);
    g_ctx = w;
    try {
      fn();
      sync();
    } catch (...) {
      err_[slot] = std::current_exception();
      cudaStreamSynchronize(w->stream);
    }
    g_ctx = nullptr;
  });
}

void TaskGroup::join() {
  std::vector<std::exception_ptr> errs = join_errors();
  for (auto &e : errs)
    if (e) std::rethrow_exception(e);
}

std::vector<std::exception_ptr> TaskGroup::join_errors() {
  for (auto &t : th_)
    if (t.joinable()) t.join();
  th_.clear();
  joined_ = true;
  Ctx *p = parent_;
  Ctx *root = p->owner ? p->owner : p;
  bool idle = true;
  {
    std::lock_guard<std::mutex> lk(root->amu);
    for (Ctx *w : used_) {
      p->launches += w->launches;
      p->syncs += w->syncs;
      w->busy = false;
    }
    for (auto &c : root->workers) idle &= !c->busy;
  }
  if (!used_.empty() && idle && p == root) {
    // no worker of the root runs any more and their streams are idle (each
    // task synchronises its stream before its thread ends), so everything the
    // root enqueues from here on is ordered after the workers' work.  (With a
    // group still open elsewhere, blocks freed by these workers keep their
    // freeing stream and are reused through a cross-stream wait.)
    neutralise_all(root);
  }
  used_.clear();
  std::vector<std::exception_ptr> errs(err_.begin(), err_.end());
  err_.clear();
  return errs;
}

void sync() {
  g_ctx->syncs++;
  MG_CUDA(cudaStreamSynchronize(g_ctx->stream));
}

bool pdl_enabled() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_PDL");
    on = !(e && *e == '0');
    return on;
  }();
  return on;
}

static bool timeline_on();

bool trace_on() {
  if (timeline_on()) return false;          // timeline mode: no synchronising trace
  if (g_ctx && g_ctx->owner) return false;  // worker threads do not trace
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_TRACE");
    on = e && *e && *e != '0';
    return on;
  }();
  return on;
}

// MG_TIMELINE=1: non-synchronising host timestamps of the trace points of both
// setup threads (parent and F-relaxation worker), dumped at the end of a setup
static std::mutex tl_mu;
static std::vector<std::pair<double, std::string>> tl_events;
static std::chrono::steady_clock::time_point tl_t0;
static bool timeline_on() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_TIMELINE");
    on = e && *e == '1';
    return on;
  }();
  return on;
}
void timeline_reset() {
  if (!timeline_on()) return;
  std::lock_guard<std::mutex> lk(tl_mu);
  tl_events.clear();
  tl_t0 = std::chrono::steady_clock::now();
}
void timeline_dump() {
  if (!timeline_on()) return;
  std::lock_guard<std::mutex> lk(tl_mu);
  for (auto &e : tl_events) fprintf(stderr, "[tl] %8.3f ms  %s\n", e.first, e.second.c_str());
  tl_events.clear();
}

void trace(const char *what) {
  static std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  static int64_t last_syncs = 0, last_launches = 0;
  if (timeline_on() && g_ctx) {
    double t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl_t0).count();
    std::lock_guard<std::mutex> lk(tl_mu);
    tl_events.emplace_back(t, std::string(g_ctx->owner ? "    [worker] " : "") + what);
    return;
  }
  if (!trace_on()) return;
  sync();
  int64_t ds = g_ctx->syncs - last_syncs, dl = g_ctx->launches - last_launches;
  last_syncs = g_ctx->syncs;
  last_launches = g_ctx->launches;
  auto now = std::chrono::steady_clock::now();
  double ms = std::chrono::duration<double, std::milli>(now - last).count();
  fprintf(stderr, "[mg] %-40s %9.3f ms  %4lld syncs %5lld launches (dev mem %.2f GiB)\n", what, ms,
          (long long)ds, (long long)dl, g_ctx->dev_bytes / 1073741824.0);
  last = std::chrono::steady_clock::now();
}

// small transfers are staged through the context's pinned buffer (a pageable
// copy goes through the driver's shared staging path and costs more per call)
static const size_t STAGE_MAX = 64 << 10;
// Host->device copies up to this size are staged in pinned memory and pulled
// by a kernel reading the mapped host buffer: every copy-engine H2D transfer
// (pinned or not, any stream) queues behind a bulk upload in flight (an
// asynchronous matrix upload on the copy stream), a kernel load does not.
static const size_t STAGE_H2D_MAX = 16 << 20;

__global__ void k_pull_host(uint4 *__restrict__ dst, const uint4 *__restrict__ src, int64_t n16, uint8_t *dtail,
                            const uint8_t *stail, int ntail) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  if (blockIdx.x == 0 && (int)threadIdx.x < ntail) dtail[threadIdx.x] = stail[threadIdx.x];
}

void h2d(void *dst, const void *src, size_t bytes) {
  if (!bytes) return;
  if (bytes <= STAGE_H2D_MAX) {
    uint8_t *hs = (uint8_t *)host_scratch((bytes + 7) / 8);
    memcpy(hs, src, bytes);
    if (((uintptr_t)dst & 15) == 0) {
      int64_t n16 = (int64_t)(bytes / 16);
      int ntail = (int)(bytes - (size_t)n16 * 16);
      k_pull_host<<<grid_for(n16 ? n16 : 1, 256, 256), 256, 0, g_ctx->stream>>>(
          (uint4 *)dst, (const uint4 *)hs, n16, (uint8_t *)dst + n16 * 16, hs + n16 * 16, ntail);
      check_launch("pull_host");
    } else {
      MG_CUDA(cudaMemcpyAsync(dst, hs, bytes, cudaMemcpyHostToDevice, g_ctx->stream));
    }
  } else {
    MG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g_ctx->stream));
  }
  sync();
}
void d2h(void *dst, const void *src, size_t bytes) {
  if (!bytes) return;
  if (bytes <= STAGE_MAX) {
    void *hs = host_scratch((bytes + 7) / 8);
    MG_CUDA(cudaMemcpyAsync(hs, src, bytes, cudaMemcpyDeviceToHost, g_ctx->stream));
    sync();
    memcpy(dst, hs, bytes);
    return;
  }
  MG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g_ctx->stream));
  sync();
}

struct I32x8 { int v[8]; };
__global__ void k_set_i32(int *dst, I32x8 vals, int n) {
  if (threadIdx.x < n) dst[threadIdx.x] = vals.v[threadIdx.x];
}
void dset_i32(int *dst, std::initializer_list<int> vals) {
  I32x8 a{};
  int n = 0;
  for (int v : vals) {
    if (n == 8) throw MgError(MG_ERR_BAD_OPTION, "dset_i32: at most 8 values");
    a.v[n++] = v;
  }
  k_set_i32<<<1, 32, 0, g_ctx->stream>>>(dst, a, n);
  check_launch("set_i32");
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
