// Shared infrastructure for libmgrgpu: context, errors, device buffers, CSR.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <array>
#include <deque>
#include <exception>
#include <functional>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>
#include <string>
#include <unordered_map>
#include <vector>
#include <stdexcept>
#include <cstring>
#include "../../include/mgrgpu.h"

namespace mg {

struct MgError {
  int code;
  std::string msg;
  int64_t row;
  MgError(int c, std::string m, int64_t r = -1) : code(c), msg(std::move(m)), row(r) {}
};

#define MG_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess)                                                               \
      throw ::mg::MgError(MG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

struct Ctx;
extern thread_local Ctx *g_ctx;  // context of the current API call

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t err_row = -1;
  int64_t launches = 0;
  int64_t syncs = 0;      // host round trips (setup latency diagnostics)
  int64_t dev_bytes = 0;
  int num_sms = 148;
  int profiling = 0;
  mg_timing timing{};
  // scratch
  double *red = nullptr;        // reduction partials (device)
  size_t red_cap = 0;
  double *hbuf = nullptr;       // pinned host scratch
  size_t hbuf_cap = 0;
  void *cub_tmp = nullptr;
  size_t cub_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // mg_timer_start / mg_timer_stop
  cudaStream_t copy_stream = nullptr;         // mg_mat_upload_bsr_async (created on first use)
  // the executable graph of the last freed MGR hierarchy, kept so the next
  // hierarchy's apply graph (same topology when the level shapes repeat) is
  // installed with cudaGraphExecUpdate instead of a fresh instantiation
  cudaGraphExec_t parked_exec = nullptr;
  // caching allocator state (common.cu); owned by the API context, shared by
  // its worker contexts under `amu`.  Every block has a home pool (the context
  // that cudaMalloc'ed it: 0 = API context, k = worker k) and returns there
  // when freed, so each context's pool converges to its own steady-state
  // needs.  A free block also remembers the stream that freed it (nullptr =
  // safe everywhere) and, for the parent stream, the fork epoch of the free:
  // a worker may reuse a parent-freed block only if it was freed before the
  // worker's fork (the worker's stream waits for that work); blocks freed by a
  // worker are neutral only after the join.
  struct FreeBlk { void *p; cudaStream_t freer; int64_t epoch; };
  struct BlkInfo { size_t size; int home; };
  std::vector<std::multimap<size_t, FreeBlk>> pools{1};
  std::unordered_map<void *, BlkInfo> block_size;
  size_t cached_bytes = 0;
  // slabs: pool misses up to SLAB/4 bytes are carved from 256 MB slabs
  // (bump pointer) instead of separate cudaMalloc calls; carved blocks are
  // pooled like any other and released with their slab at context teardown
  std::vector<char *> slabs;
  char *slab_cur = nullptr;
  size_t slab_left = 0;
  int pool_id = 0;          // this context's home pool
  int64_t epoch = 0;        // parent: number of forks so far
  int64_t fork_epoch = 0;   // worker: parent epoch at its fork
  std::mutex amu;
  // worker contexts (own stream + scratch) for concurrent setup tasks
  Ctx *owner = nullptr;      // worker: the root (API) context
  bool busy = false;         // worker: taken by an open task (root's amu)
  int open_groups = 0;       // TaskGroups open with this context as parent
  std::vector<std::unique_ptr<Ctx>> workers;  // root only
  std::map<std::array<int, 3>, Ctx *> worker_of;  // root: (parent pool, group slot, task) -> worker
  ~Ctx();
};

// Concurrent setup tasks: each task runs on its own host thread with a worker
// context (own stream, waits for the parent's work enqueued so far).  join()
// waits for all of them, makes the parent stream ordered after them and
// rethrows the first task error.
class TaskGroup {
 public:
  TaskGroup();
  ~TaskGroup();
  void run(std::function<void()> fn);
  void join();
  // join without throwing; the error of each task (nullptr if none), in run order
  std::vector<std::exception_ptr> join_errors();
 private:
  Ctx *parent_;
  int slot_ = 0;  // ordinal among the groups open on parent_ at construction
  std::vector<std::thread> th_;
  std::vector<Ctx *> used_;
  std::deque<std::exception_ptr> err_;  // stable element addresses: tasks write their slot
  bool joined_ = true;
};

void alloc_release_cache(Ctx *c);
void alloc_release_slabs(Ctx *c);
bool alloc_in_slab(const Ctx *c, const void *p);

inline cudaStream_t stream() { return g_ctx->stream; }

// ---- programmatic dependent launch (PDL) -------------------------------------------
// Solve-phase kernels are launched with programmatic stream serialisation: the
// next kernel's launch (and CTA scheduling) overlaps this kernel's tail instead
// of waiting for the grid to drain.  Every kernel launched this way calls
// pdl_wait() before its first global memory access (it returns once every
// predecessor grid has completed and its writes are visible), and
// pdl_trigger() right after, so that its own successor may start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Device-side checks of the checked build (libmgrgpu_checked.so, -DMG_BOUNDS_CHECK):
// a failed check prints its site and traps, so the launch fails with
// cudaErrorLaunchFailure and the C-ABI returns MG_ERR_CUDA.  Compiled out of
// libmgrgpu.so.  Stand-in for compute-sanitizer, which is closed on the GPU pool.
#ifdef MG_BOUNDS_CHECK
#define MG_DCHECK(cond)                                                                         \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("MG_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define MG_DCHECK(cond) \
  do {                  \
  } while (0)
#endif
#define PDL_ENTRY() \
  do {              \
    pdl_wait();     \
    pdl_trigger();  \
  } while (0)
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw MgError(MG_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}
inline void count_launch(int n = 1) { g_ctx->launches += n; }
inline void check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw MgError(MG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  g_ctx->launches++;
}

void *dmalloc(size_t bytes);
void dfree(void *p, size_t bytes);
void *cub_scratch(size_t bytes);
double *red_scratch(size_t n);
double *host_scratch(size_t n);
void sync();

// RAII device buffer (stream-ordered allocation on the context stream)
template <typename T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t n_) { alloc(n_); }
  void alloc(size_t n_) {
    release();
    n = n_;
    p = n ? (T *)dmalloc(n * sizeof(T)) : nullptr;
  }
  void release() {
    if (p) dfree(p, n * sizeof(T));
    p = nullptr;
    n = 0;
  }
  T *detach() { T *q = p; p = nullptr; n = 0; return q; }
  ~DBuf() { if (p && g_ctx) release(); }
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  T *get() const { return p; }
};

// SpMV launch plan of a matrix: a SELL-32 copy (scalar CSR) or block SELL-32
// copy (BCSR) built once at setup when it pays (spmv.cu prepare_spmv).
struct SpmvPlan {
  // SELL-32 copy (slices of 32 consecutive rows, column-major inside a slice):
  // one thread per row, coalesced value/column loads and x gathers that
  // coalesce across neighbouring stencil rows (padding caps in build_sell).
  bool sell = false;
  DBuf<int> sptr;            // slice start (elements), nslices + 1
  DBuf<int> rlen;            // row lengths, by slice position
  DBuf<int> perm;            // slice position -> row (SELL-C-sigma), empty = identity
  DBuf<int> sci;             // int32 columns (ik == 0)
  DBuf<double> sv;
  // lossless column compression (spmv.cu build_codes): col = anchor(row) + code,
  // anchor(row) = (row * mul) >> 32.  ik 1: u8 codes into `dict` (<= 256 distinct
  // codes), ik 2: int16 codes; packed 4 (2) per 32-bit word, word (k / 4, lane)
  // of a slice.  Same entries in the same order: results bit-identical.
  int ik = 0;
  unsigned long long mul = 0;
  DBuf<unsigned> scode;
  DBuf<int> dict;
  int idx_bytes() const { return ik == 1 ? 1 : ik == 2 ? 2 : 4; }
};

// Device CSR; b > 1 means block CSR with b*b row-major values per entry.
struct Csr {
  int nr = 0, nc = 0, b = 1;
  int64_t nnz = 0;
  DBuf<int> rp, ci;
  DBuf<double> v;
  mutable std::unique_ptr<SpmvPlan> plan;
  Csr() = default;
  Csr(Csr &&) = default;
  Csr &operator=(Csr &&) = default;
  void alloc(int nr_, int nc_, int64_t nnz_, int b_ = 1) {
    plan.reset();
    nr = nr_; nc = nc_; nnz = nnz_; b = b_;
    rp.alloc((size_t)nr + 1);
    ci.alloc((size_t)nnz);
    v.alloc((size_t)nnz * b * b);
  }
  // algorithmic bytes of y = A x in the stored format: int32
  // columns, or 1 / 2 B per entry when the SpMV plan holds compressed columns
  double bytes_spmv() const {
    const double ib = plan ? plan->idx_bytes() : 4.0;
    double vb = (double)nnz * (8.0 * b * b + ib) + 4.0 * (nr + 1) + (plan && plan->perm.p ? 4.0 * nr : 0.0);
    return vb + 8.0 * b * nc + 8.0 * b * nr;
  }
};

inline int grid_for(int64_t work, int block, int max_blocks = 0) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (max_blocks && g > max_blocks) g = max_blocks;
  if (g > 2147483647LL) g = 2147483647LL;
  return (int)g;
}

// MG_TRACE=1: synchronise and print the wall time since the previous mark
void trace(const char *what);
bool trace_on();
void timeline_reset();
void timeline_dump();

// host <-> device helpers (synchronous on the ctx stream)
void h2d(void *dst, const void *src, size_t bytes);
void d2h(void *dst, const void *src, size_t bytes);
void dzero(void *dst, size_t bytes);
// set up to 8 device ints from kernel parameters (stream-ordered, no host sync)
void dset_i32(int *dst, std::initializer_list<int> vals);
void d2d(void *dst, const void *src, size_t bytes);

// scans / reductions (CUB)
// out[0]=0, out[i+1] = sum in[0..i]; returns total (host)
int64_t exclusive_scan_i32_to_i32(const int *in, int *out, int n);
int64_t exclusive_scan_i32_to_i64(const int *in, int64_t *out, int n);
int64_t reduce_sum_i32(const int *in, int n);
int64_t count_u8(const uint8_t *in, int n);

// Row groups for the setup kernels that walk one CSR row per group: VS lanes
// (a power of two <= 32) per row, so short rows do not leave most of a warp
// idle on a chain of dependent loads.  Warp primitives take the group's lane
// mask; bits / sources are group-relative.
template <int VS>
struct RowGroup {
  int64_t row;
  int lane, base;
  unsigned mask;
  __device__ __forceinline__ RowGroup() {
    row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / VS;
    lane = threadIdx.x & (VS - 1);
    base = (threadIdx.x & 31) & ~(VS - 1);
    mask = VS == 32 ? 0xffffffffu : (((1u << (VS & 31)) - 1u) << base);
  }
  // grid-stride: the launch is capped at a few blocks per SM (block launch
  // overhead, not memory, bounds a grid of one tiny block per 8-32 rows)
  __device__ __forceinline__ void next() { row += ((int64_t)gridDim.x * blockDim.x) / VS; }
  __device__ __forceinline__ unsigned ballot(bool p) const { return __ballot_sync(mask, p) >> base; }
  __device__ __forceinline__ bool any(bool p) const { return ballot(p) != 0; }
  template <class T>
  __device__ __forceinline__ T sum(T v) const {
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, VS);
    return v;
  }
  __device__ __forceinline__ double max(double v) const {
#pragma unroll
    for (int o = VS / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(mask, v, o, VS));
    return v;
  }
  template <class T>
  __device__ __forceinline__ T bcast(T v, int src) const { return __shfl_sync(mask, v, src, VS); }
  // lanes below this one among the set bits of a group ballot
  __device__ __forceinline__ int rank(unsigned bits) const { return __popc(bits & ((1u << lane) - 1u)); }
};

// lanes per row from the average row length
inline int row_group_lanes(int64_t nnz, int64_t rows) {
  double avg = rows ? (double)nnz / (double)rows : 0.0;
  return avg <= 4.0 ? 4 : avg <= 8.0 ? 8 : avg <= 16.0 ? 16 : 32;
}

inline int rowgroup_grid(int64_t threads) { return grid_for(threads, 256, g_ctx->num_sms * 8); }

// launch KERNEL<VS> over `rows` rows with VS = row_group_lanes(nnz, rows)
#define MG_ROWGROUP_LAUNCH(KERNEL, rows, nnz, ...)                                                   \
  do {                                                                                              \
    int64_t rg_rows_ = (rows);                                                                      \
    switch (::mg::row_group_lanes((nnz), rg_rows_)) {                                               \
      case 4: KERNEL<4><<<::mg::rowgroup_grid(rg_rows_ * 4), 256, 0, ::mg::stream()>>>(__VA_ARGS__); break;   \
      case 8: KERNEL<8><<<::mg::rowgroup_grid(rg_rows_ * 8), 256, 0, ::mg::stream()>>>(__VA_ARGS__); break;   \
      case 16: KERNEL<16><<<::mg::rowgroup_grid(rg_rows_ * 16), 256, 0, ::mg::stream()>>>(__VA_ARGS__); break; \
      default: KERNEL<32><<<::mg::rowgroup_grid(rg_rows_ * 32), 256, 0, ::mg::stream()>>>(__VA_ARGS__); break; \
    }                                                                                               \
  } while (0)

}  // namespace mg
