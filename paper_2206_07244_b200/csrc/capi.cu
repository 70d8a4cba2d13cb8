// capi.cu -- host side of the B200-native OpSparse SpGEMM behind the C ABI in
// include/spgemm_capi.h. One TU: the stage machine of SpgemmPipeline
// (pipeline.cpp:109-472) re-designed around CUDA streams/events and
// stream-ordered allocation, driving the sm_100a kernels in kernels.cuh.
//
// Differences by design (B200-first, not a port):
//   * TaskPool/WaitGroup (task_pool.hpp) -> one stream per bin, launched in the
//     plan's launch order (pipeline.cpp:84), joined with events.
//   * MetadataArena (pipeline.cpp:89-102) -> one cudaMallocAsync arena holding
//     int32 bins, per-row-block counts, scan state, spill ids and phase info.
//   * allocate_output on std::async (pipeline.cpp:254-257) -> cudaMallocAsync
//     of C.col/C.val on a side stream while the numeric scatter runs.
//   * StepTimings from CUDA events recorded at the step boundaries.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <limits>
#include <map>
#include <tuple>
#include <mutex>
#include <new>
#include <string>
#include <unordered_set>
#include <vector>

#include "kernels.cuh"
#include "kernels_heap.cuh"
#include "kernels_coo.cuh"
#include "kernels_reuse.cuh"
#include "spgemm_capi.h"

using namespace spgemm_b200;

// ------------------------------------------------------------------ errors
namespace {

thread_local std::string g_err;
// set while multiply_into runs its row blocks: their device operands were
// staged on the context's own stream, so no ordering against the legacy
// default stream is needed (that wait would also order the blocks behind
// unrelated blocking-stream work)
thread_local bool g_inputs_stream_ordered = false;

struct Err {
  spgemm_status s;
  std::string m;
};

[[noreturn]] void fail(spgemm_status s, std::string m) { throw Err{s, std::move(m)}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? SPGEMM_OUT_OF_MEMORY : SPGEMM_CUDA_ERROR,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <class F>
spgemm_status guard(F&& f) {
  try {
    f();
    return SPGEMM_OK;
  } catch (const Err& e) {
    g_err = e.m;
    return e.s;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SPGEMM_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SPGEMM_LOGIC_ERROR;
  }
}

// -------------------------------------------------------------- presets
// binning.cpp:26-66 -- the same published ranges and capacities.
constexpr int64_t kNoUpper = std::numeric_limits<int64_t>::max();
constexpr int64_t kSharedNumMax = 8192;  // largest numeric row on chip (k_num_block<16384, 1024, 8192>)
constexpr int64_t kSymTable[kNumBins] = {32, 512, 1024, 2048, 4096, 8192, 12287, 24575};
constexpr int64_t kNumTable[kNumBins] = {31, 255, 511, 1023, 2047, 4095, 8191, 0};

struct PresetRow {
  const char* name;
  int phase;
  int64_t upper[kNumBins];
};
constexpr PresetRow kPresets[] = {
    {"sym_1x", 0, {32, 512, 1024, 2048, 4096, 8192, 12287, kNoUpper}},
    {"sym_1.2x", 0, {26, 426, 853, 1706, 3413, 6826, 10240, kNoUpper}},
    {"sym_1.5x", 0, {21, 341, 682, 1365, 2730, 5461, 8191, kNoUpper}},
    {"num_1x", 1, {31, 255, 511, 1023, 2047, 4095, 8191, kNoUpper}},
    {"num_1.5x", 1, {21, 192, 384, 768, 1536, 3072, 5460, kNoUpper}},
    {"num_2x", 1, {16, 128, 256, 512, 1024, 2048, 4096, kNoUpper}},
    {"num_3x", 1, {10, 85, 170, 341, 682, 1365, 2730, kNoUpper}},
};

bool find_preset(int phase, const char* name, spgemm_bin_config* out) {
  for (const PresetRow& r : kPresets) {
    if (r.phase == phase && std::strcmp(r.name, name) == 0) {
      out->phase = phase;
      for (int j = 0; j < kNumBins; ++j) {
        out->upper[j] = r.upper[j];
        out->table_size[j] = phase == 0 ? kSymTable[j] : kNumTable[j];
      }
      std::memset(out->preset_name, 0, sizeof(out->preset_name));
      std::strncpy(out->preset_name, r.name, sizeof(out->preset_name) - 1);
      return true;
    }
  }
  return false;
}

int classify_host(int64_t v, const spgemm_bin_config& c) {
  for (int j = 0; j < kNumBins - 1; ++j)
    if (v <= c.upper[j]) return j;
  return kNumBins - 1;
}

// pipeline.cpp:64-87
void make_plan(const spgemm_bin_config& c, spgemm_plan* plan) {
  std::memset(plan, 0, sizeof(*plan));
  plan->phase = c.phase;
  plan->config = c;
  int64_t lo = 0;
  for (int j = 0; j < kNumBins; ++j) {
    spgemm_bin_strategy& s = plan->strategies[j];
    s.bin = j;
    s.metric_lo = lo;
    s.metric_hi = c.upper[j];
    if (s.metric_hi != kNoUpper) lo = s.metric_hi + 1;
    s.table_size = c.table_size[j];
    s.tier = s.table_size > 0 ? 0 : 1;
    s.spill_threshold =
        (c.phase == 0 && j == kNumBins - 1 && s.table_size > 0) ? s.table_size * 4 / 5 : 0;
    s.launch_rank = kNumBins - 1 - j;
  }
  for (int j = 0; j < kNumBins; ++j) plan->launch_order[j] = j;
  std::stable_sort(plan->launch_order, plan->launch_order + kNumBins, [&](int x, int y) {
    return plan->strategies[x].launch_rank < plan->strategies[y].launch_rank;
  });
}

void apply_launch_order(spgemm_plan* plan, const int32_t* order) {
  int32_t sorted[kNumBins];
  std::memcpy(sorted, order, sizeof(sorted));
  std::sort(sorted, sorted + kNumBins);
  for (int j = 0; j < kNumBins; ++j)
    if (sorted[j] != j)
      fail(SPGEMM_INVALID_ARGUMENT, "launch order must be a permutation of the bin indices");
  for (int j = 0; j < kNumBins; ++j) plan->strategies[order[j]].launch_rank = j;
  for (int j = 0; j < kNumBins; ++j) plan->launch_order[j] = j;
  std::stable_sort(plan->launch_order, plan->launch_order + kNumBins, [&](int x, int y) {
    return plan->strategies[x].launch_rank < plan->strategies[y].launch_rank;
  });
}

BinUpper to_upper(const spgemm_bin_config& c) {
  BinUpper u;
  for (int j = 0; j < kNumBins; ++j) u.u[j] = c.upper[j];
  return u;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
#ifndef SPGEMM_G8_MAX
#define SPGEMM_G8_MAX 8.0
#endif
// 8-lane groups when B's rows average at most this many entries (else 32)
constexpr double kG8MaxBLen = SPGEMM_G8_MAX;
#ifndef SPGEMM_THREAD_SLOTS
#define SPGEMM_THREAD_SLOTS 24
#endif
constexpr int kThreadNumSlots = SPGEMM_THREAD_SLOTS;  // k_num_thread's per-row table (>= 1.5 x 16)
#ifndef SPGEMM_THREAD_SYM_SLOTS
#define SPGEMM_THREAD_SYM_SLOTS 48
#endif
constexpr int kThreadSymSlots = SPGEMM_THREAD_SYM_SLOTS;  // k_sym_thread's per-row table (>= 1.5 x 32)
constexpr int64_t kSpecBudget = int64_t(4) << 30;      // scratch bytes the arena may spend on it
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

// ----------------------------------------------------------------- context
struct spgemm_ctx {
  int device = 0;
  int num_sms = 0;
  int max_smem = 0;
  cudaStream_t main_s = nullptr, side_s = nullptr;
  cudaStream_t bin_s[kNumBins] = {};
  cudaEvent_t ev_fork = nullptr, ev_side = nullptr, ev_info = nullptr;
  cudaEvent_t ev_join[kNumBins] = {};
  DevInfo* h_info = nullptr;      // pinned and mapped, two slots
  DevInfo* h_info_dev = nullptr;  // h_info's device address (written by k_info_to_host)
  std::atomic<int64_t> launches{0};
  std::mutex attr_mu;
  std::unordered_set<const void*> attr_done;
  std::map<std::tuple<const void*, int, size_t>, int> occupancy;  // per-kernel resident blocks/SM
  // Optional per-kernel timing: events bracket every launch on its own stream.
  bool prof = false;
  struct ProfRec {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec> prof_recs;
  std::string prof_tag;  // appended to the names of per-bin launches while profiling
  std::vector<cudaEvent_t> ev_pool;
  // Per-call scratch (the metadata arena, staged host inputs) kept across
  // multiplies: re-allocating multi-GB arenas every call fragments the
  // stream-ordered pool, whose growth then stalls a call for 100+ ms.
  struct Scratch {
    void* p;
    size_t bytes;
    bool busy;
  };
  std::vector<Scratch> scratch;
  cudaMemPool_t pool = nullptr;  // this context's stream-ordered pool
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <typename Kern>
void prepare_kernel(spgemm_ctx* ctx, Kern kern, size_t smem) {
  const void* key = reinterpret_cast<const void*>(kern);
  std::lock_guard<std::mutex> lock(ctx->attr_mu);
  if (ctx->attr_done.count(key)) return;
  ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(std::max<size_t>(smem, 48 * 1024))),
     "cudaFuncSetAttribute");
  ctx->attr_done.insert(key);
}

// Persistent grid: enough blocks to cover the work, at most one full wave of
// resident blocks (148 SMs x occupancy).
template <typename Kern>
int persistent_grid(spgemm_ctx* ctx, Kern kern, int threads, size_t smem, int64_t work) {
  int per_sm = 0;
  {
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), threads, smem);
    std::lock_guard<std::mutex> lock(ctx->attr_mu);
    auto it = ctx->occupancy.find(key);
    if (it != ctx->occupancy.end()) {
      per_sm = it->second;
    } else {
      ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem),
         "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
      ctx->occupancy[key] = per_sm;
    }
  }
  if (per_sm < 1) fail(SPGEMM_CUDA_ERROR, "kernel cannot be resident (shared memory too large)");
  const int64_t cap = static_cast<int64_t>(per_sm) * ctx->num_sms;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(work, cap)));
}

// Rows per warp of the structure-reuse kernel: as many consecutive rows as
// keep every resident warp busy (long runs let more rows reuse their
// predecessor; a small bin needs short runs to spread over the SMs).
// SPGEMM_REUSE_ROWS overrides (experiments).
template <typename Kern>
int reuse_rows_per_warp(spgemm_ctx* ctx, Kern kern, size_t smem, int64_t rows, int block_warps = kReuseWarps) {
  if (const char* e = std::getenv("SPGEMM_REUSE_ROWS")) return std::max(1, std::min(kReuseRows, std::atoi(e)));
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * block_warps, smem), "occupancy");
  const int64_t warps = static_cast<int64_t>(std::max(per_sm, 1)) * ctx->num_sms * block_warps;
  int r = kReuseRows;
  while (r > 1 && rows < warps * r) r >>= 1;
  return r;
}

void count_launch(spgemm_ctx* ctx, const char* what) {
  ck(cudaGetLastError(), what);
  ctx->launches.fetch_add(1, std::memory_order_relaxed);
}

cudaEvent_t pooled_event(spgemm_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  ck(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

// Brackets one kernel launch: counts it and, when profiling, records events
// on the launching stream around it.
struct LaunchScope {
  spgemm_ctx* ctx;
  std::string name;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  LaunchScope(spgemm_ctx* c, std::string n, cudaStream_t st) : ctx(c), name(std::move(n)), s(st) {
    if (ctx->prof) {
      name += ctx->prof_tag;  // "#s<bin>" / "#n<bin>": the phase and bin of a per-bin launch
      a = pooled_event(ctx);
      ck(cudaEventRecord(a, s), "prof event");
    }
  }
  void done() {
    count_launch(ctx, name.c_str());
    if (a) {
      cudaEvent_t b = pooled_event(ctx);
      ck(cudaEventRecord(b, s), "prof event");
      ctx->prof_recs.push_back({name, a, b});
    }
  }
};

#define SPG_LAUNCH(CTX, NAME, STREAM, ...)       \
  do {                                           \
    LaunchScope ls_((CTX), (NAME), (STREAM));    \
    __VA_ARGS__;                                 \
    ls_.done();                                  \
  } while (0)

// Bins run concurrently on their own streams; with per-launch profiling on they
// run in order on the main stream, so each launch's events time that kernel alone
// (concurrent bins would fold their co-resident neighbours into its duration).
cudaStream_t bin_stream(spgemm_ctx* ctx, int bin) { return ctx->prof ? ctx->main_s : ctx->bin_s[bin]; }

// Stream-ordered allocations come from the context's own memory pool (not the
// device's default pool, whose settings other libraries in the process rely on).
void* dev_alloc_ctx(spgemm_ctx* ctx, size_t bytes, cudaStream_t s) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  ck(cudaMallocFromPoolAsync(&p, bytes, ctx->pool, s), "cudaMallocFromPoolAsync");
  return p;
}
#define dev_alloc(BYTES, STREAM) dev_alloc_ctx(ctx, (BYTES), (STREAM))

void dev_free(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

// Scratch blocks live on the context and are used on its main stream only, so a
// block released by one call and handed to the next is stream-ordered.
void* scratch_acquire(spgemm_ctx* ctx, size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  spgemm_ctx::Scratch* best = nullptr;
  for (auto& b : ctx->scratch)
    if (!b.busy && b.bytes >= bytes && b.bytes <= 2 * bytes + (size_t(64) << 20) && (!best || b.bytes < best->bytes))
      best = &b;
  if (best) {
    best->busy = true;
    return best->p;
  }
  // no fit: give the idle blocks back first, so the cache tracks the working set
  std::vector<spgemm_ctx::Scratch> keep;
  for (auto& b : ctx->scratch) {
    if (b.busy) keep.push_back(b);
    else dev_free(b.p, s);
  }
  ctx->scratch.swap(keep);
  void* p = dev_alloc(bytes, s);
  ctx->scratch.push_back({p, bytes, true});
  return p;
}

void scratch_release(spgemm_ctx* ctx, void* p) {
  if (!p) return;
  for (auto& b : ctx->scratch)
    if (b.p == p) {
      b.busy = false;
      return;
    }
}

}  // namespace

// -------------------------------------------------------- result matrices
struct spgemm_matrix {
  spgemm_ctx* ctx = nullptr;
  int64_t rows = 0, cols = 0, nnz = 0;
  int64_t* rpt = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
};

// ----------------------------------------------------------------- pipeline
struct spgemm_pipeline {
  enum Stage { kNew, kSetup, kSymBinned, kSymbolic, kNumBinned, kRptDone, kNumeric, kDone };

  spgemm_ctx* ctx = nullptr;
  spgemm_options opts{};
  spgemm_plan sym_plan{}, num_plan{};
  BinUpper sym_up{}, num_up{};
  DevCsr A{}, B{};
  int64_t a_nnz = 0, b_nnz = 0;
  void* owned[6] = {};
  int64_t M = 0;
  int64_t nrb = 0, ntiles = 0;
  uint32_t scale = 107;
  double avg_b_len = 0;
  bool idx32 = true;
  int64_t b_rows = 0;
  // operand sizes: known at creation for host operands, from K1 for device ones
  void set_sizes() {
    // 32-bit B/A offsets in the group and heap kernels when every offset fits;
    // SPGEMM_FORCE_IDX64=1 takes the 64-bit kernels regardless (test coverage of
    // the path inputs above 2^31 nonzeros take)
    idx32 = a_nnz < (int64_t(1) << 31) && b_nnz < (int64_t(1) << 31) && std::getenv("SPGEMM_FORCE_IDX64") == nullptr;
    avg_b_len = b_rows > 0 ? static_cast<double>(b_nnz) / static_cast<double>(b_rows) : 0;
  }
  bool sym_bins_on_device = false;

  int64_t* d_rpt = nullptr;
  unsigned char* d_arena = nullptr;
  size_t arena_bytes = 0;
  int64_t* d_bins = nullptr;
  int64_t* d_spill = nullptr;
  Spec spec{nullptr, nullptr, nullptr, 0};  // speculative numeric scratch (arena)
  bool regular_a = false;                    // A's longest row <= 4x its mean (set by setup)
  bool reuse_route = false;                  // structure-reuse kernels (set by setup, see there)
  bool symbolic_only = false;                // spgemm_forecast_nnz: no speculative numeric, no C
  int32_t* d_blk = nullptr;
  int* d_flags = nullptr;
  long long* d_sums = nullptr;
  DevInfo* d_info_sym = nullptr;
  DevInfo* d_info_num = nullptr;
  int32_t* d_ccol = nullptr;
  double* d_cval = nullptr;
  bool alloc_pending = false;

  DevInfo h_sym{}, h_num{};
  spgemm_binning_info bin_info{};
  int64_t total_nprod = 0, total_nnz = 0;
  int stage = kNew;
  cudaEvent_t ev[12] = {};
  int64_t metadata_calls = 0, metadata_bytes = 0, output_calls = 0, output_bytes = 0;
  double cleanup_s = 0;
  bool result_taken = false;

  void expect(int s, const char* op) {
    if (stage != s)
      fail(SPGEMM_LOGIC_ERROR, std::string("spgemm pipeline: ") + op + " called out of order");
  }
  void mark(int i) { ck(cudaEventRecord(ev[i], ctx->main_s), "cudaEventRecord"); }
  double span(int i, int j) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, ev[i], ev[j]), "cudaEventElapsedTime");
    return ms * 1e-3;
  }
  // DevInfo -> pinned host slot `slot` (k_info_to_host, no copy engine), stream-ordered
  void info_to_host(const DevInfo* d, int slot, int count, cudaStream_t s) {
    SPG_LAUNCH(ctx, "k_info_to_host", s, k_info_to_host<<<1, 64, 0, s>>>(d, ctx->h_info_dev + slot, count));
  }
  void fetch_info(DevInfo* d, DevInfo* h) {
    info_to_host(d, 0, 1, ctx->main_s);
    ck(cudaStreamSynchronize(ctx->main_s), "cudaStreamSynchronize");
    *h = *ctx->h_info;
  }

  void setup();
  void symbolic_binning();
  void run_symbolic();
  void numeric_binning();
  int64_t finalize_rpt(bool host_total = true);
  void run_numeric();
  void finish(spgemm_report* r);
  void allocate_output(cudaStream_t s);
  void launch_sym_bin(int bin, const RowList& rl, cudaStream_t s);
  void launch_num_bin(int bin, const RowList& rl, cudaStream_t s, int32_t* gkeys, double* gvals,
                      uint32_t* gbits, int64_t gslots, int64_t gwords, int gblocks);
  void release(bool keep_result);
  // heap-tier numeric: the ordered kernel whenever the reference's determinism
  // contract applies (options.deterministic, the default: C bitwise the
  // reference's) or options.ordered_heap forces it; bitmap rank +
  // fp64 atomics (within 1e-12, run-to-run bits may differ) only for
  // deterministic=false
  // A and B of one shape and size (C = A*A, possibly two copies of A): the
  // products whose rows repeat their neighbours' structure (stencils)
  bool square_like() const { return A.rows == B.rows && A.cols == B.cols && a_nnz == b_nnz; }
  bool heap_ordered() const { return opts.ordered_heap || opts.deterministic; }
  bool heap_bitmap() const { return idx32; }  // bitmap kernels (ordered or atomic); else k_num_global
  // numeric bins past the largest on-chip table (16384 slots: rows of <= 8192
  // nonzeros, the B200 tier) take the heap tier; so do the block-table bins
  // whose rows all have > 2048 nonzeros when B's rows are short on average, as
  // in the symbolic phase: a per-A-entry block walk leaves most threads idle on
  // skewed graphs, the bitmap walk is balanced by products
  bool heap_tier(int bin) const {
    const int64_t u = num_plan.config.upper[bin];
    const int64_t lo = bin > 0 ? num_plan.config.upper[bin - 1] + 1 : 0;
    return bin == kNumBins - 1 || u > kSharedNumMax || (heap_bitmap() && lo > 2048 && avg_b_len < 64.0);
  }
  int32_t* d_poff = nullptr;                   // ordered bitmap tier: B's column-panel offsets
  uint8_t* d_shift1 = nullptr;                 // B row k == B row k-1 shifted by one (arena)
  uint8_t* d_rflag = nullptr;                  // row i's structure == row i-1's shifted by one (arena)
};

namespace {

void stage_input(spgemm_ctx* ctx, const spgemm_csr_view* v, DevCsr* d, void** owned, int64_t* nnz) {
  d->rows = v->rows;
  d->cols = v->cols;
  if (v->rows < 0 || v->cols < 0) fail(SPGEMM_INVALID_ARGUMENT, "negative matrix shape");
  if (v->cols > std::numeric_limits<int32_t>::max())
    fail(SPGEMM_INVALID_ARGUMENT, "column count exceeds the 32-bit index range");
  if (v->rows >= std::numeric_limits<int32_t>::max())
    fail(SPGEMM_INVALID_ARGUMENT, "row count exceeds the 32-bit row-id range");
  if (!v->rpt) fail(SPGEMM_INVALID_ARGUMENT, "null rpt");
  if (v->on_device) {
    // Device operands written by work on the legacy default stream (a torch
    // copy, say) are ordered before this product's kernels.
    if (!g_inputs_stream_ordered) {
      cudaEvent_t e = pooled_event(ctx);
      ck(cudaEventRecord(e, cudaStreamLegacy), "record default stream");
      ck(cudaStreamWaitEvent(ctx->main_s, e, 0), "main waits for default stream");
      ctx->ev_pool.push_back(e);
    }
    // nnz = rpt[rows] stays on the device: K1 reports it with its phase
    // scalars (no extra host round trip per operand)
    *nnz = -1;
    d->rpt = v->rpt;
    d->col = v->col;
    d->val = v->val;
    return;
  }
  *nnz = v->rpt[v->rows];
  const size_t rb = static_cast<size_t>(v->rows + 1) * sizeof(int64_t);
  const size_t cb = static_cast<size_t>(*nnz) * sizeof(int32_t);
  const size_t vb = static_cast<size_t>(*nnz) * sizeof(double);
  owned[0] = scratch_acquire(ctx, rb, ctx->main_s);
  owned[1] = scratch_acquire(ctx, cb, ctx->main_s);
  owned[2] = scratch_acquire(ctx, vb, ctx->main_s);
  ck(cudaMemcpyAsync(owned[0], v->rpt, rb, cudaMemcpyHostToDevice, ctx->main_s), "H2D rpt");
  if (cb) ck(cudaMemcpyAsync(owned[1], v->col, cb, cudaMemcpyHostToDevice, ctx->main_s), "H2D col");
  if (vb) ck(cudaMemcpyAsync(owned[2], v->val, vb, cudaMemcpyHostToDevice, ctx->main_s), "H2D val");
  d->rpt = static_cast<const int64_t*>(owned[0]);
  d->col = static_cast<const int32_t*>(owned[1]);
  d->val = static_cast<const double*>(owned[2]);
}

}  // namespace

void spgemm_pipeline::setup() {
  expect(kNew, "setup");
  mark(0);
  cudaStream_t s = ctx->main_s;
  nrb = ceil_div(M, kRowsPerBlock);
  ntiles = ceil_div(M + 1, kScanTile);
  // Allocation 1: C.rpt, with K1's outputs behind it (phase scalars and the
  // per-row-block bin counts), so the arena can be sized after K1.
  const size_t o_info = align_up(static_cast<size_t>(M + 1) * 8, 256);
  const size_t o_blk = align_up(o_info + 2 * sizeof(DevInfo), 256);
  const size_t rpt_bytes = align_up(o_blk + static_cast<size_t>(std::max<int64_t>(nrb, 1)) * kNumBins * 4, 256);
  unsigned char* head = static_cast<unsigned char*>(dev_alloc(rpt_bytes, s));
  d_rpt = reinterpret_cast<int64_t*>(head);
  d_info_sym = reinterpret_cast<DevInfo*>(head + o_info);
  d_info_num = d_info_sym + 1;
  d_blk = reinterpret_cast<int32_t*>(head + o_blk);
  metadata_calls += 1;
  metadata_bytes += static_cast<int64_t>(rpt_bytes);
  ck(cudaMemsetAsync(d_info_sym, 0, 2 * sizeof(DevInfo), s), "memset info");
  if (M > 0) {
    SPG_LAUNCH(ctx, "k_setup_nprod", s,
               k_setup_nprod<<<static_cast<unsigned>(nrb), kBinThreads, 0, s>>>(A, B.rpt, b_rows, d_rpt, M, sym_up,
                                                                      d_blk, d_info_sym));
  } else {
    ck(cudaMemsetAsync(d_rpt, 0, 8, s), "memset rpt");
  }
  fetch_info(d_info_sym, &h_sym);
  if (a_nnz < 0) a_nnz = M > 0 ? h_sym.a_nnz : 0;
  if (b_nnz < 0) b_nnz = M > 0 ? h_sym.b_nnz : 0;
  set_sizes();
  if (h_sym.total > static_cast<unsigned long long>(std::numeric_limits<int64_t>::max()))
    fail(SPGEMM_OVERFLOW, "spgemm: intermediate-product count overflowed 64 bits");
  total_nprod = static_cast<int64_t>(h_sym.total);
  // Allocation 2: the arena -- scan state, bin row ids, spill ids and, when
  // some symbolic bin will run it, the speculative-numeric scratch (Spec in
  // kernels.cuh), decided now that K1 has reported A's row statistics.
  size_t off = 0;
  const size_t o_flags = off;
  off = align_up(off + static_cast<size_t>(ntiles) * 4, 256);
  const size_t o_sums = off;
  off = align_up(off + static_cast<size_t>(ntiles) * 16, 256);
  const size_t o_bins = off;  // row ids as int64, the reference's BinningResult layout
  off = align_up(off + static_cast<size_t>(std::max<int64_t>(M, 1)) * 8, 256);
  const size_t o_spill = off;
  off = align_up(off + static_cast<size_t>(std::max<int64_t>(M, 1)) * 8, 256);
  regular_a = M > 0 && static_cast<double>(h_sym.a_max_row) <= 4.0 * static_cast<double>(a_nnz) / static_cast<double>(M);
  // Structure-reuse route: A*A-shaped products of regular A with warp-sized A
  // and B rows and B rows of > 8 entries on average (3-D stencils, FEM). Per-row
  // flags (k_reuse_flags) drive the symbolic count (k_sym_reuse) and the
  // numeric phase writes C with k_num_reuse_multi (kernels_reuse.cuh) -- no
  // speculative scratch, no copy. SPGEMM_NO_REUSE=1 disables it.
  reuse_route = idx32 && M > 0 && h_sym.a_max_row <= 32 && h_sym.b_max_row <= 32 && regular_a &&
                avg_b_len > 8.0 && square_like() && std::getenv("SPGEMM_NO_REUSE") == nullptr;
  const bool use_spec = !reuse_route && idx32 && M > 0 && avg_b_len > 8.0 && regular_a &&
                        M * kSpecCap * 12 <= kSpecBudget &&
                        !symbolic_only && std::getenv("SPGEMM_NO_SPEC") == nullptr;
  const size_t o_sflag = off, o_scol = align_up(o_sflag + (use_spec ? static_cast<size_t>(M) : 0), 256);
  const size_t o_sval = align_up(o_scol + (use_spec ? static_cast<size_t>(M) * kSpecCap * 4 : 0), 256);
  if (use_spec) off = align_up(o_sval + static_cast<size_t>(M) * kSpecCap * 8, 256);
  // the structure-reuse kernels' per-B-row shift flags (warp-sized A and B rows)
  // (only the speculative path's products -- regular A, long B rows -- reuse structure)
  const bool use_shift = reuse_route;
  const size_t o_shift = off;
  if (use_shift) off = align_up(o_shift + static_cast<size_t>(std::max<int64_t>(b_rows, 1)), 256);
  const size_t o_rflag = off;
  if (use_shift) off = align_up(o_rflag + static_cast<size_t>(std::max<int64_t>(M, 1)), 256);
  arena_bytes = off;
  d_arena = static_cast<unsigned char*>(scratch_acquire(ctx, arena_bytes, s));
  metadata_calls += 1;
  metadata_bytes += static_cast<int64_t>(arena_bytes);
  d_flags = reinterpret_cast<int*>(d_arena + o_flags);
  d_sums = reinterpret_cast<long long*>(d_arena + o_sums);
  d_bins = reinterpret_cast<int64_t*>(d_arena + o_bins);
  d_spill = reinterpret_cast<int64_t*>(d_arena + o_spill);
  d_shift1 = nullptr;
  d_rflag = nullptr;
  if (use_shift && b_rows > 0) {
    d_shift1 = d_arena + o_shift;
    const int fg = static_cast<int>(std::min<int64_t>(ctx->num_sms * 64, ceil_div(b_rows, 256)));
    SPG_LAUNCH(ctx, "k_shift_flags", s, k_shift_flags<<<std::max(fg, 1), 256, 0, s>>>(B, d_shift1));
    d_rflag = d_arena + o_rflag;
    const int a_is_b = A.rpt == B.rpt && A.col == B.col;
    const int rg = static_cast<int>(std::min<int64_t>(ctx->num_sms * 64, ceil_div(M, 256)));
    SPG_LAUNCH(ctx, "k_reuse_flags", s, k_reuse_flags<<<std::max(rg, 1), 256, 0, s>>>(A, d_shift1, d_rflag, a_is_b));
  }
  if (use_spec) {
    spec = Spec{reinterpret_cast<int32_t*>(d_arena + o_scol), reinterpret_cast<double*>(d_arena + o_sval),
                d_arena + o_sflag, kSpecCap};
    ck(cudaMemsetAsync(spec.flag, 0, static_cast<size_t>(M), s), "memset spec flags");
  } else {
    spec = Spec{nullptr, nullptr, nullptr, 0};
  }
  mark(1);
  stage = kSetup;
}

void spgemm_pipeline::symbolic_binning() {
  expect(kSetup, "symbolic_binning");
  mark(2);
  cudaStream_t s = ctx->main_s;
  std::memset(&bin_info, 0, sizeof(bin_info));
  bin_info.max_metric = h_sym.max_metric;
  bin_info.total_metric = static_cast<int64_t>(h_sym.total);
  const bool fast = M == 0 || h_sym.max_metric <= sym_up.u[0];
  if (fast) {
    bin_info.fast_path = 1;
    bin_info.bin_size[0] = M;
  } else {
    SPG_LAUNCH(ctx, "k_bin_offsets", s,
               k_bin_offsets<<<1, 1024, 0, s>>>(d_blk, nrb, M, sym_up.u[0], d_info_sym));
    SPG_LAUNCH(ctx, "k_bin_scatter", s,
               k_bin_scatter<<<static_cast<unsigned>(nrb), kBinThreads, 0, s>>>(d_rpt, M, sym_up, d_blk,
                                                                      d_bins, d_info_sym));
    // No host round trip: the symbolic kernels read their bin's size and
    // offset from d_info_sym; binning() fetches them only if asked.
    sym_bins_on_device = true;
  }
  mark(3);
  stage = kSymBinned;
}

// ------------------------------------------------------- symbolic dispatch
// Tier choice per bin from the preset's inclusive upper bound on nprod (the
// bin invariant guarantees the table never fills). G (lanes per row) follows
// the mean B row length so the lanes striding a B row stay busy.
// Group kernels index B with 32-bit offsets when nnz(A), nnz(B) < 2^31.
#define SYMG(G, T, N, WB) (idx32 ? &k_sym_group<G, T, N, int32_t, WB> : &k_sym_group<G, T, N, int64_t, WB>)
#define NUMG(G, T, E, N) \
  (idx32 ? &k_num_group<G, T, E, N, int32_t, false> : &k_num_group<G, T, E, N, int64_t, false>)

void spgemm_pipeline::launch_sym_bin(int bin, const RowList& rl, cudaStream_t s) {
  ctx->prof_tag = "#s" + std::to_string(bin);
  struct Untag {
    spgemm_ctx* c;
    ~Untag() { c->prof_tag.clear(); }
  } untag{ctx};
  const int64_t u = sym_plan.config.upper[bin];
  const bool g8 = avg_b_len <= kG8MaxBLen;
  if (reuse_route && u > 32 && u <= 1024) {  // structure-reuse counting (kernels.cuh k_sym_reuse)
    const size_t smem = static_cast<size_t>(kSymReuseWarps) * kSymReuseWarpBytes;
    prepare_kernel(ctx, k_sym_reuse, smem);
    // (the bin's size is on the device: the kernel sizes its runs from it)
    const int grid = persistent_grid(ctx, k_sym_reuse, 32 * kSymReuseWarps, smem, ceil_div(rl.count, kSymReuseWarps));
    SPG_LAUNCH(ctx, "k_sym_reuse", s,
               k_sym_reuse<<<grid, 32 * kSymReuseWarps, smem, s>>>(rl, A, B, d_rpt, scale, 0, d_rflag, d_info_sym));
    return;
  }
  auto group = [&](auto kern, int G, int T, int NGRP, int WB) {
    // Only where the numeric phase would also run a 32-lane group on a table
    // of 256 (rows with 513..1024 products, or 257..512 when B's rows average
    // >= 16 entries) and A's rows are
    // regular (3-D stencils, FEM: the distinct count of such rows fits the
    // 128-entry scratch); shorter rows are cheaper through the small kernels,
    // and skewed rows (graphs) rarely fit.
    if (spec.flag != nullptr && G == 32 && u <= 1024 && regular_a && (u > 512 || (u > 256 && avg_b_len >= 16.0))) {
      // speculative numeric first; the symbolic kernel then skips the rows it finished
      if (square_like()) {  // C = A*A-shaped: structure reuse (stencil rows repeat)
        auto sk = &k_num_reuse<true>;
        const size_t ssm = static_cast<size_t>(kReuseWarps) * kReuseWarpBytes;
        prepare_kernel(ctx, sk, ssm);
        const int rpw = 0;  // (the symbolic bin's size is on the device: the kernel sizes its runs)
        const int sgrid = persistent_grid(ctx, sk, 32 * kReuseWarps, ssm, ceil_div(rl.count, kReuseWarps));
        SPG_LAUNCH(ctx, "k_num_reuse<spec>", s,
                   sk<<<sgrid, 32 * kReuseWarps, ssm, s>>>(rl, A, B, d_rpt, nullptr, nullptr, scale, d_info_sym,
                                                           spec, rpw, d_shift1));
      } else {
        auto sk = &k_num_lean<true>;
        const size_t ssm = static_cast<size_t>(kLeanGroups) * kLeanGroupBytes;
        prepare_kernel(ctx, sk, ssm);
        const int sgrid = persistent_grid(ctx, sk, 32 * kLeanGroups, ssm, ceil_div(rl.count, kLeanGroups));
        SPG_LAUNCH(ctx, "k_num_lean<spec>", s,
                   sk<<<sgrid, 32 * kLeanGroups, ssm, s>>>(rl, A, B, d_rpt, nullptr, nullptr, scale, d_info_sym,
                                                           spec));
      }
    }
    const size_t smem = static_cast<size_t>(NGRP) * (static_cast<size_t>(std::max(T, WB)) * 4 + G * 16);
    prepare_kernel(ctx, kern, smem);
    const int grid = persistent_grid(ctx, kern, G * NGRP, smem, ceil_div(rl.count, NGRP));
    SPG_LAUNCH(ctx, "k_sym_group<" + std::to_string(G) + "," + std::to_string(T) + ">", s,
               kern<<<grid, G * NGRP, smem, s>>>(rl, A, B, d_rpt, scale, spec));
  };
  auto block = [&](auto kern, int T, int threads) {
    const size_t smem = static_cast<size_t>(T) * 4;
    prepare_kernel(ctx, kern, smem);
    const int grid = persistent_grid(ctx, kern, threads, smem, rl.count);
    SPG_LAUNCH(ctx, "k_sym_block<" + std::to_string(T) + ">", s,
               kern<<<grid, threads, smem, s>>>(rl, A, B, d_rpt, scale, d_spill, d_info_sym,
                                     static_cast<int>(sym_plan.strategies[bin].spill_threshold)));
  };
  // Bitmap kernel for the top bin, and for the block-table bins too when the
  // rows' B rows are short on average (skewed graphs: a per-A-entry table walk
  // leaves most lanes idle there; the bitmap walk is balanced by products).
  if (idx32 && (bin == kNumBins - 1 || (u > 2048 && avg_b_len < 64.0))) {
    // bitmap kernel: exact counts, no spill recount (kernels_heap.cuh)
    prepare_kernel(ctx, k_big_sym, kBigSymSmem);
    const int grid = persistent_grid(ctx, k_big_sym, kBigThreads, kBigSymSmem, rl.count);
    SPG_LAUNCH(ctx, "k_big_sym", s,
               k_big_sym<<<grid, kBigThreads, kBigSymSmem, s>>>(
                   rl, A, B, d_rpt, d_info_sym,
                   bin == kNumBins - 1 ? static_cast<int>(sym_plan.strategies[bin].spill_threshold)
                                       : std::numeric_limits<int>::max()));
    return;
  }
  if (bin == kNumBins - 1) {
    block(k_sym_block<32768, 1024, true>, 32768, 1024);
    // Heap-tier recompute of the spilled rows (pipeline.cpp:315-348): a pool
    // of per-block global tables; the kernel reads the spill count on device.
    long long want = 2 * std::min<long long>(h_sym.max_metric, B.cols);
    int64_t slots = 2;
    while (slots < want) slots <<= 1;
    const int64_t budget = int64_t(4) << 30;
    const int blocks = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>({2LL * ctx->num_sms, rl.count, budget / (slots * 4)})));
    int32_t* pool = static_cast<int32_t*>(dev_alloc(static_cast<size_t>(slots) * 4 * blocks, s));
    SPG_LAUNCH(ctx, "k_sym_spill", s,
               k_sym_spill<<<blocks, 1024, 0, s>>>(A, B, d_rpt, d_spill, d_info_sym, pool, slots, scale));
    dev_free(pool, s);
    return;
  }
  if (u <= 32) {  // thread per row, private table of 1.5 x 32 slots (load <= 2/3)
    constexpr int TS = kThreadSymSlots;
    const size_t smem = 256 * TS * 4;
    auto kern = &k_sym_thread<TS>;
    prepare_kernel(ctx, kern, smem);
    const int grid = persistent_grid(ctx, kern, 256, smem, ceil_div(rl.count, 256));
    SPG_LAUNCH(ctx, "k_sym_thread<" + std::to_string(TS) + ">", s,
               kern<<<grid, 256, smem, s>>>(rl, A, B, d_rpt, scale));
    return;
  }
  // group kernels: (G, T, groups per block, bitmap words per group)
  if (u < 64) {
    if (g8) group(SYMG(8, 64, 32, 256), 8, 64, 32, 256);
    else group(SYMG(32, 64, 8, 256), 32, 64, 8, 256);
  } else if (u < 512) {
    if (g8) group(SYMG(8, 512, 32, 512), 8, 512, 32, 512);
    else group(SYMG(32, 512, 8, 512), 32, 512, 8, 512);
  } else if (u < 1024) {
    if (g8) group(SYMG(8, 1024, 16, 1024), 8, 1024, 16, 1024);
    else group(SYMG(32, 1024, 8, 1024), 32, 1024, 8, 1024);
  } else if (u < 2048) {
    if (g8) group(SYMG(8, 2048, 8, 2048), 8, 2048, 8, 2048);
    else group(SYMG(32, 2048, 8, 2048), 32, 2048, 8, 2048);
  } else if (u < 4096) {
    block(k_sym_block<4096, 256, false>, 4096, 256);
  } else if (u < 8192) {
    block(k_sym_block<8192, 256, false>, 8192, 256);
  } else {
    block(k_sym_block<16384, 512, false>, 16384, 512);
  }
}

void spgemm_pipeline::run_symbolic() {
  expect(kSymBinned, "run_symbolic");
  mark(4);
  ck(cudaEventRecord(ctx->ev_fork, ctx->main_s), "ev_fork");
  // bins above the one holding the max nprod are empty (max known since setup)
  int top = kNumBins - 1;
  while (top > 0 && h_sym.max_metric <= sym_plan.config.upper[top - 1]) --top;
  for (int r = 0; r < kNumBins; ++r) {
    const int bin = sym_plan.launch_order[r];
    if (sym_bins_on_device ? bin > top : bin_info.bin_size[bin] == 0) continue;
    cudaStream_t s = bin_stream(ctx, bin);
    ck(cudaStreamWaitEvent(s, ctx->ev_fork, 0), "wait fork");
    // device-resolved row list: `count` only sizes the persistent grid
    RowList rl = sym_bins_on_device
                     ? RowList{d_bins, 0, M, 0, d_info_sym, bin}
                     : RowList{d_bins, bin_info.bin_offset[bin], bin_info.bin_size[bin], bin_info.fast_path,
                               nullptr, bin};
    launch_sym_bin(bin, rl, s);
    ck(cudaEventRecord(ctx->ev_join[bin], s), "ev_join");
    ck(cudaStreamWaitEvent(ctx->main_s, ctx->ev_join[bin], 0), "wait join");
  }
  mark(5);
  stage = kSymbolic;
}

void spgemm_pipeline::allocate_output(cudaStream_t s) {
  d_ccol = static_cast<int32_t*>(dev_alloc(static_cast<size_t>(total_nnz) * 4, s));
  d_cval = static_cast<double*>(dev_alloc(static_cast<size_t>(total_nnz) * 8, s));
  output_calls += 2;
  output_bytes += total_nnz * 12;
}

void spgemm_pipeline::numeric_binning() {
  expect(kSymbolic, "numeric_binning");
  mark(6);
  cudaStream_t s = ctx->main_s;
  std::memset(&bin_info, 0, sizeof(bin_info));
  if (M > 0) {
    SPG_LAUNCH(ctx, "k_pass1", s,
               k_pass1<<<static_cast<unsigned>(nrb), kBinThreads, 0, s>>>(d_rpt, M, num_up, d_blk, d_info_num));
    SPG_LAUNCH(ctx, "k_bin_offsets", s,
               k_bin_offsets<<<1, 1024, 0, s>>>(d_blk, nrb, M, num_up.u[0], d_info_num));
  }
  // The pass-1 total sizes C; read it back while the scatter runs and start
  // the C allocation on the side lane (pipeline.cpp:245-257).
  info_to_host(d_info_num, 1, 1, s);
  ck(cudaEventRecord(ctx->ev_info, s), "ev_info");
  if (M > 0) {
    SPG_LAUNCH(ctx, "k_bin_scatter", s,
               k_bin_scatter<<<static_cast<unsigned>(nrb), kBinThreads, 0, s>>>(d_rpt, M, num_up, d_blk,
                                                                      d_bins, d_info_num));
  }
  ck(cudaEventSynchronize(ctx->ev_info), "sync num info");
  h_num = ctx->h_info[1];
  if (M == 0) h_num.fast_path = 1;
  if (h_num.total > static_cast<unsigned long long>(std::numeric_limits<int64_t>::max()))
    fail(SPGEMM_OVERFLOW, "spgemm: nonzero count overflowed 64 bits");
  total_nnz = static_cast<int64_t>(h_num.total);
  if (opts.overlap && !symbolic_only) {
    // C.col/C.val are allocated now, stream-ordered behind the scatter that is
    // still running (the allocation lane of pipeline.cpp:254-257). Same stream
    // as the previous product's free, so the pool reuses that memory directly.
    allocate_output(s);
  }
  bin_info.max_metric = h_num.max_metric;
  bin_info.total_metric = total_nnz;
  bin_info.fast_path = h_num.fast_path;
  for (int j = 0; j < kNumBins; ++j) {
    bin_info.bin_size[j] = h_num.bin_size[j];
    bin_info.bin_offset[j] = h_num.bin_offset[j];
  }
  mark(7);
  stage = kNumBinned;
}

int64_t spgemm_pipeline::finalize_rpt(bool host_total) {
  expect(kNumBinned, "finalize_rpt");
  mark(8);
  cudaStream_t s = ctx->main_s;
  ck(cudaMemsetAsync(d_flags, 0, static_cast<size_t>(ntiles) * 4, s), "memset flags");
  SPG_LAUNCH(ctx, "k_scan", s,
             k_scan<<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(d_rpt, M + 1, d_flags, d_sums,
                                                                 d_sums + ntiles, d_info_num));
  // The scan total is cross-checked against the pass-1 total on the device
  // (kErrScanMismatch, raised at finish); the step API reads it back now.
  if (host_total) {
    DevInfo tmp;
    fetch_info(d_info_num, &tmp);
    if (tmp.scan_total != total_nnz)
      fail(SPGEMM_LOGIC_ERROR, "spgemm: exclusive sum disagrees with binning total");
  }
  if (!d_ccol) allocate_output(s);  // overlap=false: allocate only now
  mark(9);
  stage = kRptDone;
  return total_nnz;
}

// -------------------------------------------------------- numeric dispatch
void spgemm_pipeline::launch_num_bin(int bin, const RowList& rl, cudaStream_t s, int32_t* gkeys,
                                     double* gvals, uint32_t* gbits, int64_t gslots,
                                     int64_t gwords, int gblocks) {
  ctx->prof_tag = "#n" + std::to_string(bin);
  struct Untag {
    spgemm_ctx* c;
    ~Untag() { c->prof_tag.clear(); }
  } untag{ctx};
  const int64_t u = num_plan.config.upper[bin];
  const bool g8 = avg_b_len <= kG8MaxBLen;
  auto group = [&](auto kern, int G, int T, int E, int NGRP) {
    const size_t smem = static_cast<size_t>(NGRP) * ((T + 2) * 8 + G * E * 8 + T * 4 + G * 16 + 16);
    prepare_kernel(ctx, kern, smem);
    const int grid = persistent_grid(ctx, kern, G * NGRP, smem, ceil_div(rl.count, NGRP));
    SPG_LAUNCH(ctx, "k_num_group<" + std::to_string(G) + "," + std::to_string(T) + ">", s,
               kern<<<grid, G * NGRP, smem, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, scale, d_info_num, spec));
  };
  auto block = [&](auto kern, int T, int threads, int nmax, bool overlay = false) {
    const size_t smem = static_cast<size_t>(T) * 12 + (overlay ? 0 : static_cast<size_t>(nmax) * 8);
    prepare_kernel(ctx, kern, smem);
    const int grid = persistent_grid(ctx, kern, threads, smem, rl.count);
    SPG_LAUNCH(ctx, "k_num_block<" + std::to_string(T) + ">", s,
               kern<<<grid, threads, smem, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, scale, d_info_num));
  };
  if (heap_tier(bin) && heap_bitmap() && heap_ordered()) {
    prepare_kernel(ctx, k_big_num_ord, kBigNumSmem);
    const int grid = persistent_grid(ctx, k_big_num_ord, kBigThreads, kBigNumSmem, rl.count);
    SPG_LAUNCH(ctx, "k_big_num_ord", s,
               k_big_num_ord<<<grid, kBigThreads, kBigNumSmem, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, d_poff,
                                                                    d_info_num));
  } else if (heap_tier(bin) && heap_bitmap()) {
    prepare_kernel(ctx, k_big_num, kBigNumSmem);
    const int grid = persistent_grid(ctx, k_big_num, kBigThreads, kBigNumSmem, rl.count);
    SPG_LAUNCH(ctx, "k_big_num", s,
               k_big_num<<<grid, kBigThreads, kBigNumSmem, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, d_info_num));
  } else if (heap_tier(bin)) {
    SPG_LAUNCH(ctx, "k_num_global", s,
               k_num_global<<<gblocks, kGlobalThreads, 0, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, scale, gkeys,
                                                    gvals, gbits, gslots, gwords, d_info_num));
  } else if (u <= 16) {  // thread per row: 24-slot private table, 16-key register sort
    constexpr int TS = kThreadNumSlots;
    const size_t smem = 128 * TS * 12;
    auto kern = &k_num_thread<TS, 16>;
    prepare_kernel(ctx, kern, smem);
    const int grid = persistent_grid(ctx, kern, 128, smem, ceil_div(rl.count, 128));
    SPG_LAUNCH(ctx, "k_num_thread<" + std::to_string(TS) + ",16>", s,
               kern<<<grid, 128, smem, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, scale, d_info_num, spec));
  } else if (u <= 32) {
    if (g8) group(NUMG(8, 64, 4, 32), 8, 64, 4, 32);
    else group(NUMG(32, 64, 1, 8), 32, 64, 1, 8);
  } else if (u <= 128) {
    if (g8) {
      group(NUMG(8, 256, 16, 16), 8, 256, 16, 16);
    } else if (idx32 && h_sym.a_max_row <= 32 && h_sym.b_max_row <= 32 && std::getenv("SPGEMM_NO_LEAN") == nullptr) {
      // C = A*A of a regular matrix (stencils: the structure repeats row to
      // row): structure reuse; other products (the RAP chain's A*P, R*AP):
      // the dense-index kernel
      if (reuse_route) {
        auto kern = &k_num_reuse_multi;
        const size_t smem = static_cast<size_t>(kMultiWarps) * kMultiWarpBytes;
        prepare_kernel(ctx, kern, smem);
        const int rpw = reuse_rows_per_warp(ctx, kern, smem, rl.count, kMultiWarps);
        const int grid = persistent_grid(ctx, kern, 32 * kMultiWarps, smem, ceil_div(rl.count, kMultiWarps * rpw));
        SPG_LAUNCH(ctx, "k_num_reuse_multi", s,
                   kern<<<grid, 32 * kMultiWarps, smem, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, scale, d_info_num, spec,
                                                            rpw, d_rflag));
      } else {
        auto kern = &k_num_lean<false>;
        const size_t smem = static_cast<size_t>(kLeanGroups) * kLeanGroupBytes;
        prepare_kernel(ctx, kern, smem);
        const int grid = persistent_grid(ctx, kern, 32 * kLeanGroups, smem, ceil_div(rl.count, kLeanGroups));
        SPG_LAUNCH(ctx, "k_num_lean", s,
                   kern<<<grid, 32 * kLeanGroups, smem, s>>>(rl, A, B, d_rpt, d_ccol, d_cval, scale, d_info_num,
                                                            spec));
      }
    } else {
      group(NUMG(32, 256, 4, 8), 32, 256, 4, 8);
    }
  } else if (u <= 256) {
    group(NUMG(32, 512, 8, 8), 32, 512, 8, 8);
  } else if (u <= 512) {
    group(NUMG(32, 1024, 16, 4), 32, 1024, 16, 4);
  } else if (u <= 1024) {
    block(k_num_block<2048, 256, 1024>, 2048, 256, 1024);
  } else if (u <= 2048) {
    block(k_num_block<4096, 256, 2048>, 4096, 256, 2048);
  } else if (u <= 4096) {
    block(k_num_block<8192, 512, 4096>, 8192, 512, 4096);
  } else {
    // B200 tier: rows of 4097..8192 nonzeros (bin 6 of num_1x / num_1.5x, whose
    // reference tier is a fixed table) stay on chip in a 16384-slot table
    block(k_num_block<16384, 1024, 8192, true>, 16384, 1024, 8192, true);
  }
}

void spgemm_pipeline::run_numeric() {
  expect(kRptDone, "run_numeric");
  mark(10);
  // Global (heap) tier pool, sized from the exact max row nnz of pass 1.
  int64_t grows = 0;
  for (int j = 0; j < kNumBins; ++j)
    if (heap_tier(j)) grows += bin_info.bin_size[j];
  int32_t* gkeys = nullptr;
  double* gvals = nullptr;
  uint32_t* gbits = nullptr;
  int64_t gslots = 0, gwords = 0;
  int gblocks = 0;
  if (grows > 0 && !heap_bitmap()) {
    gslots = 2;
    while (gslots < 2 * h_num.max_metric) gslots <<= 1;
    gwords = std::min<int64_t>(int64_t(1) << 17, std::max<int64_t>(1, ceil_div(B.cols, 32)));
    const int64_t per_block = gslots * 12 + gwords * 8;
    const int64_t budget = int64_t(8) << 30;
    gblocks = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>({2LL * ctx->num_sms, grows, budget / per_block})));
    gkeys = static_cast<int32_t*>(dev_alloc(static_cast<size_t>(gslots) * 4 * gblocks, ctx->main_s));
    gvals = static_cast<double*>(dev_alloc(static_cast<size_t>(gslots) * 8 * gblocks, ctx->main_s));
    gbits = static_cast<uint32_t*>(dev_alloc(static_cast<size_t>(gwords) * 8 * gblocks, ctx->main_s));
  }
  // Ordered bitmap tier: B's column panels (one per warp of the row's block),
  // balanced by B's column counts, and every B row's panel boundaries.
  unsigned char* panel_buf = nullptr;
  if (grows > 0 && heap_bitmap() && heap_ordered()) {
    const size_t o_colb = align_up(static_cast<size_t>(kHistBuckets) * 8, 256);
    const size_t o_poff = align_up(o_colb + (kPanels + 1) * 4, 256);
    const size_t bytes = o_poff + static_cast<size_t>(B.rows) * (kPanels + 1) * 4;
    panel_buf = static_cast<unsigned char*>(dev_alloc(bytes, ctx->main_s));
    auto* hist = reinterpret_cast<unsigned long long*>(panel_buf);
    auto* colb = reinterpret_cast<int32_t*>(panel_buf + o_colb);
    d_poff = reinterpret_cast<int32_t*>(panel_buf + o_poff);
    const int64_t bw = std::max<int64_t>(1, ceil_div(B.cols, kHistBuckets));
    ck(cudaMemsetAsync(hist, 0, static_cast<size_t>(kHistBuckets) * 8, ctx->main_s), "memset hist");
    if (b_nnz > 0) {
      const int hg = static_cast<int>(std::min<int64_t>(ctx->num_sms * 4, ceil_div(b_nnz, 256)));
      SPG_LAUNCH(ctx, "k_col_hist", ctx->main_s,
                 k_col_hist<<<std::max(hg, 1), 256, 0, ctx->main_s>>>(B.col, b_nnz, bw, hist));
    }
    SPG_LAUNCH(ctx, "k_panel_bounds", ctx->main_s,
               k_panel_bounds<<<1, 1024, 0, ctx->main_s>>>(hist, bw, B.cols, colb));
    if (B.rows > 0) {
      const int sg = static_cast<int>(std::min<int64_t>(ctx->num_sms * 16, ceil_div(B.rows, 8)));
      SPG_LAUNCH(ctx, "k_panel_split", ctx->main_s,
                 k_panel_split<<<std::max(sg, 1), 256, 0, ctx->main_s>>>(B, colb, d_poff));
    }
  }
  if (spec.flag != nullptr && M > 0) {
    const int grid = static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, ceil_div(M, 256)));
    SPG_LAUNCH(ctx, "k_spec_copy", ctx->main_s,
               k_spec_copy<<<std::max(grid, 1), 256, 0, ctx->main_s>>>(spec, d_rpt, M, d_ccol, d_cval));
  }
  ck(cudaEventRecord(ctx->ev_fork, ctx->main_s), "ev_fork");
  for (int r = 0; r < kNumBins; ++r) {
    const int bin = num_plan.launch_order[r];
    if (bin_info.bin_size[bin] == 0) continue;
    // the heap-tier bins share the k_num_global pool: one stream for them
    const bool heap_bin = heap_tier(bin);
    cudaStream_t s = heap_bin && !heap_bitmap() ? ctx->main_s : bin_stream(ctx, bin);
    ck(cudaStreamWaitEvent(s, ctx->ev_fork, 0), "wait fork");
    RowList rl{d_bins, bin_info.bin_offset[bin], bin_info.bin_size[bin], bin_info.fast_path, nullptr, bin};
    launch_num_bin(bin, rl, s, gkeys, gvals, gbits, gslots, gwords, gblocks);
    ck(cudaEventRecord(ctx->ev_join[bin], s), "ev_join");
    ck(cudaStreamWaitEvent(ctx->main_s, ctx->ev_join[bin], 0), "wait join");
  }
  dev_free(gkeys, ctx->main_s);
  dev_free(gvals, ctx->main_s);
  dev_free(gbits, ctx->main_s);
  dev_free(panel_buf, ctx->main_s);
  d_poff = nullptr;
  mark(11);
  stage = kNumeric;
}

void spgemm_pipeline::finish(spgemm_report* r) {
  expect(kNumeric, "finish");
  info_to_host(d_info_sym, 0, 2, ctx->main_s);
  ck(cudaStreamSynchronize(ctx->main_s), "cudaStreamSynchronize");
  const DevInfo sym = ctx->h_info[0], num = ctx->h_info[1];
  if (std::getenv("SPGEMM_DEBUG_REUSE"))
    std::fprintf(stderr, "reuse: symbolic-phase rows reuse %lld full %lld; numeric rows reuse %lld full %lld\n",
                 sym.reuse_rows, sym.full_rows, num.reuse_rows, num.full_rows);
  if (num.error & kErrScanMismatch)
    fail(SPGEMM_LOGIC_ERROR, "spgemm: exclusive sum disagrees with binning total");
  if (num.error & kErrNumericCount)
    fail(SPGEMM_LOGIC_ERROR, "spgemm: numeric row nnz disagrees with symbolic result");
  spgemm_report rep;
  std::memset(&rep, 0, sizeof(rep));
  rep.rows = M;
  rep.nnz = a_nnz;
  rep.nnz_per_row_mean = M > 0 ? static_cast<double>(a_nnz) / static_cast<double>(M) : 0.0;
  rep.max_nnz_per_row = sym.a_max_row;
  rep.total_nprod = total_nprod;
  rep.nnz_of_product = total_nnz;
  rep.cr = total_nnz > 0 ? static_cast<double>(total_nprod) / static_cast<double>(total_nnz) : 0.0;
  rep.spilled_rows = static_cast<int64_t>(sym.spill_count);
  rep.workers = opts.workers > 0 ? opts.workers : ctx->num_sms;
  rep.timings.setup = span(0, 1);
  rep.timings.sym_binning = span(2, 3);
  rep.timings.symbolic = span(4, 5);
  rep.timings.num_binning = span(6, 7);
  rep.timings.rpt_alloc = span(8, 9);
  rep.timings.numeric = span(10, 11);
  // Cleanup: the metadata arena goes only now, after every kernel of both
  // phases (pipeline.cpp:449-455).
  const auto t0 = std::chrono::steady_clock::now();
  scratch_release(ctx, d_arena);
  d_arena = nullptr;
  rep.timings.cleanup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  rep.timings.total = rep.timings.setup + rep.timings.sym_binning + rep.timings.symbolic +
                      rep.timings.rpt_alloc + rep.timings.num_binning + rep.timings.numeric +
                      rep.timings.cleanup;
  rep.metadata_calls = metadata_calls;
  rep.metadata_bytes = metadata_bytes;
  rep.output_calls = output_calls;
  rep.output_bytes = output_bytes;
  if (r) *r = rep;
  stage = kDone;
}

void spgemm_pipeline::release(bool keep_result) {
  cudaStream_t s = ctx->main_s;
  if (alloc_pending) {
    cudaStreamWaitEvent(s, ctx->ev_side, 0);
    alloc_pending = false;
  }
  for (void*& p : owned) {
    scratch_release(ctx, p);
    p = nullptr;
  }
  scratch_release(ctx, d_arena);
  d_arena = nullptr;
  if (!keep_result) {
    dev_free(d_rpt, s);
    dev_free(d_ccol, s);
    dev_free(d_cval, s);
  }
  d_rpt = nullptr;
  d_ccol = nullptr;
  d_cval = nullptr;
}

// ================================================================= C ABI
extern "C" {

const char* spgemm_last_error(void) { return g_err.c_str(); }

// not in the public header: lets multi.cpp report a worker thread's error on
// the calling thread
void spgemm_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }

void spgemm_options_default(spgemm_options* o) {
  std::memset(o, 0, sizeof(*o));
  std::strncpy(o->sym_preset, "sym_1.2x", sizeof(o->sym_preset) - 1);
  std::strncpy(o->num_preset, "num_2x", sizeof(o->num_preset) - 1);
  o->workers = 0;
  o->overlap = 1;
  o->deterministic = 1;
  o->chunk_rows = 4096;
  o->hash_scale = 107;
}

spgemm_status spgemm_ctx_create(int32_t device, spgemm_ctx** out) {
  *out = nullptr;
  return guard([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(SPGEMM_NO_DEVICE, "no CUDA device visible");
    }
    if (device < 0 || device >= n) fail(SPGEMM_INVALID_ARGUMENT, "device index out of range");
    auto* c = new spgemm_ctx();
    c->device = device;
    try {
      DeviceGuard g(device);
      cudaDeviceProp prop;
      ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
      if (prop.major < 10)
        fail(SPGEMM_NO_DEVICE, "this build targets sm_100a (B200); device is sm_" +
                                   std::to_string(prop.major) + std::to_string(prop.minor));
      c->num_sms = prop.multiProcessorCount;
      c->max_smem = static_cast<int>(prop.sharedMemPerBlockOptin);
      ck(cudaStreamCreateWithFlags(&c->main_s, cudaStreamNonBlocking), "stream");
      ck(cudaStreamCreateWithFlags(&c->side_s, cudaStreamNonBlocking), "stream");
      for (auto& s : c->bin_s) ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
      ck(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&c->ev_info, cudaEventDisableTiming), "event");
      for (auto& e : c->ev_join) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      ck(cudaHostAlloc(&c->h_info, 2 * sizeof(DevInfo), cudaHostAllocMapped | cudaHostAllocPortable),
         "cudaHostAlloc");
      ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_info_dev), c->h_info, 0), "cudaHostGetDevicePointer");
      // A private stream-ordered pool (the device's default pool is left as
      // other users of the process configured it). Freed blocks stay in the
      // pool, so repeated multiplies reuse HBM without returning it to the
      // driver; spgemm_ctx_trim gives it back.
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      ck(cudaMemPoolCreate(&c->pool, &props), "cudaMemPoolCreate");
      uint64_t thresh = std::numeric_limits<uint64_t>::max();
      ck(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thresh), "pool attr");
      // Never make an allocation wait on another stream's free: C freed on the
      // copy lane behind its download must not stall the next product's
      // kernels (the pool takes fresh memory instead).
      int no = 0;
      ck(cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &no), "pool attr");
    } catch (...) {
      spgemm_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

void spgemm_ctx_destroy(spgemm_ctx* c) {
  if (!c) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  if (c->main_s) cudaStreamSynchronize(c->main_s);
  for (auto& s : c->bin_s)
    if (s) cudaStreamDestroy(s);
  if (c->side_s) cudaStreamDestroy(c->side_s);
  if (c->main_s) cudaStreamDestroy(c->main_s);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_side) cudaEventDestroy(c->ev_side);
  if (c->ev_info) cudaEventDestroy(c->ev_info);
  for (auto& e : c->ev_join)
    if (e) cudaEventDestroy(e);
  for (auto& r : c->prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto& e : c->ev_pool) cudaEventDestroy(e);
  for (auto& b : c->scratch) cudaFreeAsync(b.p, 0);
  cudaDeviceSynchronize();
  // (result matrices still alive keep the pool's memory until they are freed)
  if (c->pool) cudaMemPoolDestroy(c->pool);
  if (c->h_info) cudaFreeHost(c->h_info);
  if (prev >= 0) cudaSetDevice(prev);
  delete c;
}

spgemm_status spgemm_ctx_trim(spgemm_ctx* c, uint64_t keep_bytes) {
  return guard([&] {
    DeviceGuard g(c->device);
    ck(cudaStreamSynchronize(c->main_s), "cudaStreamSynchronize");
    ck(cudaStreamSynchronize(c->side_s), "cudaStreamSynchronize");
    std::vector<spgemm_ctx::Scratch> keep;
    for (auto& b : c->scratch) {
      if (b.busy) keep.push_back(b);
      else ck(cudaFreeAsync(b.p, c->main_s), "cudaFreeAsync");
    }
    c->scratch.swap(keep);
    ck(cudaStreamSynchronize(c->main_s), "cudaStreamSynchronize");
    ck(cudaMemPoolTrimTo(c->pool, static_cast<size_t>(keep_bytes)), "cudaMemPoolTrimTo");
  });
}

int32_t spgemm_ctx_device(const spgemm_ctx* c) { return c->device; }
int32_t spgemm_ctx_num_sms(const spgemm_ctx* c) { return c->num_sms; }
int64_t spgemm_ctx_kernel_launches(const spgemm_ctx* c) { return c->launches.load(); }

void spgemm_ctx_set_profiling(spgemm_ctx* c, int32_t on) { c->prof = on != 0; }

spgemm_status spgemm_ctx_pool_stats(spgemm_ctx* c, uint64_t* reserved, uint64_t* used) {
  return guard([&] {
    ck(cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemCurrent, reserved), "pool attr");
    ck(cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrUsedMemCurrent, used), "pool attr");
  });
}

int32_t spgemm_ctx_profile_summary(spgemm_ctx* c, spgemm_kernel_time* out, int32_t max) {
  int32_t n = 0;
  guard([&] {
    DeviceGuard g(c->device);
    ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    std::vector<spgemm_kernel_time> agg;
    for (auto& r : c->prof_recs) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
      auto it = std::find_if(agg.begin(), agg.end(), [&](const spgemm_kernel_time& k) {
        return r.name.compare(0, sizeof(k.name) - 1, k.name) == 0 &&
               std::strlen(k.name) == std::min(r.name.size(), sizeof(k.name) - 1);
      });
      if (it == agg.end()) {
        spgemm_kernel_time k;
        std::memset(&k, 0, sizeof(k));
        std::strncpy(k.name, r.name.c_str(), sizeof(k.name) - 1);
        agg.push_back(k);
        it = agg.end() - 1;
      }
      it->launches += 1;
      it->total_ms += ms;
      c->ev_pool.push_back(r.a);
      c->ev_pool.push_back(r.b);
    }
    c->prof_recs.clear();
    for (const auto& k : agg)
      if (n < max) out[n++] = k;
  });
  return n;
}
void* spgemm_ctx_stream(spgemm_ctx* c) { return c->main_s; }

spgemm_status spgemm_ctx_synchronize(spgemm_ctx* c) {
  return guard([&] {
    DeviceGuard g(c->device);
    ck(cudaStreamSynchronize(c->main_s), "cudaStreamSynchronize");
  });
}

spgemm_status spgemm_preset(int32_t phase, const char* name, spgemm_bin_config* out) {
  return guard([&] {
    if (!name || !find_preset(phase, name, out))
      fail(SPGEMM_INVALID_ARGUMENT,
           std::string("unknown binning preset '") + (name ? name : "(null)") + "'");
  });
}

int32_t spgemm_classify(int64_t value, const spgemm_bin_config* c) { return classify_host(value, *c); }

spgemm_status spgemm_make_plan(const spgemm_bin_config* c, spgemm_plan* out) {
  return guard([&] { make_plan(*c, out); });
}

spgemm_status spgemm_pipeline_create(spgemm_ctx* ctx, const spgemm_csr_view* a,
                                     const spgemm_csr_view* b, const spgemm_options* o,
                                     spgemm_pipeline** out) {
  *out = nullptr;
  return guard([&] {
    auto* p = new spgemm_pipeline();
    try {
      p->ctx = ctx;
      if (o) p->opts = *o;
      else spgemm_options_default(&p->opts);
      spgemm_bin_config sc, nc;
      if (!find_preset(0, p->opts.sym_preset, &sc))
        fail(SPGEMM_INVALID_ARGUMENT,
             std::string("unknown binning preset '") + p->opts.sym_preset + "'");
      if (!find_preset(1, p->opts.num_preset, &nc))
        fail(SPGEMM_INVALID_ARGUMENT,
             std::string("unknown binning preset '") + p->opts.num_preset + "'");
      if (p->opts.hash_scale <= 0 || p->opts.hash_scale % 2 == 0)
        fail(SPGEMM_INVALID_ARGUMENT, "hash_scale must be a positive odd integer");
      p->scale = static_cast<uint32_t>(p->opts.hash_scale);
      make_plan(sc, &p->sym_plan);
      make_plan(nc, &p->num_plan);
      if (a->cols != b->rows)
        fail(SPGEMM_INVALID_ARGUMENT, "spgemm: a.cols (" + std::to_string(a->cols) +
                                          ") != b.rows (" + std::to_string(b->rows) + ")");
      if (p->opts.has_sym_launch_order) apply_launch_order(&p->sym_plan, p->opts.sym_launch_order);
      if (p->opts.has_num_launch_order) apply_launch_order(&p->num_plan, p->opts.num_launch_order);
      p->sym_up = to_upper(sc);
      p->num_up = to_upper(nc);
      DeviceGuard g(ctx->device);
      const bool alias = a->rpt == b->rpt && a->col == b->col && a->val == b->val &&
                         a->rows == b->rows && a->cols == b->cols && a->on_device == b->on_device;
      stage_input(ctx, a, &p->A, p->owned, &p->a_nnz);
      if (alias) {
        p->B = p->A;
        p->b_nnz = p->a_nnz;
      } else {
        stage_input(ctx, b, &p->B, p->owned + 3, &p->b_nnz);
      }
      p->M = a->rows;
      p->b_rows = b->rows;
      for (auto& e : p->ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    } catch (...) {
      spgemm_pipeline_destroy(p);
      throw;
    }
    *out = p;
  });
}

void spgemm_pipeline_destroy(spgemm_pipeline* p) {
  if (!p) return;
  if (p->ctx) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(p->ctx->device);
    p->release(false);
    cudaStreamSynchronize(p->ctx->main_s);
    for (auto& e : p->ev)
      if (e) cudaEventDestroy(e);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete p;
}

#define PIPE_STEP(NAME, CALL)                         \
  spgemm_status NAME(spgemm_pipeline* p) {            \
    return guard([&] {                                \
      DeviceGuard g(p->ctx->device);                  \
      CALL;                                           \
    });                                               \
  }

PIPE_STEP(spgemm_pipeline_setup, p->setup())
PIPE_STEP(spgemm_pipeline_symbolic_binning, p->symbolic_binning())
PIPE_STEP(spgemm_pipeline_run_symbolic, p->run_symbolic())
PIPE_STEP(spgemm_pipeline_numeric_binning, p->numeric_binning())
PIPE_STEP(spgemm_pipeline_run_numeric, p->run_numeric())

spgemm_status spgemm_pipeline_finalize_rpt(spgemm_pipeline* p, int64_t* total) {
  return guard([&] {
    DeviceGuard g(p->ctx->device);
    const int64_t t = p->finalize_rpt();
    if (total) *total = t;
  });
}

spgemm_status spgemm_pipeline_finish(spgemm_pipeline* p, spgemm_report* r) {
  return guard([&] {
    DeviceGuard g(p->ctx->device);
    p->finish(r);
  });
}

spgemm_status spgemm_pipeline_run(spgemm_pipeline* p, spgemm_report* r) {
  return guard([&] {
    DeviceGuard g(p->ctx->device);
    p->setup();
    p->symbolic_binning();
    p->run_symbolic();
    p->numeric_binning();
    p->finalize_rpt(false);
    p->run_numeric();
    p->finish(r);
  });
}

spgemm_status spgemm_pipeline_rpt_region(spgemm_pipeline* p, int64_t* host_out) {
  return guard([&] {
    DeviceGuard g(p->ctx->device);
    if (p->stage == spgemm_pipeline::kNew || !p->d_rpt)
      fail(SPGEMM_LOGIC_ERROR, "spgemm pipeline: rpt_region before setup");
    ck(cudaMemcpyAsync(host_out, p->d_rpt, static_cast<size_t>(p->M) * 8, cudaMemcpyDeviceToHost,
                       p->ctx->main_s),
       "D2H rpt region");
    ck(cudaStreamSynchronize(p->ctx->main_s), "cudaStreamSynchronize");
  });
}

spgemm_status spgemm_pipeline_binning(spgemm_pipeline* p, spgemm_binning_info* info,
                                      int64_t* bins_host) {
  return guard([&] {
    DeviceGuard g(p->ctx->device);
    if (p->sym_bins_on_device && p->stage >= spgemm_pipeline::kSymBinned &&
        p->stage < spgemm_pipeline::kNumBinned && p->d_arena) {
      DevInfo tmp;
      p->fetch_info(p->d_info_sym, &tmp);
      for (int j = 0; j < kNumBins; ++j) {
        p->bin_info.bin_size[j] = tmp.bin_size[j];
        p->bin_info.bin_offset[j] = tmp.bin_offset[j];
      }
    }
    if (info) *info = p->bin_info;
    if (!bins_host || p->M == 0) return;
    if (p->stage < spgemm_pipeline::kSymBinned || !p->d_arena)
      fail(SPGEMM_LOGIC_ERROR, "spgemm pipeline: binning not available at this stage");
    if (p->bin_info.fast_path) {
      SPG_LAUNCH(p->ctx, "k_iota", p->ctx->main_s,
                 k_iota<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(p->M, 256), 4096)), 256, 0,
               p->ctx->main_s>>>(p->d_bins, p->M));
    }
    ck(cudaMemcpyAsync(bins_host, p->d_bins, static_cast<size_t>(p->M) * 8, cudaMemcpyDeviceToHost,
                       p->ctx->main_s),
       "D2H bins");
    ck(cudaStreamSynchronize(p->ctx->main_s), "cudaStreamSynchronize");
  });
}

spgemm_status spgemm_pipeline_plan(spgemm_pipeline* p, int32_t phase, spgemm_plan* out) {
  return guard([&] { *out = phase == 0 ? p->sym_plan : p->num_plan; });
}

spgemm_status spgemm_pipeline_take_result(spgemm_pipeline* p, spgemm_matrix** c) {
  *c = nullptr;
  return guard([&] {
    if (p->stage != spgemm_pipeline::kDone) fail(SPGEMM_LOGIC_ERROR, "take_result before finish");
    if (p->result_taken) fail(SPGEMM_LOGIC_ERROR, "result already taken");
    auto* m = new spgemm_matrix();
    m->ctx = p->ctx;
    m->rows = p->M;
    m->cols = p->B.cols;
    m->nnz = p->total_nnz;
    m->rpt = p->d_rpt;
    m->col = p->d_ccol;
    m->val = p->d_cval;
    p->d_rpt = nullptr;
    p->d_ccol = nullptr;
    p->d_cval = nullptr;
    p->result_taken = true;
    *c = m;
  });
}

spgemm_status spgemm_multiply(spgemm_ctx* ctx, const spgemm_csr_view* a, const spgemm_csr_view* b,
                              const spgemm_options* o, spgemm_matrix** c, spgemm_report* r) {
  spgemm_pipeline* p = nullptr;
  spgemm_status st = spgemm_pipeline_create(ctx, a, b, o, &p);
  if (st != SPGEMM_OK) return st;
  st = spgemm_pipeline_run(p, r);
  if (st == SPGEMM_OK) st = spgemm_pipeline_take_result(p, c);
  std::string keep = g_err;
  spgemm_pipeline_destroy(p);
  g_err = keep;
  return st;
}

void spgemm_matrix_shape(const spgemm_matrix* m, int64_t* rows, int64_t* cols, int64_t* nnz) {
  *rows = m->rows;
  *cols = m->cols;
  *nnz = m->nnz;
}

void spgemm_matrix_device_ptrs(const spgemm_matrix* m, const int64_t** rpt, const int32_t** col,
                               const double** val) {
  *rpt = m->rpt;
  *col = m->col;
  *val = m->val;
}

spgemm_status spgemm_matrix_as_operand(const spgemm_matrix* m, spgemm_csr_view* out) {
  return guard([&] {
    if (!m || !out) fail(SPGEMM_INVALID_ARGUMENT, "spgemm_matrix_as_operand: null argument");
    if (!m->rpt) fail(SPGEMM_INVALID_ARGUMENT, "spgemm_matrix_as_operand: C's buffers were released");
    out->rows = m->rows;
    out->cols = m->cols;
    out->rpt = m->rpt;
    out->col = m->col;
    out->val = m->val;
    out->on_device = 1;
  });
}

spgemm_status spgemm_ctx_wait_stream(spgemm_ctx* ctx, void* stream) {
  return guard([&] {
    if (!ctx) fail(SPGEMM_INVALID_ARGUMENT, "spgemm_ctx_wait_stream: null context");
    DeviceGuard g(ctx->device);
    cudaEvent_t e = pooled_event(ctx);
    ck(cudaEventRecord(e, stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy), "record producer stream");
    ck(cudaStreamWaitEvent(ctx->main_s, e, 0), "context waits for producer stream");
    ctx->ev_pool.push_back(e);
  });
}

spgemm_status spgemm_matrix_download(spgemm_ctx* ctx, const spgemm_matrix* m, int64_t* rpt,
                                     int32_t* col, double* val) {
  return guard([&] {
    DeviceGuard g(ctx->device);
    // on the copy lane, behind the work queued on the context's stream (the
    // product): the compute stream is not held by the transfer
    cudaStream_t cs = ctx->side_s;
    cudaEvent_t ready = pooled_event(ctx);
    ck(cudaEventRecord(ready, ctx->main_s), "record product");
    ck(cudaStreamWaitEvent(cs, ready, 0), "copy lane waits");
    ctx->ev_pool.push_back(ready);
    ck(cudaMemcpyAsync(rpt, m->rpt, static_cast<size_t>(m->rows + 1) * 8, cudaMemcpyDeviceToHost, cs),
       "D2H C.rpt");
    if (m->nnz > 0) {
      ck(cudaMemcpyAsync(col, m->col, static_cast<size_t>(m->nnz) * 4, cudaMemcpyDeviceToHost, cs),
         "D2H C.col");
      ck(cudaMemcpyAsync(val, m->val, static_cast<size_t>(m->nnz) * 8, cudaMemcpyDeviceToHost, cs),
         "D2H C.val");
    }
    ck(cudaStreamSynchronize(cs), "cudaStreamSynchronize(copy lane)");
  });
}

spgemm_status spgemm_matrix_download_async(spgemm_ctx* ctx, spgemm_matrix* m, int64_t* rpt, int32_t* col,
                                           double* val, int32_t release) {
  return guard([&] {
    DeviceGuard g(ctx->device);
    cudaStream_t cs = ctx->side_s;  // the copy lane
    cudaEvent_t ready = pooled_event(ctx);
    ck(cudaEventRecord(ready, ctx->main_s), "record product");
    ck(cudaStreamWaitEvent(cs, ready, 0), "copy lane waits");
    ck(cudaMemcpyAsync(rpt, m->rpt, static_cast<size_t>(m->rows + 1) * 8, cudaMemcpyDeviceToHost, cs),
       "D2H C.rpt");
    if (m->nnz > 0) {
      ck(cudaMemcpyAsync(col, m->col, static_cast<size_t>(m->nnz) * 4, cudaMemcpyDeviceToHost, cs), "D2H C.col");
      ck(cudaMemcpyAsync(val, m->val, static_cast<size_t>(m->nnz) * 8, cudaMemcpyDeviceToHost, cs), "D2H C.val");
    }
    if (release) {
      dev_free(m->rpt, cs);
      dev_free(m->col, cs);
      dev_free(m->val, cs);
      m->rpt = nullptr;
      m->col = nullptr;
      m->val = nullptr;
    } else {
      // C stays owned by the handle: order the context's later work (a free
      // of C included) behind the copy
      cudaEvent_t done = pooled_event(ctx);
      ck(cudaEventRecord(done, cs), "record copy");
      ck(cudaStreamWaitEvent(ctx->main_s, done, 0), "main waits for copy");
      ctx->ev_pool.push_back(done);
    }
    ctx->ev_pool.push_back(ready);  // a wait captures the record it follows, so reuse is safe
  });
}

spgemm_status spgemm_ctx_wait_downloads(spgemm_ctx* ctx) {
  return guard([&] {
    DeviceGuard g(ctx->device);
    ck(cudaStreamSynchronize(ctx->side_s), "cudaStreamSynchronize(copy lane)");
  });
}

spgemm_status spgemm_matrix_checksum(spgemm_ctx* ctx, const spgemm_matrix* m, int64_t row_offset,
                                     int64_t col_offset, double* val_sum, uint64_t* pattern_hash) {
  return guard([&] {
    DeviceGuard g(ctx->device);
    cudaStream_t s = ctx->main_s;
    void* acc = dev_alloc(16, s);
    ck(cudaMemsetAsync(acc, 0, 16, s), "memset checksum");
    double* dv = static_cast<double*>(acc);
    unsigned long long* dh = reinterpret_cast<unsigned long long*>(dv + 1);
    if (m->rows > 0) {
      const int grid = static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, ceil_div(m->rows, 8)));
      SPG_LAUNCH(ctx, "k_checksum", s,
                 k_checksum<<<std::max(grid, 1), 256, 0, s>>>(m->rpt, m->col, m->val, m->rows, row_offset,
                                                              col_offset, dv, dh));
    }
    double hv[2];
    ck(cudaMemcpyAsync(hv, acc, 16, cudaMemcpyDeviceToHost, s), "D2H checksum");
    dev_free(acc, s);
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    *val_sum = hv[0];
    std::memcpy(pattern_hash, &hv[1], 8);
  });
}

void spgemm_matrix_free(spgemm_matrix* m) {
  if (!m) return;
  if (m->ctx) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(m->ctx->device);
    dev_free(m->rpt, m->ctx->main_s);
    dev_free(m->col, m->ctx->main_s);
    dev_free(m->val, m->ctx->main_s);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete m;
}

spgemm_status spgemm_compute_nprod(spgemm_ctx* ctx, const spgemm_csr_view* a,
                                   const spgemm_csr_view* b, int64_t* out_host, int64_t* total) {
  spgemm_pipeline* p = nullptr;
  spgemm_status st = spgemm_pipeline_create(ctx, a, b, nullptr, &p);
  if (st != SPGEMM_OK) return st;
  st = spgemm_pipeline_setup(p);
  if (st == SPGEMM_OK && out_host) st = spgemm_pipeline_rpt_region(p, out_host);
  if (st == SPGEMM_OK && total) *total = p->total_nprod;
  std::string keep = g_err;
  spgemm_pipeline_destroy(p);
  g_err = keep;
  return st;
}

spgemm_status spgemm_multiply_into(spgemm_ctx* ctx, const spgemm_csr_view* a, const spgemm_csr_view* b,
                                   const spgemm_options* opts, int32_t parts, int64_t* rpt, int64_t capacity,
                                   int32_t* col, double* val, int64_t* nnz_out, spgemm_report* report) {
  std::vector<void*> staged;
  std::vector<spgemm_matrix*> pending;
  auto cleanup = [&] {
    for (spgemm_matrix* m : pending) spgemm_matrix_free(m);
    cudaStreamSynchronize(ctx->side_s);
    for (void* p : staged) scratch_release(ctx, p);
  };
  const spgemm_status st = guard([&] {
    DeviceGuard g(ctx->device);
    if (!a || !b || !rpt || (capacity > 0 && (!col || !val)))
      fail(SPGEMM_INVALID_ARGUMENT, "spgemm_multiply_into: null argument");
    if (a->on_device || b->on_device)
      fail(SPGEMM_INVALID_ARGUMENT, "spgemm_multiply_into: operands must be host-resident");
    if (a->cols != b->rows)
      fail(SPGEMM_INVALID_ARGUMENT, "spgemm: a.cols (" + std::to_string(a->cols) + ") != b.rows (" +
                                        std::to_string(b->rows) + ")");
    // 1. stage A and B once (B aliasing A is staged once)
    DevCsr da{}, db{};
    void* own[3] = {nullptr, nullptr, nullptr};
    int64_t a_nnz = 0, b_nnz = 0;
    stage_input(ctx, a, &da, own, &a_nnz);
    staged.insert(staged.end(), own, own + 3);
    const bool alias = a->rpt == b->rpt && a->col == b->col && a->val == b->val && a->rows == b->rows;
    if (alias) {
      db = da;
      b_nnz = a_nnz;
    } else {
      void* ownb[3] = {nullptr, nullptr, nullptr};
      stage_input(ctx, b, &db, ownb, &b_nnz);
      staged.insert(staged.end(), ownb, ownb + 3);
    }
    const spgemm_csr_view vb{b->rows, b->cols, db.rpt, db.col, db.val, 1};
    // 2. the block split: equal shares of A's nonzeros, from the host row
    // pointers (no device round trip); the block count from the estimated size
    // of C (nnz(A) x mean B row length products)
    const int64_t M = a->rows;
    if (parts <= 0) {  // ~1.5 GB of (upper-bound) C per block, at most 8 blocks
      const double est = static_cast<double>(a_nnz) * (b->rows > 0 ? static_cast<double>(b_nnz) / b->rows : 0.0) * 12.0;
      parts = static_cast<int32_t>(std::min(8.0, std::max(1.0, est / (1536.0 * (1 << 20)))));
    }
    parts = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(parts, std::max<int64_t>(M, 1))));
    std::vector<int64_t> bounds(static_cast<size_t>(parts) + 1, 0);
    for (int32_t g2 = 1; g2 < parts; ++g2) {
      const int64_t target = static_cast<int64_t>((static_cast<__int128>(a_nnz) * g2) / parts);
      const int64_t* it = std::lower_bound(a->rpt, a->rpt + M + 1, target);
      bounds[static_cast<size_t>(g2)] =
          std::max(bounds[static_cast<size_t>(g2) - 1], std::min<int64_t>(M, static_cast<int64_t>(it - a->rpt)));
    }
    bounds[static_cast<size_t>(parts)] = M;
    // 3. blocks in order; block i's download overlaps block i+1's kernels
    const bool dbg = std::getenv("SPGEMM_INTO_DEBUG") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto ms_since = [&] {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    };
    int64_t* brpt = static_cast<int64_t*>(scratch_acquire(ctx, static_cast<size_t>(M + 1) * 8, ctx->main_s));
    staged.push_back(brpt);
    int64_t off = 0;
    spgemm_report combined{};
    bool first = true;
    for (int32_t i = 0; i < parts; ++i) {
      const int64_t r0 = bounds[static_cast<size_t>(i)], r1 = bounds[static_cast<size_t>(i) + 1];
      if (r1 == r0 && !(M == 0 && i == 0)) continue;
      // the block's row pointers, rebased to start at 0
      const int64_t p0 = a->rpt[r0];
      if (r1 > r0 || M == 0) {
        const int64_t n = r1 - r0 + 1;
        const int grid = static_cast<int>(std::min<int64_t>(ctx->num_sms * 4, ceil_div(n, 256)));
        k_add_offset<<<std::max(grid, 1), 256, 0, ctx->main_s>>>(brpt + r0, da.rpt + r0, n, -p0);
        ck(cudaGetLastError(), "k_add_offset");
        ctx->launches.fetch_add(1);
      }
      const spgemm_csr_view blk{r1 - r0, a->cols, brpt + r0, da.col ? da.col + p0 : nullptr,
                                da.val ? da.val + p0 : nullptr, 1};
      spgemm_matrix* m = nullptr;
      spgemm_report rep{};
      g_inputs_stream_ordered = true;
      const spgemm_status s2 = spgemm_multiply(ctx, &blk, &vb, opts, &m, &rep);
      g_inputs_stream_ordered = false;
      if (s2 != SPGEMM_OK) fail(s2, g_err);
      pending.push_back(m);
      if (off + m->nnz > capacity)
        fail(SPGEMM_INVALID_ARGUMENT, "spgemm_multiply_into: C has more than the " + std::to_string(capacity) +
                                          " entries the output buffers hold");
      if (off != 0 && m->rows + 1 > 0) {
        const int grid = static_cast<int>(std::min<int64_t>(ctx->num_sms * 4, ceil_div(m->rows + 1, 256)));
        k_add_offset<<<std::max(grid, 1), 256, 0, ctx->main_s>>>(m->rpt, m->rpt, m->rows + 1, off);
        ck(cudaGetLastError(), "k_add_offset");
        ctx->launches.fetch_add(1);
      }
      const spgemm_status s3 =
          spgemm_matrix_download_async(ctx, m, rpt + r0, col ? col + off : nullptr, val ? val + off : nullptr, 1);
      if (s3 != SPGEMM_OK) fail(s3, g_err);
      off += m->nnz;
      if (dbg) std::fprintf(stderr, "into: block %d rows [%lld,%lld) nnz %lld issued at %.2f ms\n", i,
                            static_cast<long long>(r0), static_cast<long long>(r1), static_cast<long long>(m->nnz),
                            ms_since());
      if (first) {
        combined = rep;
        first = false;
      } else {
        combined.total_nprod += rep.total_nprod;
        combined.spilled_rows += rep.spilled_rows;
        combined.max_nnz_per_row = std::max(combined.max_nnz_per_row, rep.max_nnz_per_row);
        combined.timings.total += rep.timings.total;
        combined.metadata_calls += rep.metadata_calls;
        combined.metadata_bytes += rep.metadata_bytes;
        combined.output_calls += rep.output_calls;
        combined.output_bytes += rep.output_bytes;
      }
    }
    ck(cudaStreamSynchronize(ctx->side_s), "cudaStreamSynchronize(copy lane)");
    if (dbg) std::fprintf(stderr, "into: downloads done at %.2f ms\n", ms_since());
    if (M == 0) rpt[0] = 0;
    for (spgemm_matrix* m : pending) spgemm_matrix_free(m);
    pending.clear();
    combined.rows = M;
    combined.nnz = a_nnz;
    combined.nnz_per_row_mean = M > 0 ? static_cast<double>(a_nnz) / static_cast<double>(M) : 0.0;
    combined.nnz_of_product = off;
    combined.cr = off > 0 ? static_cast<double>(combined.total_nprod) / static_cast<double>(off) : 0.0;
    if (nnz_out) *nnz_out = off;
    if (report) *report = combined;
  });
  cleanup();
  return st;
}

spgemm_status spgemm_forecast_nnz(spgemm_ctx* ctx, const spgemm_csr_view* a, const spgemm_csr_view* b,
                                  const spgemm_options* opts, int64_t* row_nnz, int64_t* total_nnz,
                                  int64_t* total_nprod) {
  spgemm_pipeline* p = nullptr;
  spgemm_status st = spgemm_pipeline_create(ctx, a, b, opts, &p);
  if (st != SPGEMM_OK) return st;
  st = guard([&] {
    DeviceGuard g(p->ctx->device);
    p->symbolic_only = true;
    p->setup();
    p->symbolic_binning();
    p->run_symbolic();
    // per-row counts are in the C.rpt block now; the numeric pass 1 sums them
    // on the device (no C allocation when symbolic_only)
    if (row_nnz && p->M > 0)
      ck(cudaMemcpyAsync(row_nnz, p->d_rpt, static_cast<size_t>(p->M) * 8, cudaMemcpyDeviceToHost,
                         p->ctx->main_s),
         "D2H row nnz");
    p->numeric_binning();
    ck(cudaStreamSynchronize(p->ctx->main_s), "cudaStreamSynchronize");
    if (total_nnz) *total_nnz = p->total_nnz;
    if (total_nprod) *total_nprod = p->total_nprod;
  });
  std::string keep = g_err;
  spgemm_pipeline_destroy(p);
  g_err = keep;
  return st;
}

// csr_from_coo (csr.cpp:12-72) on the device (kernels_coo.cuh).
spgemm_status spgemm_csr_from_coo(spgemm_ctx* ctx, int64_t rows, int64_t cols, int64_t n, const int64_t* row,
                                  const int64_t* col, const double* val, int32_t on_device, spgemm_matrix** out) {
  return guard([&] {
    if (!ctx || !out) fail(SPGEMM_INVALID_ARGUMENT, "csr_from_coo: null argument");
    *out = nullptr;
    if (rows < 0 || cols < 0) fail(SPGEMM_INVALID_ARGUMENT, "csr_from_coo: negative matrix shape");
    if (cols > std::numeric_limits<int32_t>::max())
      fail(SPGEMM_INVALID_ARGUMENT, "csr_from_coo: column count exceeds 32-bit index range");
    if (n < 0 || n >= (int64_t(1) << 32)) fail(SPGEMM_INVALID_ARGUMENT, "csr_from_coo: entry count out of range");
    if (n > 0 && (!row || !col || !val)) fail(SPGEMM_INVALID_ARGUMENT, "csr_from_coo: null triples");
    DeviceGuard g(ctx->device);
    cudaStream_t s = ctx->main_s;
    std::vector<void*> tmp;
    auto scratch = [&](size_t bytes) {
      void* p = dev_alloc(bytes, s);
      tmp.push_back(p);
      return p;
    };
    struct Cleanup {
      std::vector<void*>* t;
      cudaStream_t s;
      ~Cleanup() {
        for (void* p : *t) dev_free(p, s);
      }
    } cleanup{&tmp, s};
    const int64_t* drow = row;
    const int64_t* dcol = col;
    const double* dval = val;
    if (!on_device && n > 0) {
      auto* r = static_cast<int64_t*>(scratch(static_cast<size_t>(n) * 8));
      auto* c = static_cast<int64_t*>(scratch(static_cast<size_t>(n) * 8));
      auto* v = static_cast<double*>(scratch(static_cast<size_t>(n) * 8));
      ck(cudaMemcpyAsync(r, row, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s), "H2D row");
      ck(cudaMemcpyAsync(c, col, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s), "H2D col");
      ck(cudaMemcpyAsync(v, val, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s), "H2D val");
      drow = r;
      dcol = c;
      dval = v;
    } else if (on_device) {
      cudaEvent_t e = pooled_event(ctx);
      ck(cudaEventRecord(e, cudaStreamLegacy), "record default stream");
      ck(cudaStreamWaitEvent(s, e, 0), "wait default stream");
      ctx->ev_pool.push_back(e);
    }
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 8, ceil_div(n, 256))));
    // shape check: the first offending entry, reported like the reference
    auto* bad = static_cast<unsigned long long*>(scratch(8));
    ck(cudaMemsetAsync(bad, 0xff, 8, s), "memset");
    if (n > 0) {
      SPG_LAUNCH(ctx, "k_coo_check", s, k_coo_check<<<grid, 256, 0, s>>>(drow, dcol, n, rows, cols, bad));
    }
    unsigned long long hbad = ~0ull;
    ck(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    if (hbad != ~0ull) {
      int64_t br = 0, bc = 0;
      ck(cudaMemcpy(&br, drow + hbad, 8, cudaMemcpyDeviceToHost), "D2H");
      ck(cudaMemcpy(&bc, dcol + hbad, 8, cudaMemcpyDeviceToHost), "D2H");
      fail(SPGEMM_INVALID_ARGUMENT, "csr_from_coo: entry (" + std::to_string(br) + ", " + std::to_string(bc) +
                                        ") outside " + std::to_string(rows) + "x" + std::to_string(cols) + " shape");
    }
    // two stable counting sorts: by column, then by row
    auto* perm_a = static_cast<uint32_t*>(scratch(static_cast<size_t>(std::max<int64_t>(n, 1)) * 4));
    auto* perm_b = static_cast<uint32_t*>(scratch(static_cast<size_t>(std::max<int64_t>(n, 1)) * 4));
    const int64_t ntile = ceil_div(n, kCooTile);
    auto* done = static_cast<int*>(scratch(static_cast<size_t>(std::max<int64_t>(ntile, 1)) * 4 + 64));
    auto* info = static_cast<DevInfo*>(scratch(sizeof(DevInfo)));
    auto scan = [&](int64_t* data, int64_t len) {  // exclusive, in place
      const int64_t nt = ceil_div(len, kScanTile);
      auto* flags = static_cast<int*>(scratch(static_cast<size_t>(nt) * 4));
      auto* sums = static_cast<long long*>(scratch(static_cast<size_t>(nt) * 16));
      ck(cudaMemsetAsync(flags, 0, static_cast<size_t>(nt) * 4, s), "memset");
      ck(cudaMemsetAsync(info, 0, sizeof(DevInfo), s), "memset");
      SPG_LAUNCH(ctx, "k_scan", s,
                 k_scan<<<static_cast<unsigned>(nt), kScanThreads, 0, s>>>(data, len, flags, sums, sums + nt, info));
    };
    auto pass = [&](const int64_t* key, int64_t nkeys, const uint32_t* pin, uint32_t* pout) {
      auto* cnt = static_cast<int64_t*>(scratch(static_cast<size_t>(nkeys + 1) * 8));
      ck(cudaMemsetAsync(cnt, 0, static_cast<size_t>(nkeys + 1) * 8, s), "memset");
      SPG_LAUNCH(ctx, "k_coo_count", s,
                 k_coo_count<<<grid, 256, 0, s>>>(key, n, reinterpret_cast<unsigned long long*>(cnt)));
      scan(cnt, nkeys + 1);
      ck(cudaMemsetAsync(done, 0, static_cast<size_t>(ntile) * 4 + 64, s), "memset");
      int* tiles = done + ntile;
      SPG_LAUNCH(ctx, "k_coo_scatter", s,
                 k_coo_scatter<<<static_cast<unsigned>(ntile), kCooThreads, 0, s>>>(
                     key, pin, n, reinterpret_cast<long long*>(cnt), done, tiles, pout));
    };
    auto* m = new spgemm_matrix();
    m->ctx = ctx;
    m->rows = rows;
    m->cols = cols;
    try {
      m->rpt = static_cast<int64_t*>(dev_alloc(static_cast<size_t>(rows + 1) * 8, s));
      ck(cudaMemsetAsync(m->rpt, 0, static_cast<size_t>(rows + 1) * 8, s), "memset");
      int64_t nnz = 0;
      if (n > 0) {
        pass(dcol, cols, nullptr, perm_a);
        pass(drow, rows, perm_a, perm_b);
        auto* head = static_cast<int64_t*>(scratch(static_cast<size_t>(n + 1) * 8));
        ck(cudaMemsetAsync(head + n, 0, 8, s), "memset");
        SPG_LAUNCH(ctx, "k_coo_heads", s,
                   k_coo_heads<<<grid, 256, 0, s>>>(drow, dcol, perm_b, n, head,
                                                   reinterpret_cast<unsigned long long*>(m->rpt)));
        scan(head, n + 1);  // head -> compacted index of each run head; total = nnz
        scan(m->rpt, rows + 1);
        ck(cudaMemcpyAsync(&nnz, head + n, 8, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
        m->col = static_cast<int32_t*>(dev_alloc(static_cast<size_t>(std::max<int64_t>(nnz, 1)) * 4, s));
        m->val = static_cast<double*>(dev_alloc(static_cast<size_t>(std::max<int64_t>(nnz, 1)) * 8, s));
        SPG_LAUNCH(ctx, "k_coo_fold", s,
                   k_coo_fold<<<grid, 256, 0, s>>>(drow, dcol, dval, perm_b, n, head, m->col, m->val));
      }
      m->nnz = nnz;
      ck(cudaStreamSynchronize(s), "sync");
    } catch (...) {
      spgemm_matrix_free(m);
      throw;
    }
    *out = m;
  });
}

spgemm_status spgemm_build_rpt(spgemm_ctx* ctx, int64_t* values, int64_t n, int64_t* total) {
  return guard([&] {
    DeviceGuard g(ctx->device);
    if (n <= 0) {
      if (total) *total = 0;
      return;
    }
    cudaStream_t s = ctx->main_s;
    const int64_t ntiles = ceil_div(n, kScanTile);
    auto* d = static_cast<int64_t*>(dev_alloc(static_cast<size_t>(n) * 8, s));
    auto* flags = static_cast<int*>(dev_alloc(static_cast<size_t>(ntiles) * 4, s));
    auto* sums = static_cast<long long*>(dev_alloc(static_cast<size_t>(ntiles) * 16, s));
    auto* info = static_cast<DevInfo*>(dev_alloc(sizeof(DevInfo), s));
    ck(cudaMemcpyAsync(d, values, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s), "H2D");
    ck(cudaMemsetAsync(flags, 0, static_cast<size_t>(ntiles) * 4, s), "memset");
    ck(cudaMemsetAsync(info, 0, sizeof(DevInfo), s), "memset");
    SPG_LAUNCH(ctx, "k_scan", s,
               k_scan<<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(d, n, flags, sums, sums + ntiles, info));
    ck(cudaMemcpyAsync(values, d, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaMemcpyAsync(ctx->h_info, info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    if (total) *total = ctx->h_info->scan_total;
    dev_free(d, s);
    dev_free(flags, s);
    dev_free(sums, s);
    dev_free(info, s);
  });
}

spgemm_status spgemm_run_binning(spgemm_ctx* ctx, const int64_t* metric, int64_t m,
                                 const spgemm_bin_config* cfg, int32_t deterministic,
                                 int64_t* bins_host, spgemm_binning_info* out) {
  (void)deterministic;  // the device scatter is stable in both modes
  return guard([&] {
    DeviceGuard g(ctx->device);
    if (m < 0) fail(SPGEMM_INVALID_ARGUMENT, "run_binning: bad storage sizes");
    spgemm_binning_info bi;
    std::memset(&bi, 0, sizeof(bi));
    if (m == 0) {
      bi.fast_path = 1;
      if (out) *out = bi;
      return;
    }
    cudaStream_t s = ctx->main_s;
    const BinUpper up = to_upper(*cfg);
    const int64_t nrb = ceil_div(m, kRowsPerBlock);
    auto* d_metric = static_cast<int64_t*>(dev_alloc(static_cast<size_t>(m) * 8, s));
    auto* d_bins = static_cast<int64_t*>(dev_alloc(static_cast<size_t>(m) * 8, s));
    auto* d_blk = static_cast<int32_t*>(dev_alloc(static_cast<size_t>(nrb) * kNumBins * 4, s));
    auto* d_info = static_cast<DevInfo*>(dev_alloc(sizeof(DevInfo), s));
    ck(cudaMemcpyAsync(d_metric, metric, static_cast<size_t>(m) * 8, cudaMemcpyHostToDevice, s), "H2D");
    ck(cudaMemsetAsync(d_info, 0, sizeof(DevInfo), s), "memset");
    SPG_LAUNCH(ctx, "k_pass1", s,
               k_pass1<<<static_cast<unsigned>(nrb), kBinThreads, 0, s>>>(d_metric, m, up, d_blk, d_info));
    SPG_LAUNCH(ctx, "k_bin_offsets", s,
               k_bin_offsets<<<1, 1024, 0, s>>>(d_blk, nrb, m, up.u[0], d_info));
    SPG_LAUNCH(ctx, "k_bin_scatter", s,
               k_bin_scatter<<<static_cast<unsigned>(nrb), kBinThreads, 0, s>>>(d_metric, m, up, d_blk, d_bins,
                                                                      d_info));
    ck(cudaMemcpyAsync(ctx->h_info, d_info, sizeof(DevInfo), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    const DevInfo hi = *ctx->h_info;
    if (hi.fast_path) {
      SPG_LAUNCH(ctx, "k_iota", s,
                 k_iota<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(m, 256), 4096)), 256, 0, s>>>(d_bins, m));
    }
    ck(cudaMemcpyAsync(bins_host, d_bins, static_cast<size_t>(m) * 8, cudaMemcpyDeviceToHost, s), "D2H bins");
    ck(cudaStreamSynchronize(s), "sync");
    for (int j = 0; j < kNumBins; ++j) {
      bi.bin_size[j] = hi.bin_size[j];
      bi.bin_offset[j] = hi.bin_offset[j];
    }
    bi.max_metric = hi.max_metric;
    bi.total_metric = static_cast<int64_t>(hi.total);
    bi.fast_path = hi.fast_path;
    if (out) *out = bi;
    dev_free(d_metric, s);
    dev_free(d_bins, s);
    dev_free(d_blk, s);
    dev_free(d_info, s);
  });
}

}  // extern "C"
