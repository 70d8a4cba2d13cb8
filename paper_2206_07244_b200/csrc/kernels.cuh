// kernels.cuh -- sm_100a kernels of the B200-native OpSparse SpGEMM.
//
// Reference semantics (paths relative to /root/reference/proj/core):
//   K1  k_setup_nprod   pipeline.cpp:178-191 (nprod_chunk) + binning.cpp:84-115 (pass 1), fused
//   K2  k_pass1         binning.cpp:84-115 (binning_pass1) over a device metric
//   K3  k_bin_offsets   binning.cpp:304-305 + the per-chunk reservation of binning.cpp:205-229
//   K3  k_bin_scatter   binning.cpp:176-242 (deterministic pass 2: a stable partition by bin)
//   K5  k_scan          binning.cpp:117-168 (exclusive_sum_inplace) / pipeline.cpp:104-107
//   K6  k_sym_group / k_sym_block / k_sym_spill
//                       pipeline.cpp:364-379 -> hash_tables.cpp:94-111 (symbolic_row),
//                       hash_tables.hpp:62-84 (single-access insert), spill pipeline.cpp:315-348
//   K7  k_num_group / k_num_block / k_num_global
//                       pipeline.cpp:380-418 -> hash_tables.cpp:179-201 (numeric_row),
//                       hash_tables.cpp:125-177 (condense + sort), heap tier pipeline.cpp:396-410
//
// Value parity. The reference folds the products of output entry (i, c) as
// ((0.0 + a[i,p0]*b[p0,c]) + a[i,p1]*b[p1,c]) + ... in A-row order
// (hash_tables.cpp:182-193, reference.cpp:21-27), with separate multiply and
// add. Every numeric kernel here walks the A row in order ("ordered steps":
// one A entry per step, the lanes of the row's group stride the B row, whose
// columns are distinct, so no two lanes touch the same slot within a step),
// orders steps with a group/block barrier, and uses __dmul_rn/__dadd_rn (no FMA
// contraction). The result is bitwise the reference's, independent of bin,
// preset, launch order or kernel choice.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spgemm_b200 {

constexpr int kNumBins = 8;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kBinThreads = 256;                       // binning / pass-1 blocks
constexpr int kRowsPerThread = 8;
constexpr int kRowsPerBlock = kBinThreads * kRowsPerThread;  // 2048 rows per row block
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

struct DevCsr {
  int64_t rows;
  int64_t cols;
  const int64_t* __restrict__ rpt;
  const int32_t* __restrict__ col;
  const double* __restrict__ val;
};

struct BinUpper {
  long long u[kNumBins];
};

// Device-side scalars of one phase; lives in the metadata arena.
struct DevInfo {
  unsigned long long total;      // pass-1 metric total
  long long max_metric;          // pass-1 max
  long long bin_size[kNumBins];
  long long bin_offset[kNumBins];
  int fast_path;
  int error;                     // bit 0: numeric count mismatch; bit 1: misbinned
  unsigned long long spill_count;
  long long scan_total;
  long long a_max_row;           // max nnz per A row (input_stats)
  long long a_nnz, b_nnz;        // A.rpt[M], B.rpt[B.rows] (device operands: read by K1)
  int tile_counter;
  int pad_;
  long long b_max_row;           // longest B row any A entry refers to (K1)
  long long reuse_rows, full_rows;  // k_num_reuse: rows through the reuse / full path
};

constexpr int kErrNumericCount = 1;
constexpr int kErrTableFull = 2;
constexpr int kErrScanMismatch = 4;

// Rows of one bin: either the identity (fast path) or a segment of bins[].
struct RowList {
  const int64_t* __restrict__ bins;
  long long offset;
  long long count;
  int identity;
  // When set, offset/count/identity are read from the phase's device-side
  // binning result instead (no host round trip between binning and launch).
  const DevInfo* dev;
  int bin;
  __device__ __forceinline__ int64_t row(int64_t idx) const {
    return identity ? idx : bins[offset + idx];
  }
  __device__ __forceinline__ RowList resolved() const;
};

__device__ __forceinline__ RowList RowList::resolved() const {
  RowList r = *this;
  if (dev) {
    r.identity = dev->fast_path;
    r.count = dev->bin_size[bin];
    r.offset = dev->bin_offset[bin];
  }
  return r;
}


// Speculative numeric during the symbolic phase. Rows of the warp-group
// symbolic bins are multiplied outright (ordered, exactly as the numeric
// kernels do) into a scratch of `cap` entries per row; the row's count goes to
// rpt like the symbolic kernel's and `flag` marks it done, so the symbolic
// kernel skips it and the numeric phase only copies it into C. A row with more
// than `cap` distinct columns is abandoned (flag stays 0) and counted by the
// symbolic kernel as usual. The symbolic walk (~1/3 of the stencil step) is
// saved for every row that fits.
constexpr int kSpecCap = 128;  // entries per row of the speculative scratch

struct Spec {
  int32_t* col;   // [rows * cap]
  double* val;    // [rows * cap]
  uint8_t* flag;  // [rows], zeroed before the symbolic phase
  int cap;
  __device__ __forceinline__ bool done(int64_t row) const { return flag != nullptr && flag[row] != 0; }
};

__device__ __forceinline__ int classify_bin(long long v, const BinUpper& up) {
  int j = 0;
#pragma unroll
  for (int b = kNumBins - 2; b >= 0; --b) j += v > up.u[b] ? 1 : 0;
  return j;  // upper[] is strictly increasing, so this is the smallest j with v <= upper[j]
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) {
    return kFull;
  } else {
    const unsigned lane = threadIdx.x & 31u;
    return ((1u << G) - 1u) << (lane & ~(G - 1u));
  }
}

template <int G>
__device__ __forceinline__ int group_sum(int v, unsigned gm) {
  if constexpr (G == 32) {
    return static_cast<int>(__reduce_add_sync(gm, static_cast<unsigned>(v)));  // one REDUX
  } else {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gm, v, o, G);
    return v;
  }
}

// ------------------------------------------------------------ hash tables
// Open addressing with linear probing over a pow2 table of 2^lg slots. The home
// slot takes the HIGH lg bits of key*scale*phi (Fibonacci hashing): the
// reference's key*scale & (t-1) (hash_tables.hpp:54-57) keeps only the low
// bits, so stencil columns that differ by a multiple of 2^lg (every y/z plane
// of a grid) share one probe chain. The slot a key lands in never affects the
// result (only the probe count), and hash_scale is still the odd multiplier
// the reference validates. The plain read doubles as the claim check
// (hash_tables.hpp:66-83): a slot that holds a key never changes
// again, so only an empty slot needs the atomicCAS.
struct Hash {
  uint32_t mult;   // scale * 0x9E3779B1 (odd)
  uint32_t shift;  // 32 - lg
  uint32_t mask;   // 2^lg - 1
  __device__ __forceinline__ uint32_t home(int32_t key) const {
    return (static_cast<uint32_t>(key) * mult) >> shift;
  }
};

__device__ __forceinline__ Hash make_hash(uint32_t scale, int lg) {
  Hash h;
  h.mult = scale * 0x9E3779B1u;
  h.shift = 32u - static_cast<uint32_t>(lg);
  h.mask = lg >= 32 ? 0xffffffffu : ((1u << lg) - 1u);
  if (lg == 0) h.shift = 31u, h.mask = 0u;
  return h;
}

template <int T>
__host__ __device__ constexpr int log2_const() {
  int l = 0;
  while ((1 << l) < T) ++l;
  return l;
}

template <typename Slot>
__device__ __forceinline__ int sym_insert_slow(Slot* tab, int32_t key, const Hash& hs, uint32_t h,
                                            int32_t cur) {
  while (true) {
    if (cur == key) return 0;
    if (cur == -1) {
      cur = atomicCAS(reinterpret_cast<int*>(tab + h), -1, key);
      if (cur == -1) return 1;
      if (cur == key) return 0;
    }
    h = (h + 1) & hs.mask;
    cur = *reinterpret_cast<volatile int32_t*>(tab + h);
  }
}

// Common case first: one read of the home slot; only a miss (empty slot to
// claim, or a collision) leaves the straight-line path.
template <typename Slot>
__device__ __forceinline__ int sym_insert(Slot* tab, int32_t key, const Hash& hs) {
  const uint32_t h = hs.home(key) & hs.mask;
  const int32_t cur = *reinterpret_cast<volatile int32_t*>(tab + h);
  if (cur == key) return 0;
  return sym_insert_slow(tab, key, hs, h, cur);
}

// Probing after a first-probe miss. `claims` (may be null) counts this lane's
// new keys -- the speculative numeric's budget, summed over the group per step.
__device__ __forceinline__ uint32_t num_slot_slow(int32_t* keys, int32_t key, const Hash& hs, uint32_t h,
                                               int32_t cur, int* claims = nullptr) {
  while (true) {
    if (cur == key) return h;
    if (cur == -1) {
      cur = atomicCAS(reinterpret_cast<int*>(keys + h), -1, key);
      if (cur == -1) {
        if (claims) ++*claims;
        return h;
      }
      if (cur == key) return h;
    }
    h = (h + 1) & hs.mask;
    cur = *reinterpret_cast<volatile int32_t*>(keys + h);
  }
}

__device__ __forceinline__ uint32_t num_slot(int32_t* keys, int32_t key, const Hash& hs) {
  const uint32_t h = hs.home(key) & hs.mask;
  const int32_t cur = *reinterpret_cast<volatile int32_t*>(keys + h);
  if (cur == key) return h;
  return num_slot_slow(keys, key, hs, h, cur);
}

// Batched lookups: the V first-probe reads are issued back to back (a plain
// read is safe: an occupied slot never changes), and only misses take the
// probing loop. Invalid entries (key < 0) count as hits.
template <int V>
__device__ __forceinline__ int sym_insert_batch(int32_t* tab, const int32_t (&key)[V], const Hash& hs) {
  uint32_t h[V];
  int32_t cur[V];
#pragma unroll
  for (int v = 0; v < V; ++v) h[v] = hs.home(key[v]) & hs.mask;
#pragma unroll
  for (int v = 0; v < V; ++v) cur[v] = key[v] >= 0 ? tab[h[v]] : key[v];
  int n = 0;
#pragma unroll
  for (int v = 0; v < V; ++v)
    if (cur[v] != key[v]) n += sym_insert_slow(tab, key[v], hs, h[v], cur[v]);
  return n;
}

// Slot of each key (claimed if new); invalid entries (key < 0) get `dummy`.
template <int V>
__device__ __forceinline__ void num_slot_batch(int32_t* keys, const int32_t (&key)[V], const Hash& hs,
                                               uint32_t dummy, uint32_t (&slot)[V], int* claims = nullptr) {
  int32_t cur[V];
#pragma unroll
  for (int v = 0; v < V; ++v) slot[v] = hs.home(key[v]) & hs.mask;
#pragma unroll
  for (int v = 0; v < V; ++v) cur[v] = key[v] >= 0 ? keys[slot[v]] : key[v];
  // empty home slots: the V claims are issued back to back (straight-line,
  // predicated) before any probing loop
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (key[v] >= 0 && cur[v] == -1) {
      cur[v] = atomicCAS(reinterpret_cast<int*>(keys + slot[v]), -1, key[v]);
      if (cur[v] == -1) {
        cur[v] = key[v];
        if (claims) ++*claims;
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (key[v] < 0) slot[v] = dummy;
    else if (cur[v] != key[v])
      slot[v] = num_slot_slow(keys, key[v], hs, (slot[v] + 1) & hs.mask,
                              *reinterpret_cast<volatile int32_t*>(keys + ((slot[v] + 1) & hs.mask)), claims);
  }
}

// --------------------------------------------------- block-level helpers
template <int THREADS>
__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
  constexpr int NW = THREADS / 32;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  long long t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < NW ? red[threadIdx.x] : 0;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Exclusive block scan of one long long per thread; returns the exclusive
// prefix and writes the block total to *total.
template <int THREADS>
__device__ __forceinline__ long long block_exclusive_scan(long long v, long long* red,
                                                          long long* total) {
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long w = threadIdx.x < NW ? red[threadIdx.x] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (threadIdx.x < NW) red[threadIdx.x] = w;  // inclusive over warps
  }
  __syncthreads();
  const long long warp_excl = warp > 0 ? red[warp - 1] : 0;
  *total = red[NW - 1];
  __syncthreads();
  return warp_excl + x - v;
}

// ---------------------------------------------------------------- K1 + K2
// Shared tail of both pass-1 kernels: per-row-block bin histogram (the
// per-chunk counts the deterministic pass 2 reserves from), block max/total.
__device__ __forceinline__ void pass1_finish(int* s_hist, long long mx, unsigned long long tot,
                                             int32_t* blk_counts, DevInfo* info,
                                             long long* s_red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    tot += __shfl_xor_sync(kFull, tot, o);
  }
  if (lane == 0) {
    s_red[warp] = mx;
    s_red[8 + warp] = static_cast<long long>(tot);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long m = 0;
    unsigned long long t = 0;
    for (int w = 0; w < kBinThreads / 32; ++w) {
      m = max(m, s_red[w]);
      t += static_cast<unsigned long long>(s_red[8 + w]);
    }
    atomicMax(&info->max_metric, m);
    atomicAdd(&info->total, t);
  }
  if (threadIdx.x < kNumBins) blk_counts[blockIdx.x * kNumBins + threadIdx.x] = s_hist[threadIdx.x];
}

// K1: nprod[i] = sum over A(i,:) of nnz(B(k,:)), written into C.rpt[0..M);
// fused with the symbolic pass-1 histogram and input_stats' max row length.
// Rows are read coalesced (thread per row); rows longer than 32 entries are
// summed cooperatively by their warp so power-law rows do not serialise.
__global__ void __launch_bounds__(kBinThreads)
    k_setup_nprod(DevCsr A, const int64_t* __restrict__ brpt, int64_t b_rows, int64_t* __restrict__ rpt,
                  int64_t M, BinUpper up, int32_t* __restrict__ blk_counts, DevInfo* info) {
  __shared__ int s_hist[kNumBins];
  __shared__ long long s_red[16];
  if (threadIdx.x < kNumBins) s_hist[threadIdx.x] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // operand sizes, so the host never reads them separately
    info->a_nnz = A.rpt[M];
    info->b_nnz = brpt[b_rows];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  long long mx = 0, amax = 0, bmax = 0;
  unsigned long long tot = 0;
#pragma unroll 1
  for (int it = 0; it < kRowsPerThread; ++it) {
    const int64_t row = base + it * kBinThreads + threadIdx.x;
    const bool valid = row < M;
    int64_t a0 = 0, a1 = 0;
    if (valid) {
      a0 = A.rpt[row];
      a1 = A.rpt[row + 1];
    }
    const bool longrow = (a1 - a0) > 32;
    long long n = 0;
    if (!longrow) {
      // 4 entries per round: their column loads, then their B-row bounds, in flight together
      int64_t p = a0;
      for (; p + 4 <= a1; p += 4) {
        int32_t k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) k[u] = A.col[p + u];
        long long l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) l[u] = brpt[k[u] + 1] - brpt[k[u]];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          n += l[u];
          bmax = max(bmax, l[u]);
        }
      }
      for (; p < a1; ++p) {
        const int32_t k = A.col[p];
        const long long l = brpt[k + 1] - brpt[k];
        n += l;
        bmax = max(bmax, l);
      }
    }
    unsigned lm = __ballot_sync(kFull, longrow);
    while (lm) {
      const int src = __ffs(lm) - 1;
      lm &= lm - 1;
      const int64_t s0 = __shfl_sync(kFull, a0, src), s1 = __shfl_sync(kFull, a1, src);
      long long part = 0;
      for (int64_t p = s0 + lane; p < s1; p += 32) {
        const int32_t k = A.col[p];
        const long long l = brpt[k + 1] - brpt[k];
        part += l;
        bmax = max(bmax, l);
      }
      part = warp_sum(part);
      if (lane == src) n = part;
    }
    if (valid) {
      rpt[row] = n;
      atomicAdd(&s_hist[classify_bin(n, up)], 1);
      mx = max(mx, n);
      tot += static_cast<unsigned long long>(n);
      amax = max(amax, static_cast<long long>(a1 - a0));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    amax = max(amax, __shfl_xor_sync(kFull, amax, o));
    bmax = max(bmax, __shfl_xor_sync(kFull, bmax, o));
  }
  if (lane == 0 && amax > 0) atomicMax(&info->a_max_row, amax);
  if (lane == 0 && bmax > 0) atomicMax(&info->b_max_row, bmax);
  __syncthreads();
  pass1_finish(s_hist, mx, tot, blk_counts, info, s_red);
  if (blockIdx.x == 0 && threadIdx.x == 0) rpt[M] = 0;
}

// K2: pass 1 over an arbitrary device metric (numeric phase: per-row nnz).
__global__ void __launch_bounds__(kBinThreads)
    k_pass1(const int64_t* __restrict__ metric, int64_t M, BinUpper up,
            int32_t* __restrict__ blk_counts, DevInfo* info) {
  __shared__ int s_hist[kNumBins];
  __shared__ long long s_red[16];
  if (threadIdx.x < kNumBins) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  long long mx = 0;
  unsigned long long tot = 0;
#pragma unroll
  for (int it = 0; it < kRowsPerThread; ++it) {
    const int64_t row = base + it * kBinThreads + threadIdx.x;
    if (row < M) {
      const long long v = metric[row];
      atomicAdd(&s_hist[classify_bin(v, up)], 1);
      mx = max(mx, v);
      tot += static_cast<unsigned long long>(v);
    }
  }
  __syncthreads();
  pass1_finish(s_hist, mx, tot, blk_counts, info, s_red);
}

// K3a: bin sizes, bin offsets (exclusive sum over bins, binning.cpp:304-305),
// fast-path flag, and the per-row-block write cursors in row-block order
// (the deterministic reservation of binning.cpp:220-229). One block; thread t
// holds row block t's 8 bin counts (one 32-byte load) and the 8 bins are
// scanned together -- per bin one warp-shuffle scan over the lanes and one
// over the 32 warp totals, three barriers per 1024 row blocks.
__global__ void __launch_bounds__(1024)
    k_bin_offsets(int32_t* __restrict__ blk_counts, int64_t nrb, int64_t M, long long upper0,
                  DevInfo* info) {
  static_assert(kNumBins == 8, "one int4 pair per row block");
  __shared__ int s_warp[32][kNumBins];
  __shared__ int s_wpre[32][kNumBins];
  __shared__ int s_tile[kNumBins];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool single = nrb <= 1024;  // one tile: totals and cursors from one scan
  long long carry[kNumBins];         // per bin: counts of the earlier tiles
  long long off[kNumBins];           // per bin: segment start (exclusive sum over bins)
#pragma unroll
  for (int j = 0; j < kNumBins; ++j) carry[j] = off[j] = 0;
  // pass 0: per-bin totals (sizes, offsets); pass 1 (several tiles only): cursors
  for (int pass = 0; pass < (single ? 1 : 2); ++pass) {
    for (int64_t t0 = 0; t0 < nrb; t0 += 1024) {
      const int64_t b = t0 + threadIdx.x;
      int v[kNumBins];
      if (b < nrb) {
        const int4* src = reinterpret_cast<const int4*>(blk_counts + b * kNumBins);
        const int4 x = src[0], y = src[1];
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
      } else {
#pragma unroll
        for (int j = 0; j < kNumBins; ++j) v[j] = 0;
      }
      int inc[kNumBins];  // inclusive within the warp (a tile holds < 2^31 rows)
#pragma unroll
      for (int j = 0; j < kNumBins; ++j) {
        int x = v[j];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        inc[j] = x;
      }
      if (lane == 31) {
#pragma unroll
        for (int j = 0; j < kNumBins; ++j) s_warp[warp][j] = inc[j];
      }
      __syncthreads();
      if (warp < kNumBins) {  // warp j scans bin j's 32 warp totals
        const int j = warp;
        const int x0 = s_warp[lane][j];
        int x = x0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        s_wpre[lane][j] = x - x0;
        if (lane == 31) s_tile[j] = x;
      }
      __syncthreads();
      long long before[kNumBins], tile[kNumBins];
#pragma unroll
      for (int j = 0; j < kNumBins; ++j) {
        before[j] = s_wpre[warp][j];
        tile[j] = s_tile[j];
      }
      if (single) {
        long long run = 0;
#pragma unroll
        for (int j = 0; j < kNumBins; ++j) {
          off[j] = run;
          run += tile[j];
        }
      }
      if ((single || pass == 1) && b < nrb) {
        int cur[kNumBins];
#pragma unroll
        for (int j = 0; j < kNumBins; ++j)
          cur[j] = static_cast<int32_t>(off[j] + carry[j] + before[j] + inc[j] - v[j]);
        int4* dst = reinterpret_cast<int4*>(blk_counts + b * kNumBins);
        dst[0] = make_int4(cur[0], cur[1], cur[2], cur[3]);
        dst[1] = make_int4(cur[4], cur[5], cur[6], cur[7]);
      }
#pragma unroll
      for (int j = 0; j < kNumBins; ++j) carry[j] += tile[j];
      __syncthreads();  // s_warp is reused by the next tile
    }
    if (pass == 0) {
      long long run = 0;
#pragma unroll
      for (int j = 0; j < kNumBins; ++j) {
        off[j] = run;
        run += carry[j];
      }
      if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < kNumBins; ++j) {
          info->bin_size[j] = carry[j];
          info->bin_offset[j] = off[j];
        }
        info->fast_path = (M == 0 || info->max_metric <= upper0) ? 1 : 0;
      }
#pragma unroll
      for (int j = 0; j < kNumBins; ++j) carry[j] = 0;
    }
  }
}

// K3b: scatter row ids into their bin segments. Within a row block the ids
// are ranked with warp ballots in ascending row order, so every segment lists
// its rows ascending: exactly the reference's deterministic layout
// (binning.cpp:205-241), whatever the chunk size. Skipped on the fast path.
__global__ void __launch_bounds__(kBinThreads)
    k_bin_scatter(const int64_t* __restrict__ metric, int64_t M, BinUpper up,
                  const int32_t* __restrict__ blk_offsets, int64_t* __restrict__ bins,
                  const DevInfo* info) {
  if (info->fast_path) return;
  constexpr int NW = kBinThreads / 32;
  __shared__ int s_wcnt[NW][kNumBins];
  __shared__ int s_run[kNumBins];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < kNumBins) s_run[threadIdx.x] = blk_offsets[blockIdx.x * kNumBins + threadIdx.x];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll 1
  for (int it = 0; it < kRowsPerThread; ++it) {
    const int64_t row = base + it * kBinThreads + threadIdx.x;
    const bool valid = row < M;
    const int bin = valid ? classify_bin(metric[row], up) : -1;
    int rank = 0;
#pragma unroll
    for (int j = 0; j < kNumBins; ++j) {
      const unsigned m = __ballot_sync(kFull, bin == j);
      if (bin == j) rank = __popc(m & lt);
      if (lane == j) s_wcnt[warp][j] = __popc(m);
    }
    __syncthreads();
    if (valid) {
      int pos = s_run[bin] + rank;
      for (int w = 0; w < warp; ++w) pos += s_wcnt[w][bin];
      bins[pos] = row;
    }
    __syncthreads();
    if (threadIdx.x < kNumBins) {
      int add = 0;
      for (int w = 0; w < NW; ++w) add += s_wcnt[w][threadIdx.x];
      s_run[threadIdx.x] += add;
    }
    __syncthreads();
  }
}

// Phase scalars to pinned, mapped host memory: written by the SMs rather than
// by a copy engine, so the read-back never queues behind a large device->host
// transfer on the copy lane (multiply_into's downloads).
static_assert(sizeof(DevInfo) % 8 == 0, "DevInfo moves as 8-byte words");
__global__ void k_info_to_host(const DevInfo* __restrict__ src, DevInfo* dst, int count) {
  const int words = count * static_cast<int>(sizeof(DevInfo) / 8);
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  volatile unsigned long long* d = reinterpret_cast<volatile unsigned long long*>(dst);
  // kernel completion + the host's stream synchronisation make the writes visible
  for (int i = threadIdx.x; i < words; i += blockDim.x) d[i] = s[i];
}

// dst[i] = src[i] + delta (row-pointer rebasing of row blocks; dst may be src)
__global__ void k_add_offset(int64_t* dst, const int64_t* src, int64_t n, int64_t delta) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i] + delta;
}

__global__ void k_iota(int64_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = i;
}

// K5: single-pass in-place exclusive scan (decoupled look-back) of n int64.
// Tiles are claimed in launch order through an atomic ticket so look-back
// always waits on tiles that are already running. A tile publishes its
// aggregate (flag 1) and later its inclusive prefix (flag 2) in separate
// slots, so a reader never sees one overwritten by the other. The look-back
// is done by a whole warp, 32 predecessor tiles per round: it stops at the
// nearest tile with an inclusive prefix and adds the aggregates in between.
// Each thread's kScanItems values are moved with 16-byte accesses.
__global__ void __launch_bounds__(kScanThreads)
    k_scan(int64_t* __restrict__ data, int64_t n, int* __restrict__ flags,
           long long* __restrict__ aggs, long long* __restrict__ incl, DevInfo* info) {
  static_assert(kScanItems % 2 == 0, "16-byte accesses");
  __shared__ int s_tile;
  __shared__ long long s_red[32];
  __shared__ long long s_excl;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_tile = atomicAdd(&info->tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = static_cast<int64_t>(tile) * kScanTile + threadIdx.x * kScanItems;
  long long v[kScanItems];
  long long tsum = 0;
  const bool full = base + kScanItems <= n;
  if (full) {
#pragma unroll
    for (int i = 0; i < kScanItems; i += 2) {
      const longlong2 x = *reinterpret_cast<const longlong2*>(data + base + i);
      v[i] = x.x;
      v[i + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) v[i] = (base + i < n) ? data[base + i] : 0;
  }
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) tsum += v[i];
  long long agg;
  const long long texcl = block_exclusive_scan<kScanThreads>(tsum, s_red, &agg);
  if (threadIdx.x < 32) {
    long long excl = 0;
    if (tile == 0) {
      if (lane == 0) {
        incl[0] = agg;
        __threadfence();
        atomicExch(&flags[0], 2);
      }
    } else {
      if (lane == 0) {
        aggs[tile] = agg;
        __threadfence();
        atomicExch(&flags[tile], 1);
      }
      int p = tile - 1;  // lane l looks at tile p - l
      while (true) {
        const int q = p - lane;
        int f;
        do {
          f = q >= 0 ? *reinterpret_cast<volatile int*>(&flags[q]) : 2;
        } while (__any_sync(kFull, f == 0));
        __threadfence();
        long long val = 0;
        if (q >= 0) val = f == 2 ? *reinterpret_cast<volatile long long*>(&incl[q])
                                 : *reinterpret_cast<volatile long long*>(&aggs[q]);
        const unsigned m2 = __ballot_sync(kFull, f == 2);
        if (m2) {
          const int first = __ffs(m2) - 1;  // nearest tile holding an inclusive prefix
          excl += warp_sum(lane <= first ? val : 0ll);
          break;
        }
        excl += warp_sum(val);
        p -= 32;
      }
      if (lane == 0) {
        incl[tile] = excl + agg;
        __threadfence();
        atomicExch(&flags[tile], 2);
      }
    }
    if (lane == 0) {
      s_excl = excl;
      if ((static_cast<int64_t>(tile) + 1) * kScanTile >= n) {
        info->scan_total = excl + agg;
        if (static_cast<unsigned long long>(excl + agg) != info->total) atomicOr(&info->error, kErrScanMismatch);
      }
    }
  }
  __syncthreads();
  long long run = s_excl + texcl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const long long x = v[i];
    v[i] = run;
    run += x;
  }
  if (full) {
#pragma unroll
    for (int i = 0; i < kScanItems; i += 2)
      *reinterpret_cast<longlong2*>(data + base + i) = make_longlong2(v[i], v[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      if (base + i < n) data[base + i] = v[i];
  }
}

// Row order of the persistent group kernels ("sweep"): group g of block b takes
// R consecutive rows at (b*NGRP + g)*R of every sweep of S = grid*NGRP*R rows.
// A group's consecutive rows share most of their B rows (L1 reuse), and at any
// time the whole GPU works inside one window of S rows, so the B rows those
// rows gather stay L2-resident (a fully block-contiguous order measured 2x the
// compulsory DRAM traffic on the 27-point stencil).
constexpr int kSweepRows = 8;  // power of two
struct Sweep {
  int64_t first, step;
  __device__ __forceinline__ Sweep(int ngrp, int grp) {
    first = (static_cast<int64_t>(blockIdx.x) * ngrp + grp) * kSweepRows;
    step = static_cast<int64_t>(gridDim.x) * ngrp * kSweepRows;
  }
  // increment from idx: the next of the group's R rows, or the next sweep
  __device__ __forceinline__ int64_t next(int64_t idx) const {
    return (idx & (kSweepRows - 1)) == kSweepRows - 1 ? step - (kSweepRows - 1) : 1;
  }
};

// ------------------------------------------------------------- row walker
template <int G>
__device__ __forceinline__ int group_max(int v, unsigned gm) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(gm, v, o, G));
  return v;
}

// Visits the products of one output row in the reference's (A entry, B entry)
// order. The group's lanes first load up to G A entries at once (column k,
// value, B row start/length: one round of latency instead of a dependent
// A.col -> B.rpt -> B.col chain per entry). When every B row of the chunk fits
// in G lanes, entry j is one "step" (lane q takes B(k_j, q)), and the B loads
// of U steps are issued before any of them is consumed, so U (x2 with
// values) independent loads are in flight per lane. Otherwise the group
// strides each B row. ORDERED inserts a group barrier after each A entry:
// within an entry the B columns are distinct (no two lanes share a slot), and
// the barrier orders entry j's updates before entry j+1's -- the reference's
// per-column summation order.
// Per-entry metadata of one A-row chunk, staged in shared memory so each step
// reads it with one broadcast 16-byte load.
// shared-window f64 load/store by 32-bit address; volatile: kept in program order
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v));
}
// predicated shared-window f64 load / store (no access when !on)
__device__ __forceinline__ double lds_f64_if(uint32_t a, bool on) {
  double v = 0.0;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f64 %0, [%1];\n\t}"
      : "+d"(v)
      : "r"(a), "r"(static_cast<int>(on)));
  return v;
}
__device__ __forceinline__ void sts_f64_if(uint32_t a, double v, bool on) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f64 [%0], %1;\n\t}" ::"r"(a),
               "d"(v), "r"(static_cast<int>(on)));
}
// predicated read-only global f64 load (0.0 when !on)
__device__ __forceinline__ double ldg_f64_if(const void* p, bool on) {
  double v = 0.0;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.f64 %0, [%1];\n\t}"
      : "+d"(v)
      : "l"(p), "r"(static_cast<int>(on)));
  return v;
}

struct EntryMeta {
  int32_t b0;   // B row start (32-bit index path)
  int32_t len;  // B row length
  double av;    // A value
};

template <int G, int U, bool VALS, bool ORDERED, typename IT, typename F>
__device__ __forceinline__ int walk_row(const DevCsr& A, const DevCsr& B, int64_t a0, int64_t a1,
                                        int lane, unsigned gm, EntryMeta* meta, F visit) {
  int acc = 0;  // sum of visit()'s return values (symbolic: new keys)
  for (int64_t c0 = a0; c0 < a1; c0 += G) {
    const int nc = static_cast<int>(min(static_cast<int64_t>(G), a1 - c0));
    IT b0 = 0;
    int len = 0;
    double av = 0.0;
    if (lane < nc) {
      const int32_t k = A.col[c0 + lane];
      if constexpr (VALS) av = A.val[c0 + lane];
      const int64_t r0 = B.rpt[k];
      b0 = static_cast<IT>(r0);
      len = static_cast<int>(B.rpt[k + 1] - r0);
    }
    const int maxlen = group_max<G>(len, gm);
    if (sizeof(IT) == 4 && maxlen <= G) {
      if (lane < nc) meta[lane] = EntryMeta{static_cast<int32_t>(b0), len, av};
      __syncwarp(gm);
      for (int j0 = 0; j0 < nc; j0 += U) {
        int32_t kc[U];
        double bv[U];
        double aj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const EntryMeta m = meta[min(j0 + u, G - 1)];
          aj[u] = m.av;
          const bool ok = (j0 + u < nc) && lane < m.len;
          const int at = m.b0 + lane;
          kc[u] = ok ? B.col[at] : -1;
          if constexpr (VALS) bv[u] = ok ? B.val[at] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (j0 + u < nc) {
            if (kc[u] >= 0) acc += visit(kc[u], VALS ? __dmul_rn(aj[u], bv[u]) : 0.0);
            if constexpr (ORDERED) __syncwarp(gm);
          }
        }
      }
      __syncwarp(gm);
    } else {
      for (int j = 0; j < nc; ++j) {
        const IT bj = __shfl_sync(gm, b0, j, G);
        const int lj = __shfl_sync(gm, len, j, G);
        const double a = VALS ? __shfl_sync(gm, av, j, G) : 0.0;
        for (int q = lane; q < lj; q += G) {
          const int32_t key = B.col[bj + q];
          acc += visit(key, VALS ? __dmul_rn(a, B.val[bj + q]) : 0.0);
        }
        if constexpr (ORDERED) __syncwarp(gm);
      }
    }
  }
  return acc;
}

// Ordered walker for the numeric phase, 32-bit index path. As walk_row, but
// the U steps' slot lookups/claims are batched (order-independent), then the
// U value updates run in step order with a group barrier between them; lanes
// without a product add 0.0 into a dummy slot so the update is branch-free.
// cap > 0 (speculative rows): the group's claims are counted per batch (a
// register, summed with one group reduction) and the walk stops as soon as
// they exceed cap -- returns the count (> cap: abandoned). A batch adds at most
// U*G claims and the walk only continues while claims <= cap, so with the
// table >= 2*cap slots (or more slots than the row has products) every claim
// finds a free slot.
template <int G, int U>
__device__ __forceinline__ int walk_row_num(const DevCsr& A, const DevCsr& B, int64_t a0, int64_t a1,
                                            int lane, unsigned gm, EntryMeta* meta, int32_t* keys,
                                            double* vals, const Hash& hs, uint32_t dummy, int32_t* kmin_out,
                                            int32_t* kmax_out, int cap = 0) {
  static_assert(G * U <= 128, "batch claims bounded by the speculative cap");
  // The row's column range, from the first/last column of each (sorted) B row:
  // two extra loads per A entry instead of a min/max pass over the table.
  int32_t kmin = 0x7fffffff, kmax = -1;
  int claimed = 0;  // uniform over the group
  for (int64_t c0 = a0; c0 < a1; c0 += G) {
    const int nc = static_cast<int>(min(static_cast<int64_t>(G), a1 - c0));
    int len = 0;
    if (lane < nc) {
      const int32_t k = A.col[c0 + lane];
      const double av = A.val[c0 + lane];
      const int64_t r0 = B.rpt[k];
      len = static_cast<int>(B.rpt[k + 1] - r0);
      meta[lane] = EntryMeta{static_cast<int32_t>(r0), len, av};
      if (len > 0) {
        kmin = min(kmin, B.col[r0]);
        kmax = max(kmax, B.col[r0 + len - 1]);
      }
    }
    const int maxlen = group_max<G>(len, gm);
    __syncwarp(gm);
    if (maxlen <= G) {
      for (int j0 = 0; j0 < nc; j0 += U) {
        if (cap && claimed > cap) break;
        int32_t kc[U];
        double x[U];
        uint32_t slot[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const EntryMeta m = meta[min(j0 + u, G - 1)];
          const bool ok = (j0 + u < nc) && lane < m.len;
          const int at = m.b0 + lane;
          kc[u] = ok ? B.col[at] : -1;
          x[u] = ok ? __dmul_rn(m.av, B.val[at]) : 0.0;
        }
        int mine = 0;
        num_slot_batch<U>(keys, kc, hs, dummy, slot, cap ? &mine : nullptr);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (j0 + u < nc) {
            vals[slot[u]] = __dadd_rn(vals[slot[u]], x[u]);
            __syncwarp(gm);
          }
        }
        if (cap) claimed += group_sum<G>(mine, gm);
      }
    } else {
      for (int j = 0; j < nc; ++j) {
        const EntryMeta m = meta[j];
        for (int qb = 0; qb < m.len; qb += G) {
          if (cap && claimed > cap) break;
          const int q = qb + lane;
          int32_t kc[1] = {q < m.len ? B.col[m.b0 + q] : -1};
          const double xv = q < m.len ? __dmul_rn(m.av, B.val[m.b0 + q]) : 0.0;
          uint32_t slot[1];
          int mine = 0;
          num_slot_batch<1>(keys, kc, hs, dummy, slot, cap ? &mine : nullptr);
          vals[slot[0]] = __dadd_rn(vals[slot[0]], xv);
          if (cap) claimed += group_sum<G>(mine, gm);
        }
        __syncwarp(gm);
      }
    }
    __syncwarp(gm);
    if (cap && claimed > cap) break;
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(gm, kmin, o, G));
    kmax = max(kmax, __shfl_xor_sync(gm, kmax, o, G));
  }
  *kmin_out = kmin;
  *kmax_out = kmax;
  return claimed;
}

// Unordered walk of ONE staged chunk (the symbolic phase has no summation
// order to keep): a step covers R = G/S A entries at once, S lanes per entry,
// V products per lane (lane sl of a sub-group takes B(k, qb + sl + S*v), v < V:
// coalesced within the sub-group). S is the smallest power of two with
// S*V >= the chunk's longest B row (capped at G; longer rows loop). Per-step
// bookkeeping is paid once per R*S*V products and each lane has V independent
// inserts in flight. visit(keys[V]) gets -1 for empty positions.
template <int G, int V, typename F>
__device__ __forceinline__ int walk_chunk_multi(const DevCsr& B, int nc, int maxlen, int lane,
                                                const EntryMeta* meta, F visit) {
  int acc = 0;
  int lgS = 0;
  while ((1 << lgS) * V < maxlen && (1 << lgS) < G) ++lgS;
  const int S = 1 << lgS;
  const int R = G >> lgS;
  const int sub = lane >> lgS, sl = lane & (S - 1);
  for (int j0 = 0; j0 < nc; j0 += R) {
    const int j = j0 + sub;
    const EntryMeta m = meta[min(j, G - 1)];
    const int lj = j < nc ? m.len : 0;
    for (int qb = 0; qb < lj; qb += S * V) {
      int32_t kc[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int q = qb + sl + S * v;
        kc[v] = q < lj ? B.col[m.b0 + q] : -1;
      }
      acc += visit(kc);
    }
  }
  return acc;
}

// Stages one chunk of up to G A entries (B row start/length, A value) in
// shared memory; returns the chunk's longest B row. With SPAN, also reduces the
// chunk's column range [lo, hi] (first/last column of each B row).
template <int G, bool SPAN>
__device__ __forceinline__ int stage_chunk(const DevCsr& A, const DevCsr& B, int64_t c0, int nc, int lane,
                                           unsigned gm, EntryMeta* meta, bool vals, int32_t* lo,
                                           int32_t* hi) {
  int len = 0;
  int32_t first = 0x7fffffff, last = -1;
  if (lane < nc) {
    const int32_t k = A.col[c0 + lane];
    const double av = vals ? A.val[c0 + lane] : 0.0;
    const int64_t r0 = B.rpt[k];
    len = static_cast<int>(B.rpt[k + 1] - r0);
    meta[lane] = EntryMeta{static_cast<int32_t>(r0), len, av};
    if (SPAN && len > 0) {
      first = B.col[r0];
      last = B.col[r0 + len - 1];
    }
  }
  if constexpr (SPAN) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      first = min(first, __shfl_xor_sync(gm, first, o, G));
      last = max(last, __shfl_xor_sync(gm, last, o, G));
    }
    *lo = first;
    *hi = last;
  }
  const int maxlen = group_max<G>(len, gm);
  __syncwarp(gm);
  return maxlen;
}

template <int G, int V, typename F>
__device__ __forceinline__ int walk_row_multi(const DevCsr& A, const DevCsr& B, int64_t a0, int64_t a1,
                                              int lane, unsigned gm, EntryMeta* meta, F visit) {
  int acc = 0;
  for (int64_t c0 = a0; c0 < a1; c0 += G) {
    const int nc = static_cast<int>(min(static_cast<int64_t>(G), a1 - c0));
    const int maxlen = stage_chunk<G, false>(A, B, c0, nc, lane, gm, meta, false, nullptr, nullptr);
    acc += walk_chunk_multi<G, V>(B, nc, maxlen, lane, meta, visit);
    __syncwarp(gm);
  }
  return acc;
}

// Window bitmap insert: one bit per column of the row's column range; a set
// returns whether the bit was new. Shared atomicOr runs at LDS throughput on
// sm_100 (tools/micro/smem_atomics.cu), and there is no probing.
template <int V>
__device__ __forceinline__ int bm_insert_batch(uint32_t* bm, const int32_t (&key)[V], int32_t lo) {
  int n = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (key[v] >= 0) {
      const uint32_t off = static_cast<uint32_t>(key[v] - lo);
      const uint32_t bit = 1u << (off & 31u);
      n += (atomicOr(bm + (off >> 5), bit) & bit) == 0u;
    }
  }
  return n;
}

// Fills n (multiple of 4 or not) int32 slots with -1 using 16-byte stores.
template <int G>
__device__ __forceinline__ void fill_empty(int32_t* tab, int n, int lane) {
  int4* t4 = reinterpret_cast<int4*>(tab);
  const int n4 = n >> 2;
  for (int s = lane; s < n4; s += G) t4[s] = make_int4(-1, -1, -1, -1);
  for (int s = (n4 << 2) + lane; s < n; s += G) tab[s] = -1;
}

template <int G>
__device__ __forceinline__ void fill_zero_words(uint32_t* w, int n, int lane) {
  uint4* w4 = reinterpret_cast<uint4*>(w);
  const int n4 = n >> 2;
  for (int s = lane; s < n4; s += G) w4[s] = make_uint4(0u, 0u, 0u, 0u);
  for (int s = (n4 << 2) + lane; s < n; s += G) w[s] = 0u;
}

template <int G>
__device__ __forceinline__ void fill_zero(double* v, int n, int lane) {
  double2* v2 = reinterpret_cast<double2*>(v);
  const int n2 = n >> 1;
  for (int s = lane; s < n2; s += G) v2[s] = make_double2(0.0, 0.0);
  if ((n & 1) && lane == 0) v[n - 1] = 0.0;
}

// --------------------------------------------------------- K6 symbolic
// Group kernel: G lanes per output row, NGRP rows in flight per block, one
// pow2 table of T int32 slots per row in shared memory. Persistent over the
// bin's rows (grid = resident blocks). The A row is walked entry by entry and
// the group's lanes stride the entry's B row.
__device__ __forceinline__ int ceil_log2_ll(long long x) {  // x >= 1
  return x <= 1 ? 0 : 64 - __clzll(x - 1);
}

// Symbolic group kernel. Per group: WB words of shared memory (>= T) used
// either as the row's window bitmap -- when the row is one chunk (<= G A
// entries) and its column span fits WB*32 bits -- or as its hash table
// (2*nprod slots, capped at T > the bin's nprod bound, so it never fills).
template <int G, int T, int NGRP, typename IT, int WB>
__global__ void __launch_bounds__(G* NGRP)
    k_sym_group(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, uint32_t scale, Spec sp) {
  const RowList rl = rl_in.resolved();
  static_assert(WB >= T, "bitmap region doubles as the hash table");
  constexpr int LOG_T = log2_const<T>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int32_t* tab = reinterpret_cast<int32_t*>(smem_raw) + (threadIdx.x / G) * WB;
  EntryMeta* meta = reinterpret_cast<EntryMeta*>(smem_raw + static_cast<size_t>(NGRP) * WB * 4) +
                    (threadIdx.x / G) * G;
  const int lane = threadIdx.x % G;
  const unsigned gm = group_mask<G>();
  const Sweep sw(NGRP, threadIdx.x / G);
  for (int64_t idx = sw.first; idx < rl.count; idx += sw.next(idx)) {
    if (sp.flag != nullptr && (idx & (kSweepRows - 1)) == 0) {
      // a run whose rows the speculative numeric kernel all finished is
      // skipped with one test of its kSweepRows rows (G >= kSweepRows lanes)
      static_assert(G >= kSweepRows, "one lane per row of the run");
      const bool open = lane < kSweepRows && idx + lane < rl.count && !sp.done(rl.row(idx + lane));
      if (__ballot_sync(gm, open) == 0u) {
        idx += kSweepRows - 1;  // the increment moves on to the next run
        continue;
      }
    }
    const int64_t row = rl.row(idx);
    if (sp.done(row)) continue;  // counted by the speculative numeric kernel
    const long long np = rpt[row];
    if (np == 0) continue;  // no products: nnz 0 (pipeline.cpp:368-371)
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    int cnt = 0;
    bool done = false;
    if constexpr (sizeof(IT) == 4) {
      if (a1 - a0 <= G) {
        const int nc = static_cast<int>(a1 - a0);
        int32_t lo, hi;
        const int maxlen = stage_chunk<G, true>(A, B, a0, nc, lane, gm, meta, false, &lo, &hi);
        const int64_t span = static_cast<int64_t>(hi) - lo + 1;
        if (span <= static_cast<int64_t>(WB) * 32) {
          const int words = static_cast<int>((span + 31) >> 5);
          uint32_t* bm = reinterpret_cast<uint32_t*>(tab);
          fill_zero_words<G>(bm, words, lane);
          __syncwarp(gm);
          cnt = walk_chunk_multi<G, 4>(B, nc, maxlen, lane, meta,
                                       [bm, lo](const int32_t(&k)[4]) { return bm_insert_batch<4>(bm, k, lo); });
        } else {
          const int lg = min(LOG_T, ceil_log2_ll(2 * np));
          const Hash hs = make_hash(scale, lg);
          fill_empty<G>(tab, 1 << lg, lane);
          __syncwarp(gm);
          cnt = walk_chunk_multi<G, 4>(B, nc, maxlen, lane, meta,
                                       [tab, hs](const int32_t(&k)[4]) { return sym_insert_batch<4>(tab, k, hs); });
        }
        done = true;
      }
    }
    if (!done) {
      const int lg = min(LOG_T, ceil_log2_ll(2 * np));
      const Hash hs = make_hash(scale, lg);
      fill_empty<G>(tab, 1 << lg, lane);
      __syncwarp(gm);
      if constexpr (sizeof(IT) == 4)
        cnt = walk_row_multi<G, 4>(A, B, a0, a1, lane, gm, meta,
                                   [tab, hs](const int32_t(&k)[4]) { return sym_insert_batch<4>(tab, k, hs); });
      else
        cnt = walk_row<G, 8, false, false, IT>(A, B, a0, a1, lane, gm, meta,
                                               [tab, hs](int32_t key, double) { return sym_insert(tab, key, hs); });
    }
    cnt = group_sum<G>(cnt, gm);
    __syncwarp(gm);
    if (lane == 0) rpt[row] = cnt;
  }
}

// Thread-per-row symbolic kernel for the smallest bin (nprod <= 2*TS/3; any TS,
// home slot = high product of the Fibonacci hash and TS): each
// thread owns one row and a private TS-slot table in shared memory laid out
// interleaved (slot s of lane l at [s*32 + l]: every lane always hits its own
// bank, whatever slot it probes). No atomics, barriers or shuffles.
template <int TS>
__global__ void __launch_bounds__(256)
    k_sym_thread(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, uint32_t scale) {
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* tab = reinterpret_cast<int32_t*>(smem_raw) + warp * TS * 32 + lane;
  const Hash hs = make_hash(scale, 5);  // its multiplier; the slot range is TS
  auto home = [&](int32_t key) { return __umulhi(static_cast<uint32_t>(key) * hs.mult, static_cast<uint32_t>(TS)); };
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < rl.count; idx += stride) {
    const int64_t row = rl.row(idx);
    if (rpt[row] == 0) continue;
#pragma unroll
    for (int s = 0; s < TS; ++s) tab[s * 32] = -1;
    int cnt = 0;
    const int64_t a1 = A.rpt[row + 1];
    for (int64_t p = A.rpt[row]; p < a1; ++p) {
      const int32_t k = A.col[p];
      const int64_t b1 = B.rpt[k + 1];
      for (int64_t q = B.rpt[k]; q < b1; ++q) {
        const int32_t key = B.col[q];
        uint32_t h = home(key);
        while (true) {
          const int32_t c = tab[h * 32];
          if (c == key) break;
          if (c == -1) {
            tab[h * 32] = key;
            ++cnt;
            break;
          }
          h = h + 1 == TS ? 0u : h + 1;
        }
      }
    }
    rpt[row] = cnt;
  }
}

// One row of k_num_thread (lane-private TS-slot table at keys/vals, lane
// stride 32): hash, compact, sort, write C(row,:).
template <int TS, int NMAX>
__device__ __forceinline__ void num_thread_row(int32_t* keys, double* vals, uint32_t mult, DevCsr A, DevCsr B,
                                               int64_t row, int64_t base, int n, int32_t* __restrict__ ccol,
                                               double* __restrict__ cval, DevInfo* info) {
  auto home = [&](int32_t key) { return __umulhi(static_cast<uint32_t>(key) * mult, static_cast<uint32_t>(TS)); };
#pragma unroll
  for (int s = 0; s < TS; ++s) {
    keys[s * 32] = -1;
    vals[s * 32] = 0.0;
  }
  const int64_t a1 = A.rpt[row + 1];
  // A entries two at a time: both B row ranges, then up to QB entries of each
  // B row, are loaded before any is inserted (independent loads in flight
  // instead of one dependent chain per product)
  constexpr int QB = 8;
  for (int64_t p = A.rpt[row]; p < a1; p += 2) {
    const bool two = p + 1 < a1;
    const int32_t k0 = A.col[p];
    const int32_t k1 = two ? A.col[p + 1] : k0;
    const double av0 = A.val[p];
    const double av1 = two ? A.val[p + 1] : 0.0;
    const int64_t q0 = B.rpt[k0], e0 = B.rpt[k0 + 1];
    const int64_t q1 = B.rpt[k1], e1 = two ? B.rpt[k1 + 1] : q1;
    auto insert = [&](int32_t key, double x) {
      uint32_t h = home(key);
      while (true) {
        const int32_t c = keys[h * 32];
        if (c == key) break;
        if (c == -1) {
          keys[h * 32] = key;
          break;
        }
        h = h + 1 == TS ? 0u : h + 1;
      }
      vals[h * 32] = __dadd_rn(vals[h * 32], x);
    };
    int32_t c0[QB], c1[QB];
    double v0[QB], v1[QB];
#pragma unroll
    for (int i = 0; i < QB; ++i) {
      c0[i] = q0 + i < e0 ? B.col[q0 + i] : -1;
      v0[i] = q0 + i < e0 ? B.val[q0 + i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < QB; ++i) {
      c1[i] = q1 + i < e1 ? B.col[q1 + i] : -1;
      v1[i] = q1 + i < e1 ? B.val[q1 + i] : 0.0;
    }
    // entry p (its whole B row) strictly before entry p + 1: the reference's order
#pragma unroll
    for (int i = 0; i < QB; ++i)
      if (c0[i] >= 0) insert(c0[i], __dmul_rn(av0, v0[i]));
    for (int64_t q = q0 + QB; q < e0; ++q) insert(B.col[q], __dmul_rn(av0, B.val[q]));
#pragma unroll
    for (int i = 0; i < QB; ++i)
      if (c1[i] >= 0) insert(c1[i], __dmul_rn(av1, v1[i]));
    for (int64_t q = q1 + QB; q < e1; ++q) insert(B.col[q], __dmul_rn(av1, B.val[q]));
  }
  // compact in place: entry m <- slot s (m <= s), keys and values together
  int m = 0;
  int32_t kmin = 0x7fffffff, kmax = -1;
#pragma unroll
  for (int s = 0; s < TS; ++s) {
    const int32_t c = keys[s * 32];
    if (c != -1) {
      keys[m * 32] = c;
      vals[m * 32] = vals[s * 32];
      kmin = min(kmin, c);
      kmax = max(kmax, c);
      ++m;
    }
  }
  if (m != n) atomicOr(&info->error, kErrNumericCount);
  constexpr int LG = log2_const<NMAX>();
  if (static_cast<uint32_t>(kmax - kmin) < (0xffffffffu >> LG)) {
    // narrow row: 32-bit keys (col - kmin) << LG | entry, sorted with min/max pairs
    uint32_t v[NMAX];
#pragma unroll
    for (int i = 0; i < NMAX; ++i)
      v[i] = i < m ? (static_cast<uint32_t>(keys[i * 32] - kmin) << LG) | static_cast<uint32_t>(i) : 0xffffffffu;
#pragma unroll
    for (int k = 2; k <= NMAX; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
        for (int i = 0; i < NMAX; ++i) {
          const int pi = i ^ j;
          if (pi > i) {
            const uint32_t a = v[i], b = v[pi];
            const bool up = (i & k) == 0;
            v[i] = up ? min(a, b) : max(a, b);
            v[pi] = up ? max(a, b) : min(a, b);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
      if (i < m) {
        ccol[base + i] = kmin + static_cast<int32_t>(v[i] >> LG);
        cval[base + i] = vals[(v[i] & (NMAX - 1u)) * 32];
      }
    }
    return;
  }
  unsigned long long v[NMAX];
#pragma unroll
  for (int i = 0; i < NMAX; ++i)
    v[i] = i < m ? (static_cast<unsigned long long>(static_cast<uint32_t>(keys[i * 32])) << 32) | static_cast<uint32_t>(i)
                 : ~0ull;
#pragma unroll
  for (int k = 2; k <= NMAX; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < NMAX; ++i) {
        const int pi = i ^ j;
        if (pi > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = v[i], b = v[pi];
          const bool sw = up ? (a > b) : (a < b);
          v[i] = sw ? b : a;
          v[pi] = sw ? a : b;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    if (i < m) {
      ccol[base + i] = static_cast<int32_t>(v[i] >> 32);
      cval[base + i] = vals[static_cast<uint32_t>(v[i]) * 32];
    }
  }
}

// Thread-per-row numeric kernel for rows with nnz <= NMAX (TS >= 1.5*NMAX slots,
// any TS: the home slot is the high product of the Fibonacci hash and TS, so a
// 24-slot table (288 B/thread instead of 384) fits 6 blocks per SM instead of 4):
// the thread walks its row in the reference's order (so the fold is trivially
// the reference's), compacts its private table in place, sorts the NMAX packed
// (col, slot) keys with a register bitonic network, and writes C(i,:).
template <int TS, int NMAX>
__global__ void __launch_bounds__(128)
    k_num_thread(RowList rl_in, DevCsr A, DevCsr B, const int64_t* __restrict__ rpt,
                 int32_t* __restrict__ ccol, double* __restrict__ cval, uint32_t scale, DevInfo* info,
                 Spec sp) {
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* vals = reinterpret_cast<double*>(smem_raw) + warp * TS * 32 + lane;
  int32_t* keys = reinterpret_cast<int32_t*>(smem_raw + static_cast<size_t>(blockDim.x) * TS * 8) +
                  warp * TS * 32 + lane;
  const Hash hs = make_hash(scale, 5);  // its multiplier; the slot range is TS
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < rl.count; idx += stride) {
    const int64_t row = rl.row(idx);
    const int64_t base = rpt[row];
    const int n = static_cast<int>(rpt[row + 1] - base);
    if (n == 0) continue;
    if (sp.done(row)) continue;  // computed in the symbolic phase, copied by k_spec_copy
    num_thread_row<TS, NMAX>(keys, vals, hs.mult, A, B, row, base, n, ccol, cval, info);
  }
}

// Block kernel: one row per block iteration, warps take A entries, lanes
// stride B rows. SPILL (the last bin): the fixed table aborts a row once its
// distinct count exceeds the reference's 0.8*24575 = 19660 threshold
// (hash_tables.hpp:18-21) and queues it for k_sym_spill.
template <int T, int THREADS, bool SPILL>
__global__ void __launch_bounds__(THREADS)
    k_sym_block(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, uint32_t scale,
                int64_t* __restrict__ spill_ids, DevInfo* info, int thresh) {
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int32_t* tab = reinterpret_cast<int32_t*>(smem_raw);
  __shared__ int s_cnt, s_abort;
  __shared__ long long s_red[32];
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Hash hs = make_hash(scale, log2_const<T>());
  for (int64_t idx = blockIdx.x; idx < rl.count; idx += gridDim.x) {
    const int64_t row = rl.row(idx);
    if (rpt[row] == 0) continue;
    for (int s = threadIdx.x; s < T; s += THREADS) tab[s] = -1;
    if (threadIdx.x == 0) {
      s_cnt = 0;
      s_abort = 0;
    }
    __syncthreads();
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    int cnt = 0;
    for (int64_t p = a0 + warp; p < a1; p += NW) {
      const int32_t k = A.col[p];
      const int64_t b0 = B.rpt[k], b1 = B.rpt[k + 1];
      for (int64_t qb = b0; qb < b1; qb += 32) {
        const int64_t q = qb + lane;
        const int nw = q < b1 ? sym_insert(tab, B.col[q], hs) : 0;
        if constexpr (SPILL) {
          const unsigned bal = __ballot_sync(kFull, nw);
          int abort = 0;
          if (lane == 0) {
            if (bal) {
              const int c = __popc(bal);
              if (atomicAdd(&s_cnt, c) + c > thresh) s_abort = 1;
            }
            abort = *reinterpret_cast<volatile int*>(&s_abort);
          }
          if (__shfl_sync(kFull, abort, 0)) goto row_done;
        } else {
          cnt += nw;
        }
      }
    }
  row_done:
    if constexpr (SPILL) {
      __syncthreads();
      if (threadIdx.x == 0) {
        if (s_abort) {
          const unsigned long long i = atomicAdd(&info->spill_count, 1ull);
          spill_ids[i] = row;
        } else {
          rpt[row] = s_cnt;
        }
      }
      __syncthreads();
    } else {
      const long long total = block_sum_ll<THREADS>(cnt, s_red);
      if (threadIdx.x == 0) rpt[row] = total;
    }
  }
}

// Spilled rows (pipeline.cpp:315-348, hash_tables.cpp:113-123): recount with a
// global-memory table. Instead of one heap table per row, each resident block
// reuses one region of a pool; the row's table is bit_ceil(2*min(nprod, cols)).
__global__ void __launch_bounds__(1024)
    k_sym_spill(DevCsr A, DevCsr B, int64_t* __restrict__ rpt, const int64_t* __restrict__ spill_ids,
                const DevInfo* info, int32_t* __restrict__ pool, int64_t slots_per_block,
                uint32_t scale) {
  __shared__ long long s_red[32];
  int32_t* tab = pool + static_cast<int64_t>(blockIdx.x) * slots_per_block;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long count = static_cast<long long>(info->spill_count);
  for (long long idx = blockIdx.x; idx < count; idx += gridDim.x) {
    const int64_t row = spill_ids[idx];
    const long long nprod = rpt[row];
    long long want = 2 * min(nprod, static_cast<long long>(B.cols));
    long long t = 2;
    while (t < want) t <<= 1;
    if (t > slots_per_block) t = slots_per_block;
    int lg = 0;
    while ((1ll << lg) < t) ++lg;
    const Hash hs = make_hash(scale, lg);
    for (long long s = threadIdx.x; s < t; s += 1024) tab[s] = -1;
    __syncthreads();
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    int cnt = 0;
    for (int64_t p = a0 + warp; p < a1; p += 32) {
      const int32_t k = A.col[p];
      const int64_t b1 = B.rpt[k + 1];
      for (int64_t q = B.rpt[k] + lane; q < b1; q += 32) cnt += sym_insert(tab, B.col[q], hs);
    }
    const long long total = block_sum_ll<1024>(cnt, s_red);
    if (threadIdx.x == 0) rpt[row] = total;
  }
}

// ---------------------------------------------------------- K7 numeric
// Bitonic sort of N = G*E keys held E per lane (blocked layout: element
// lane*E+i) across a G-lane group; ascending.
template <int G, int E, typename K>
__device__ __forceinline__ void group_bitonic(K (&v)[E], int lane, unsigned gm) {
  constexpr int N = G * E;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {
        const int lj = j / E;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int e = lane * E + i;
          const K other = __shfl_xor_sync(gm, v[i], lj, G);
          const bool up = (e & k) == 0;
          const bool lower = (e & j) == 0;
          v[i] = (lower == up) ? min(v[i], other) : max(v[i], other);
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int pi = i ^ j;
          if (pi > i) {
            const int e = lane * E + i;
            const bool up = (e & k) == 0;
            const K a = v[i], b = v[pi];
            const bool sw = up ? (a > b) : (a < b);
            v[i] = sw ? b : a;
            v[pi] = sw ? a : b;
          }
        }
      }
    }
  }
}

// Sorts the n condensed keys of buf (n <= G*E) in place, with the smallest
// network that covers n.
template <int G, int E, typename K>
__device__ __forceinline__ void group_sort_inplace(K* buf, int n, int lane, unsigned gm) {
  if constexpr (E > 1) {
    if (n <= G * E / 2) {
      group_sort_inplace<G, (E > 1 ? E / 2 : 1), K>(buf, n, lane, gm);
      return;
    }
  }
  K v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int e = lane * E + i;
    v[i] = e < n ? buf[e] : static_cast<K>(~static_cast<K>(0));
  }
  group_bitonic<G, E, K>(v, lane, gm);
#pragma unroll
  for (int i = 0; i < E; ++i) buf[lane * E + i] = v[i];
}

// Group kernel: G lanes per row; per group T key slots + T fp64 values +
// G*E sort keys in shared memory. Ordered steps over the A row (see the
// header comment); then condense (hash_tables.cpp:125-135), a bitonic sort by
// column (hash_tables.cpp:137-177) and a coalesced write of C(i,:) at rpt[i].
// The sort key packs (col - min col) with the slot index into 32 bits when the
// row's column span allows (64 bits otherwise).
// The 32x256 instance (3-D stencil rows) is latency-bound: capping it at 51
// registers (5 resident blocks, 40 warps/SM) measured 3% faster than 64.
// SPEC = the speculative numeric of the symbolic phase (see Spec): rows come
// from a symbolic bin, the table is T slots, at most sp.cap = NMAX claims, and
// the result goes to the Spec scratch with its count in rpt. Otherwise rows
// already done speculatively are copied from the scratch into C.
template <int G, int T, int E, int NGRP, typename IT, bool SPEC>
__global__ void __launch_bounds__(G* NGRP, (G == 32 && T == 256) ? 5 : 1)
    k_num_group(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt,
                int32_t* __restrict__ ccol, double* __restrict__ cval, uint32_t scale,
                DevInfo* info, Spec sp) {
  const RowList rl = rl_in.resolved();
  constexpr int NMAX = G * E;
  constexpr int LOG_T = log2_const<T>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int grp = threadIdx.x / G;
  // per group: vals[T + 2] (slot T is the dummy), packed[NMAX], keys[T], meta[G], 16 spare bytes
  constexpr size_t kGroupBytes = (T + 2) * 8 + NMAX * 8 + T * 4 + G * 16 + 16;
  unsigned char* gbase = smem_raw + static_cast<size_t>(grp) * kGroupBytes;
  double* vals = reinterpret_cast<double*>(gbase);
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(gbase + (T + 2) * 8);
  uint32_t* packed32 = reinterpret_cast<uint32_t*>(packed);
  int32_t* keys = reinterpret_cast<int32_t*>(gbase + (T + 2) * 8 + NMAX * 8);
  EntryMeta* meta = reinterpret_cast<EntryMeta*>(gbase + (T + 2) * 8 + NMAX * 8 + T * 4);
  const int lane = threadIdx.x % G;
  const unsigned gm = group_mask<G>();
  const unsigned gshift = (threadIdx.x & 31u) & ~(G - 1u);
  const Sweep sw(NGRP, grp);
  for (int64_t idx = sw.first; idx < rl.count; idx += sw.next(idx)) {
    const int64_t row = rl.row(idx);
    int64_t base = 0;
    int n = 0;
    int lg = LOG_T;
    if constexpr (SPEC) {
      const long long np = rpt[row];
      if (np == 0) continue;  // no products: the symbolic kernel writes the 0
      lg = min(LOG_T, ceil_log2_ll(2 * min(np, static_cast<long long>(NMAX))));  // nnz <= min(nprod, cap)
    } else {
      if (sp.done(row)) continue;  // computed in the symbolic phase, copied by k_spec_copy
      base = rpt[row];
      n = static_cast<int>(rpt[row + 1] - base);
      if (n == 0) continue;
      lg = min(LOG_T, ceil_log2_ll(2 * static_cast<long long>(n)));
    }
    const int tsz = 1 << lg;
    const Hash hs = make_hash(scale, lg);
    fill_empty<G>(keys, tsz, lane);
    fill_zero<G>(vals, tsz, lane);
    __syncwarp(gm);
    int kmin = 0x7fffffff, kmax = -1;
    int claimed = 0;
    if constexpr (sizeof(IT) == 4) {
      claimed = walk_row_num<G, 4>(A, B, A.rpt[row], A.rpt[row + 1], lane, gm, meta, keys, vals, hs,
                                   static_cast<uint32_t>(T), &kmin, &kmax, SPEC ? NMAX : 0);
    } else {
      walk_row<G, 4, true, true, IT>(A, B, A.rpt[row], A.rpt[row + 1], lane, gm, meta,
                                     [keys, vals, hs](int32_t key, double x) {
                                       const uint32_t s = num_slot(keys, key, hs);
                                       vals[s] = __dadd_rn(vals[s], x);
                                       return 0;
                                     });
    }
    if constexpr (sizeof(IT) != 4) {  // 64-bit index path: range from the table
      for (int s = lane; s < tsz; s += G) {
        const int32_t key = keys[s];
        if (key != -1) {
          kmin = min(kmin, key);
          kmax = max(kmax, key);
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(gm, kmin, o, G));
        kmax = max(kmax, __shfl_xor_sync(gm, kmax, o, G));
      }
    }
    if constexpr (SPEC) {
      __syncwarp(gm);
      if (claimed > NMAX) continue;  // abandoned (uniform): the symbolic kernel counts this row
      n = claimed;
    }
    int32_t* ocol = SPEC ? sp.col + row * sp.cap : ccol + base;
    double* oval = SPEC ? sp.val + row * sp.cap : cval + base;
    const bool narrow = static_cast<unsigned>(kmax - kmin) < ((0xffffffffu >> lg) - 1u);
    int run = 0;
    auto emit = [&](int at, int32_t key, int s) {
      if (narrow)
        packed32[at] = (static_cast<uint32_t>(key - kmin) << lg) | static_cast<uint32_t>(s);
      else
        packed[at] = (static_cast<unsigned long long>(static_cast<uint32_t>(key)) << 32) | static_cast<uint32_t>(s);
    };
    if (tsz >= 4 * G) {
      // 4 slots per lane per pass (one 16-byte load); a lane's rank is the
      // count of occupied slots in lower lanes over the 4 per-position ballots
      const unsigned lt = (1u << lane) - 1u;
      for (int s0 = 0; s0 < tsz; s0 += 4 * G) {
        const int4 k4 = reinterpret_cast<const int4*>(keys + s0)[lane];
        const unsigned b0 = __ballot_sync(gm, k4.x != -1) >> gshift, b1 = __ballot_sync(gm, k4.y != -1) >> gshift;
        const unsigned b2 = __ballot_sync(gm, k4.z != -1) >> gshift, b3 = __ballot_sync(gm, k4.w != -1) >> gshift;
        int at = run + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
        const int s = s0 + 4 * lane;
        if (k4.x != -1) emit(at++, k4.x, s);
        if (k4.y != -1) emit(at++, k4.y, s + 1);
        if (k4.z != -1) emit(at++, k4.z, s + 2);
        if (k4.w != -1) emit(at++, k4.w, s + 3);
        run += __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
      }
    } else {
      for (int s0 = 0; s0 < tsz; s0 += G) {
        const int s = s0 + lane;
        const int32_t key = s < tsz ? keys[s] : -1;
        const bool occ = key != -1;
        const unsigned bal = __ballot_sync(gm, occ) >> gshift;
        if (occ) emit(run + __popc(bal & ((1u << lane) - 1u)), key, s);
        run += __popc(bal);
      }
    }
    if (run != n && lane == 0) atomicOr(&info->error, kErrNumericCount);
    __syncwarp(gm);
    if (narrow) {
      group_sort_inplace<G, E, uint32_t>(packed32, n, lane, gm);
      __syncwarp(gm);
      const uint32_t smask = (1u << lg) - 1u;
      for (int e = lane; e < n; e += G) {
        const uint32_t v = packed32[e];
        ocol[e] = kmin + static_cast<int32_t>(v >> lg);
        oval[e] = vals[v & smask];
      }
    } else {
      group_sort_inplace<G, E, unsigned long long>(packed, n, lane, gm);
      __syncwarp(gm);
      for (int e = lane; e < n; e += G) {
        const unsigned long long v = packed[e];
        ocol[e] = static_cast<int32_t>(v >> 32);
        oval[e] = vals[static_cast<uint32_t>(v)];
      }
    }
    if constexpr (SPEC) {
      if (lane == 0) {
        rpt[row] = n;
        sp.flag[row] = 1;
      }
    }
    __syncwarp(gm);
  }
}

// Lean ordered numeric for warp-sized rows (3-D stencils, FEM, the RAP chain):
// one warp per row. A row whose A row has <= 32 entries and whose B rows all
// have <= 32 entries (the common case for these bins) is walked one A entry per
// step: lane q takes B(k_j, q), step j+1's loads issued before step j's
// updates. The column table is sparse (<= 512 slots, load <= 1/4, so a probe
// rarely goes past the home slot) and maps a column to a DENSE index: the
// column's values live in vals[0..n) and its column in cols[0..n), in claim
// order. A step's claims are ranked with one ballot (the claim count is warp-
// uniform, so a speculative row gives up as soon as it exceeds NMAX, before any
// out-of-range write). The claiming lane writes the column's first product as
// 0.0 + x -- the reference's +0.0 start (hash_tables.hpp:130) -- and every
// later product is a read-modify-write of vals[idx]. Within a step the B row's
// columns are distinct; __syncwarp orders the steps, so each column folds in
// the reference's A-row order. No condense pass: the n dense columns are sorted
// directly (packed with their index) and written with their values.
// Numeric launches are made only when A's and B's longest rows are <= 32
// (K1 reports both); a speculative row with longer rows is abandoned.
constexpr int kLeanGroups = 8;
constexpr int kLeanT = 512;     // sparse column table slots
constexpr int kLeanN = 128;     // dense entries (the numeric bin's nnz bound / the speculative cap)
constexpr size_t kLeanGroupBytes = kLeanT * 4 + kLeanT + kLeanN * 8 + kLeanN * 4 + 32 * 16;
template <bool SPEC>
__global__ void __launch_bounds__(32 * kLeanGroups, 5)
    k_num_lean(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, int32_t* __restrict__ ccol,
               double* __restrict__ cval, uint32_t scale, DevInfo* info, Spec sp) {
  constexpr int G = 32, NMAX = kLeanN, E = 4;
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int grp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* gbase = smem_raw + static_cast<size_t>(grp) * kLeanGroupBytes;
  int32_t* keys = reinterpret_cast<int32_t*>(gbase);                       // [kLeanT]; after the walk: sort keys
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(gbase);  // (aliases keys: 128 x 8 B)
  uint32_t* packed32 = reinterpret_cast<uint32_t*>(gbase);
  uint8_t* sidx = gbase + kLeanT * 4;                                       // [kLeanT] dense index per slot
  double* vals = reinterpret_cast<double*>(gbase + kLeanT * 5);            // [NMAX]
  int32_t* cols = reinterpret_cast<int32_t*>(gbase + kLeanT * 5 + NMAX * 8);  // [NMAX]
  EntryMeta* meta = reinterpret_cast<EntryMeta*>(gbase + kLeanT * 5 + NMAX * 12);
  const unsigned lt = (1u << lane) - 1u;
  const Sweep sw(kLeanGroups, grp);
  for (int64_t idx = sw.first; idx < rl.count; idx += sw.next(idx)) {
    const int64_t row = rl.row(idx);
    int64_t base = 0;
    int n = 0;
    long long bound;  // >= the row's distinct columns
    if constexpr (SPEC) {
      const long long np = rpt[row];
      if (np == 0) continue;  // no products: the symbolic kernel writes the 0
      bound = min(np, static_cast<long long>(NMAX));
    } else {
      if (sp.done(row)) continue;  // computed in the symbolic phase, copied by k_spec_copy
      base = rpt[row];
      n = static_cast<int>(rpt[row + 1] - base);
      if (n == 0) continue;
      bound = n;
    }
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    const int na = static_cast<int>(min(a1 - a0, static_cast<int64_t>(1 << 30)));
    int len = 0;
    int32_t kmin = 0x7fffffff, kmax = -1;
    if (lane < na) {
      const int32_t k = A.col[a0 + lane];
      const double av = A.val[a0 + lane];
      const int64_t r0 = B.rpt[k];
      len = static_cast<int>(B.rpt[k + 1] - r0);
      meta[lane] = EntryMeta{static_cast<int32_t>(r0), len, av};
      if (len > 0) {
        kmin = B.col[r0];
        kmax = B.col[r0 + len - 1];
      }
    }
    const int maxlen = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(len)));
    kmin = static_cast<int32_t>(__reduce_min_sync(kFull, static_cast<unsigned>(kmin)));
    kmax = static_cast<int32_t>(__reduce_max_sync(kFull, static_cast<unsigned>(kmax + 1))) - 1;
    int nk = 0;  // distinct columns claimed (warp-uniform)
    if (na <= G && maxlen <= G) {
      const int lg = min(log2_const<kLeanT>(), max(2, ceil_log2_ll(4 * bound)));
      const int tsz = 1 << lg;
      const Hash hs = make_hash(scale, lg);
      fill_empty<G>(keys, tsz, lane);
      __syncwarp();
      EntryMeta m = meta[0];
      int32_t cn = lane < m.len ? B.col[m.b0 + lane] : -1;
      double vn = lane < m.len ? B.val[m.b0 + lane] : 0.0;
      for (int j = 0; j < na; ++j) {
        const double a = m.av;
        const int32_t c = cn;
        const double bv = vn;
        if (j + 1 < na) {
          m = meta[j + 1];
          cn = lane < m.len ? B.col[m.b0 + lane] : -1;
          vn = lane < m.len ? B.val[m.b0 + lane] : 0.0;
        }
        const double x = __dmul_rn(a, bv);
        uint32_t h = c >= 0 ? hs.home(c) : 0u;
        int32_t cur = c >= 0 ? keys[h] : c;
        bool fresh = false;
        if (__any_sync(kFull, cur != c)) {
          while (cur != c) {
            if (cur == -1) {
              cur = atomicCAS(reinterpret_cast<int*>(keys + h), -1, c);
              if (cur == -1) {
                fresh = true;
                break;
              }
              continue;
            }
            h = (h + 1) & hs.mask;
            cur = *reinterpret_cast<volatile int32_t*>(keys + h);
          }
        }
        const unsigned cb = __ballot_sync(kFull, fresh);
        if constexpr (SPEC) {
          if (nk + __popc(cb) > NMAX) {  // more columns than the scratch holds: abandon the row
            nk = NMAX + 1;
            break;
          }
        }
        if (fresh) {
          const int ix = nk + __popc(cb & lt);
          sidx[h] = static_cast<uint8_t>(ix);
          cols[ix] = c;
          vals[ix] = __dadd_rn(0.0, x);
        } else if (c >= 0) {
          const int ix = sidx[h];
          vals[ix] = __dadd_rn(vals[ix], x);
        }
        nk += __popc(cb);
        __syncwarp();
      }
    } else {
      // longer A or B rows: never here for numeric launches (the host checks
      // A's and B's longest rows); a speculative row is left to the symbolic
      // kernel and the generic numeric kernels
      nk = NMAX + 1;
    }
    __syncwarp();
    if constexpr (SPEC) {
      if (nk > NMAX) continue;  // abandoned (uniform): the symbolic kernel counts this row
      n = nk;
    } else {
      if (nk != n && lane == 0) atomicOr(&info->error, kErrNumericCount);
    }
    int32_t* ocol = SPEC ? sp.col + row * sp.cap : ccol + base;
    double* oval = SPEC ? sp.val + row * sp.cap : cval + base;
    // sort the n columns (with their dense index) and write C(i,:)
    const bool narrow = static_cast<unsigned>(kmax - kmin) < (1u << 25);
    for (int e = lane; e < n; e += G) {
      const int32_t c = cols[e];
      if (narrow) packed32[e] = (static_cast<uint32_t>(c - kmin) << 7) | static_cast<uint32_t>(e);
      else packed[e] = (static_cast<unsigned long long>(static_cast<uint32_t>(c)) << 32) | static_cast<uint32_t>(e);
    }
    __syncwarp();
    if (narrow) {
      group_sort_inplace<G, E, uint32_t>(packed32, n, lane, kFull);
      __syncwarp();
      for (int e = lane; e < n; e += G) {
        const uint32_t v = packed32[e];
        ocol[e] = kmin + static_cast<int32_t>(v >> 7);
        oval[e] = vals[v & 127u];
      }
    } else {
      group_sort_inplace<G, E, unsigned long long>(packed, n, lane, kFull);
      __syncwarp();
      for (int e = lane; e < n; e += G) {
        const unsigned long long v = packed[e];
        ocol[e] = static_cast<int32_t>(v >> 32);
        oval[e] = vals[static_cast<uint32_t>(v) & 127u];
      }
    }
    if constexpr (SPEC) {
      if (lane == 0) {
        rpt[row] = n;
        sp.flag[row] = 1;
      }
    }
    __syncwarp();
  }
}

// Sort of the n valid keys of buf where the network size is chosen from
// `nsel` (the same for every group of the warp, so groups sorting different
// rows stay converged); entries n..network are padded with the maximum key.
template <int G, int E, typename K>
__device__ __forceinline__ void group_sort_padded(K* buf, int n, int nsel, int lane, unsigned gm) {
  if constexpr (E > 1) {
    if (nsel <= G * E / 2) {
      group_sort_padded<G, (E > 1 ? E / 2 : 1), K>(buf, n, nsel, lane, gm);
      return;
    }
  }
  K v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int e = lane * E + i;
    v[i] = e < n ? buf[e] : static_cast<K>(~static_cast<K>(0));
  }
  group_bitonic<G, E, K>(v, lane, gm);
#pragma unroll
  for (int i = 0; i < E; ++i) buf[lane * E + i] = v[i];
}

// Paired-row ordered numeric (the 3-D stencil / FEM bins): TWO rows per warp,
// a half-warp (16 lanes) per row, so every per-step instruction -- entry
// metadata, loads, hashing, the miss vote, the barrier -- serves two rows, and
// each lane carries two products of the step (B positions q and q+16 of the
// entry's B row, distinct columns). Preconditions (host-checked for numeric
// launches, per row for speculative ones): A rows and B rows of <= 32 entries.
// Per row: a sparse column table of 256 slots (load <= 1/2) mapping a column
// to a DENSE index -- values in vals[0..n), columns in cols[0..n) in claim
// order -- claims ranked by ballots within the half-warp. The first product of
// a column (its claim, in step order) is written as 0.0 + x, the reference's
// +0.0 start (hash_tables.hpp:130); later products are read-modify-writes;
// __syncwarp orders the steps (per column: the reference's A-row order). A
// speculative row abandons (flagged, left to the symbolic kernel) once it
// claims more than NMAX columns. The n columns are then sorted with their index
// packed in (the two halves run one network sized for the larger row) and
// written with their values.
constexpr int kPairWarps = 8;
constexpr int kPairT = 256, kPairN = 128;
constexpr size_t kPairRowBytes = kPairT * 4 + kPairT + kPairN * 8 + kPairN * 4 + 32 * 16;  // 3328
template <typename T>
__device__ __forceinline__ T half_min(T v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o, 16));
  return v;
}
template <typename T>
__device__ __forceinline__ T half_max(T v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o, 16));
  return v;
}

template <bool SPEC>
__global__ void __launch_bounds__(32 * kPairWarps, 4)
    k_num_pair(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, int32_t* __restrict__ ccol,
               double* __restrict__ cval, uint32_t scale, DevInfo* info, Spec sp) {
  constexpr int HG = 16, NMAX = kPairN, E = 8, LOG_T = 8;
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;
  const unsigned hm = 0xffffu << (16 * half);                // this row's lanes
  const unsigned hlt = ((1u << hl) - 1u) << (16 * half);     // lower lanes of this row
  unsigned char* rbase = smem_raw + (static_cast<size_t>(warp) * 2 + half) * kPairRowBytes;
  int32_t* keys = reinterpret_cast<int32_t*>(rbase);  // [kPairT]; after the walk: sort keys
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(rbase);
  uint32_t* packed32 = reinterpret_cast<uint32_t*>(rbase);
  uint8_t* sidx = rbase + kPairT * 4;
  double* vals = reinterpret_cast<double*>(rbase + kPairT * 5);
  int32_t* cols = reinterpret_cast<int32_t*>(rbase + kPairT * 5 + NMAX * 8);
  EntryMeta* meta = reinterpret_cast<EntryMeta*>(rbase + kPairT * 5 + NMAX * 12);
  const int64_t npairs = (rl.count + 1) >> 1;
  const Sweep sw(kPairWarps, warp);
  for (int64_t pidx = sw.first; pidx < npairs; pidx += sw.next(pidx)) {
    const int64_t ridx = 2 * pidx + half;
    bool live = ridx < rl.count;
    const int64_t row = live ? rl.row(ridx) : 0;
    int64_t base = 0;
    int n = 0;
    long long bound = 1;
    if (live) {
      if constexpr (SPEC) {
        const long long np = rpt[row];
        live = np > 0;  // no products: the symbolic kernel writes the 0
        bound = min(np, static_cast<long long>(NMAX));
      } else {
        live = !sp.done(row);  // rows done speculatively are copied by k_spec_copy
        if (live) {
          base = rpt[row];
          n = static_cast<int>(rpt[row + 1] - base);
          live = n > 0;
          bound = n;
        }
      }
    }
    int na = 0, len = 0;
    int32_t kmin = 0x7fffffff, kmax = -1;
    if (live) {
      const int64_t a0 = A.rpt[row];
      na = static_cast<int>(min(A.rpt[row + 1] - a0, static_cast<int64_t>(33)));
      for (int q = hl; q < min(na, 32); q += HG) {
        const int32_t k = A.col[a0 + q];
        const double av = A.val[a0 + q];
        const int64_t r0 = B.rpt[k];
        const int l = static_cast<int>(B.rpt[k + 1] - r0);
        meta[q] = EntryMeta{static_cast<int32_t>(r0), l, av};
        len = max(len, l);
        if (l > 0) {
          kmin = min(kmin, B.col[r0]);
          kmax = max(kmax, B.col[r0 + l - 1]);
        }
      }
    }
    len = half_max(len);
    kmin = half_min(kmin);
    kmax = half_max(kmax);
    if (na > 32 || len > 32) live = false;  // SPEC only: the row is left to the symbolic + generic kernels
    const int lg = min(LOG_T, max(2, ceil_log2_ll(2 * bound)));
    const uint32_t hshift = 32u - static_cast<uint32_t>(lg), hmask = (1u << lg) - 1u;
    const uint32_t mult = scale * 0x9E3779B1u;
    {
      int4* t4 = reinterpret_cast<int4*>(keys);
      for (int s = hl; s < (1 << lg) / 4; s += HG) t4[s] = make_int4(-1, -1, -1, -1);
    }
    if (!live) na = 0;
    const int steps = max(na, __shfl_xor_sync(kFull, na, 16));
    __syncwarp();
    int nk = 0;  // this row's claimed columns (uniform within the half)
    const int32_t* __restrict__ bcol = B.col;
    const double* __restrict__ bval = B.val;
    // loads of step j (B positions hl and hl + 16 of the entry's B row)
    auto load = [&](int j, int32_t& c0, double& v0, int32_t& c1, double& v1, double& a) {
      c0 = -1;
      c1 = -1;
      v0 = 0.0;
      v1 = 0.0;
      a = 0.0;
      if (j < na) {
        const EntryMeta mm = meta[j];
        a = mm.av;
        if (hl < mm.len) {
          c0 = bcol[mm.b0 + hl];
          v0 = bval[mm.b0 + hl];
        }
        if (hl + HG < mm.len) {
          c1 = bcol[mm.b0 + hl + HG];
          v1 = bval[mm.b0 + hl + HG];
        }
      }
    };
    // one step: both products of the lane (distinct columns of one B row)
    auto step = [&](double a, int32_t c0, double v0, int32_t c1, double v1) {
      const double x0 = __dmul_rn(a, v0), x1 = __dmul_rn(a, v1);
      uint32_t h0 = (static_cast<uint32_t>(c0) * mult) >> hshift;
      uint32_t h1 = (static_cast<uint32_t>(c1) * mult) >> hshift;
      int32_t k0 = c0 >= 0 ? keys[h0] : c0;
      int32_t k1 = c1 >= 0 ? keys[h1] : c1;
      bool f0 = false, f1 = false;
      if (__any_sync(kFull, k0 != c0)) {
        while (k0 != c0) {
          if (k0 == -1) {
            k0 = atomicCAS(reinterpret_cast<int*>(keys + h0), -1, c0);
            f0 = k0 == -1;
            if (f0) break;
          } else {
            h0 = (h0 + 1) & hmask;
            k0 = *reinterpret_cast<volatile int32_t*>(keys + h0);
          }
        }
      }
      if (__any_sync(kFull, k1 != c1)) {
        while (k1 != c1) {
          if (k1 == -1) {
            k1 = atomicCAS(reinterpret_cast<int*>(keys + h1), -1, c1);
            f1 = k1 == -1;
            if (f1) break;
          } else {
            h1 = (h1 + 1) & hmask;
            k1 = *reinterpret_cast<volatile int32_t*>(keys + h1);
          }
        }
      }
      const unsigned cb0 = __ballot_sync(kFull, f0) & hm, cb1 = __ballot_sync(kFull, f1) & hm;
      const int nc0 = __popc(cb0);
      const int claims = nc0 + __popc(cb1);
      if (SPEC && nk + claims > NMAX) {  // more columns than the scratch holds: abandon (no write past NMAX)
        nk = NMAX + 1;
        na = 0;
        return;
      }
      if (c0 >= 0) {
        const int ix = f0 ? nk + __popc(cb0 & hlt) : sidx[h0];
        const double prev = f0 ? 0.0 : vals[ix];
        vals[ix] = __dadd_rn(prev, x0);
        if (f0) {
          sidx[h0] = static_cast<uint8_t>(ix);
          cols[ix] = c0;
        }
      }
      if (c1 >= 0) {
        const int ix = f1 ? nk + nc0 + __popc(cb1 & hlt) : sidx[h1];
        const double prev = f1 ? 0.0 : vals[ix];
        vals[ix] = __dadd_rn(prev, x1);
        if (f1) {
          sidx[h1] = static_cast<uint8_t>(ix);
          cols[ix] = c1;
        }
      }
      nk += claims;
    };
    // two register sets, step j+1's loads in flight during step j
    int32_t pa0, pa1, pb0, pb1;
    double ua0, ua1, ub0, ub1, aa, ab;
    load(0, pa0, ua0, pa1, ua1, aa);
    for (int j = 0; j < steps; j += 2) {
      load(j + 1, pb0, ub0, pb1, ub1, ab);
      step(aa, pa0, ua0, pa1, ua1);
      __syncwarp();
      if (j + 1 >= steps) break;
      load(j + 2, pa0, ua0, pa1, ua1, aa);
      step(ab, pb0, ub0, pb1, ub1);
      __syncwarp();
    }
    if constexpr (SPEC) {
      if (nk > NMAX) live = false;  // abandoned
      n = nk;
    } else if (live && nk != n && hl == 0) {
      atomicOr(&info->error, kErrNumericCount);
    }
    if (!live) n = 0;
    // sort the n columns with their dense index; one network for both rows
    const bool narrow = static_cast<unsigned>(kmax - kmin) < (1u << 25);
    const bool narrow_all = __all_sync(kFull, narrow || !live);
    for (int e = hl; e < n; e += HG) {
      const int32_t c = cols[e];
      if (narrow_all) packed32[e] = (static_cast<uint32_t>(c - kmin) << 7) | static_cast<uint32_t>(e);
      else packed[e] = (static_cast<unsigned long long>(static_cast<uint32_t>(c)) << 32) | static_cast<uint32_t>(e);
    }
    const int nsel = max(n, __shfl_xor_sync(kFull, n, 16));
    __syncwarp();
    if (nsel > 0) {
      if (narrow_all) group_sort_padded<HG, E, uint32_t>(packed32, n, nsel, hl, kFull);
      else group_sort_padded<HG, E, unsigned long long>(packed, n, nsel, hl, kFull);
    }
    __syncwarp();
    if (live) {
      int32_t* ocol = SPEC ? sp.col + row * sp.cap : ccol + base;
      double* oval = SPEC ? sp.val + row * sp.cap : cval + base;
      for (int e = hl; e < n; e += HG) {
        int32_t c;
        uint32_t ix;
        if (narrow_all) {
          const uint32_t v = packed32[e];
          c = kmin + static_cast<int32_t>(v >> 7);
          ix = v & 127u;
        } else {
          const unsigned long long v = packed[e];
          c = static_cast<int32_t>(v >> 32);
          ix = static_cast<uint32_t>(v) & 127u;
        }
        ocol[e] = c;
        oval[e] = vals[ix];
      }
      if constexpr (SPEC) {
        if (hl == 0) {
          rpt[row] = n;
          sp.flag[row] = 1;
        }
      }
    }
    __syncwarp();
  }
}

// Structure-reuse numeric for warp-sized rows, one row at a time: the
// speculative numeric of the symbolic phase (SPEC) for C = A*A-shaped products
// outside the reuse route; the reuse route itself runs k_num_reuse_multi
// (kernels_reuse.cuh). One warp per row, a warp takes kReuseRows consecutive rows of its bin.
// Row i's output STRUCTURE is that of the warp's previous row i' shifted by
// d = k_1(i) - k_1(i') exactly when both rows have the same number of A
// entries, entry j's B rows have the same length, and every product column
// satisfies B(k_j(i), q) - B(k_j(i'), q) = d (with k_j(i) - k_j(i') = d): then
// the products group into columns the same way, in the same sorted order.
// The check is exact (every product is compared), so any matrix is handled;
// translation-invariant structure (interior rows of a grid stencil) passes it.
// A row that passes skips hashing, claiming and sorting: product (j, q) adds
// into vals[map[j][q]] -- its output position recorded for row i' -- one A
// entry per step with __syncwarp between steps (per column the reference's
// A-row order, starting from +0.0), and C(i,:) is written as
// (cols(i') + d, vals). A row that fails (or the warp's first row) takes the
// full path -- the dense-index column table of k_num_lean -- and records the
// map for the next row. Numeric launches are made only when A's and B's
// longest rows are <= 32 (K1); a speculative row outside that, or with more
// than NMAX columns, is abandoned (left to the symbolic kernel).
#ifndef SPGEMM_REUSE_U
#define SPGEMM_REUSE_U 4      // steps' value loads in flight in the reuse path
#endif
#ifndef SPGEMM_REUSE_MINB
#define SPGEMM_REUSE_MINB 4   // resident blocks per SM (64 registers)
#endif
constexpr int kReuseWarps = 8;
constexpr int kReuseRows = 32;  // consecutive rows per warp (power of two)
constexpr size_t kReuseWarpBytes = 256 * 4 + 256 + 128 * 8 + 128 * 4 + 128 * 4 + 2 * 32 * 16 + 32 * 32 * 2;  // 6400
// the map holds 16-bit shared-window addresses: the block's window must stay below 64 KB
static_assert(kReuseWarps * kReuseWarpBytes + 1024 < 65536, "k_num_reuse map addresses are 16-bit");
template <bool SPEC>
__global__ void __launch_bounds__(32 * kReuseWarps, SPGEMM_REUSE_MINB)
    k_num_reuse(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, int32_t* __restrict__ ccol,
                double* __restrict__ cval, uint32_t scale, DevInfo* info, Spec sp, int rows_per_warp,
                const uint8_t* __restrict__ shift1) {
  constexpr int G = 32, NMAX = 128, T = 256, E = 4;
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = smem_raw + static_cast<size_t>(warp) * kReuseWarpBytes;
  int32_t* keys = reinterpret_cast<int32_t*>(wb);             // [T]; after the walk: sort keys
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(wb);
  uint32_t* packed32 = reinterpret_cast<uint32_t*>(wb);
  uint8_t* sidx = wb + T * 4;                                 // [T] dense index per slot; after: rank
  double* vals = reinterpret_cast<double*>(wb + T * 5);       // [NMAX]
  int32_t* cols = reinterpret_cast<int32_t*>(wb + T * 5 + NMAX * 8);      // [NMAX] claim order
  int32_t* ocols = reinterpret_cast<int32_t*>(wb + T * 5 + NMAX * 12);    // [NMAX] previous row's output
  EntryMeta* metab = reinterpret_cast<EntryMeta*>(wb + T * 5 + NMAX * 16);  // [2][32]
  // [32][32] product -> the shared address of its output's accumulator (during
  // the full path's walk: the product's dense index)
  uint16_t* map = reinterpret_cast<uint16_t*>(wb + T * 5 + NMAX * 16 + 2 * 32 * 16);
  const uint32_t vals_sa = static_cast<uint32_t>(__cvta_generic_to_shared(vals));
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t mult = scale * 0x9E3779B1u;
  // previous row (warp-uniform except the per-lane entry fields)
  bool pvalid = false;
  int pna = 0, pn = 0, mb = 0;
  int32_t pk = 0;
  int plen = 0;
  // runs of R (<= kReuseRows, a power of two) consecutive rows per warp per
  // sweep: as many as keep every warp busy, from the bin's size read on the
  // device (rows_per_warp > 0 overrides)
  int64_t R = rows_per_warp;
  if (R <= 0) {
    const int64_t warps = static_cast<int64_t>(gridDim.x) * kReuseWarps;
    R = kReuseRows;
    while (R > 1 && rl.count < warps * R) R >>= 1;
  }
  const int64_t first = (static_cast<int64_t>(blockIdx.x) * kReuseWarps + warp) * R;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kReuseWarps * R;
  unsigned nreuse = 0, nfull = 0;  // rows through each path (DevInfo counters)
  for (int64_t run0 = first; run0 < rl.count; run0 += stride) {
   // the run's row ids and skip tests, 32 at a time; then its rows in order
   // the run's row ids, skip tests, C offsets / nprod and A-row bounds, one row per lane
   int64_t lrow = -1, lbase = 0, lnext = 0, la0 = 0, la1 = 0;
   bool need = false;
   if (lane < R && run0 + lane < rl.count) {
     lrow = rl.row(run0 + lane);
     lbase = rpt[lrow];
     if constexpr (SPEC) {
       need = lbase != 0;  // no products: the symbolic kernel writes the 0
     } else {
       lnext = rpt[lrow + 1];
       need = !sp.done(lrow) && lnext > lbase;  // done speculatively (k_spec_copy) or empty
     }
     if (need) {
       la0 = A.rpt[lrow];
       la1 = A.rpt[lrow + 1];
     }
   }
   unsigned todo = __ballot_sync(kFull, need);
   while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1u;
    const int64_t row = __shfl_sync(kFull, lrow, src);
    int64_t base = 0;
    int n = 0;
    long long bound;
    if constexpr (SPEC) {
      const long long np = __shfl_sync(kFull, lbase, src);
      bound = min(np, static_cast<long long>(NMAX));
    } else {
      base = __shfl_sync(kFull, lbase, src);
      n = static_cast<int>(__shfl_sync(kFull, lnext, src) - base);
      bound = n;
    }
    EntryMeta* meta = metab + mb * 32;
    const EntryMeta* pmeta = metab + (mb ^ 1) * 32;
    const int64_t a0 = __shfl_sync(kFull, la0, src);
    const int na = static_cast<int>(min(__shfl_sync(kFull, la1, src) - a0, static_cast<int64_t>(33)));
    int len = 0;
    int32_t k = 0;
    double av = 0.0;
    int32_t b0 = 0;
    if (lane < na) {
      k = A.col[a0 + lane];
      av = A.val[a0 + lane];
      const int64_t r0 = B.rpt[k];
      len = static_cast<int>(B.rpt[k + 1] - r0);
      b0 = static_cast<int32_t>(r0);
    }
    meta[lane] = EntryMeta{b0, len, av};  // rows j >= na: len 0 (the reuse loop's padding)
    const int maxlen = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(len)));
    if (na > G || maxlen > G) {  // (speculative rows only) left to the symbolic + generic kernels
      pvalid = false;
      continue;
    }
    __syncwarp();
    // ---- reuse path
    const int32_t d = __shfl_sync(kFull, k, 0) - __shfl_sync(kFull, pk, 0);
    bool reuse = pvalid && na == pna && (SPEC || n == pn) &&
                 __all_sync(kFull, lane >= na || (len == plen && k - pk == d));
    if (reuse) {
      bool ok = true;
      if (d == 1 && shift1 != nullptr && __all_sync(kFull, lane >= na || shift1[k] != 0)) {
        // every B row of the row is its predecessor shifted by one column
        // (precomputed per B row): the structure matches without a per-product
        // check, and the columns need not be loaded -- only the values, U
        // steps' loads in flight at once, their updates in step order
        // Branch-free: a lane without a product in a step adds 0.0 into the
        // spare slot vals[NMAX] (it overlays cols[0..1], unused on this path).
        constexpr int U = SPGEMM_REUSE_U;
        static_assert(G % U == 0, "U must divide the warp width (meta/map rows >= na are padding)");
        // per-lane base pointer: a step's address is one 32x32->64 multiply-add
        const char* bvl = reinterpret_cast<const char*>(B.val + lane);
        const uint16_t* mapl = map + lane;
        // accumulators start at +0.0 (the reference's fold starts from 0.0)
        for (int e = lane; e < pn; e += G) vals[e] = 0.0;
        __syncwarp();
#pragma unroll 1
        for (int j0 = 0; j0 < na; j0 += U) {
          const EntryMeta* mj = meta + j0;
          const uint16_t* mp = mapl + j0 * G;
          double bv[U], av[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            // rows j >= na: len 0 (their map rows are all spare)
            const EntryMeta m = mj[u];
            av[u] = m.av;
            bv[u] = ldg_f64_if(bvl + static_cast<size_t>(static_cast<uint32_t>(m.b0)) * 8u, lane < m.len);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            // a lane without a product (lane >= len, or j >= na) maps to the
            // spare slot vals[NMAX] (it overlays cols[0..1], unused here); the
            // volatile shared accesses keep the steps in order (the warp is
            // converged: no branch inside the loop)
            const uint32_t a = mp[u * G];
            sts_f64(a, __dadd_rn(lds_f64(a), __dmul_rn(av[u], bv[u])));
          }
        }
        __syncwarp();
      } else {
        for (int e = lane; e < pn; e += G) vals[e] = 0.0;
        __syncwarp();
        for (int j = 0; j < na; ++j) {
          const EntryMeta m = meta[j];
          if (lane < m.len) {
            const int32_t c = B.col[m.b0 + lane];
            const int32_t cp = B.col[pmeta[j].b0 + lane];
            const double x = __dmul_rn(m.av, B.val[m.b0 + lane]);
            ok = ok && c - cp == d;
            const uint32_t a = map[j * G + lane];
            sts_f64(a, __dadd_rn(lds_f64(a), x));
          }
          __syncwarp();
          if (!__all_sync(kFull, ok)) break;  // structure differs: stop early (the full path recomputes)
        }
      }
      if (__all_sync(kFull, ok)) {
        n = pn;
        int32_t* ocp = SPEC ? sp.col + row * sp.cap : ccol + base;
        double* ovp = SPEC ? sp.val + row * sp.cap : cval + base;
        for (int e = lane; e < n; e += G) {
          const int32_t c = ocols[e] + d;
          ocols[e] = c;
          ocp[e] = c;
          ovp[e] = vals[e];
        }
        if constexpr (SPEC) {
          if (lane == 0) {
            rpt[row] = n;
            sp.flag[row] = 1;
          }
        }
        pk = k;
        plen = len;
        mb ^= 1;
        ++nreuse;
        __syncwarp();
        continue;
      }
      __syncwarp();  // structure differs after all: the full path below
    }
    // ---- full path: dense-index column table
    int32_t kmin = 0x7fffffff, kmax = -1;
    if (lane < na && len > 0) {
      kmin = B.col[b0];
      kmax = B.col[b0 + len - 1];
    }
    kmin = static_cast<int32_t>(__reduce_min_sync(kFull, static_cast<unsigned>(kmin)));
    kmax = static_cast<int32_t>(__reduce_max_sync(kFull, static_cast<unsigned>(kmax + 1))) - 1;
    const int lg = min(log2_const<T>(), max(2, ceil_log2_ll(2 * bound)));
    const uint32_t hshift = 32u - static_cast<uint32_t>(lg), hmask = (1u << lg) - 1u;
    fill_empty<G>(keys, 1 << lg, lane);
    __syncwarp();
    int nk = 0;
    for (int j = 0; j < na; ++j) {
      const EntryMeta m = meta[j];
      const int32_t c = lane < m.len ? B.col[m.b0 + lane] : -1;
      const double x = lane < m.len ? __dmul_rn(m.av, B.val[m.b0 + lane]) : 0.0;
      uint32_t h = (static_cast<uint32_t>(c) * mult) >> hshift;
      int32_t cur = c >= 0 ? keys[h] : c;
      bool fresh = false;
      if (__any_sync(kFull, cur != c)) {
        while (cur != c) {
          if (cur == -1) {
            cur = atomicCAS(reinterpret_cast<int*>(keys + h), -1, c);
            fresh = cur == -1;
            if (fresh) break;
          } else {
            h = (h + 1) & hmask;
            cur = *reinterpret_cast<volatile int32_t*>(keys + h);
          }
        }
      }
      const unsigned cb = __ballot_sync(kFull, fresh);
      if (SPEC && nk + __popc(cb) > NMAX) {  // more columns than the scratch holds: abandon
        nk = NMAX + 1;
        break;
      }
      if (c >= 0) {
        const int ix = fresh ? nk + __popc(cb & lt) : sidx[h];
        const double prev = fresh ? 0.0 : vals[ix];
        vals[ix] = __dadd_rn(prev, x);
        map[j * G + lane] = static_cast<uint16_t>(ix);
        if (fresh) {
          sidx[h] = static_cast<uint8_t>(ix);
          cols[ix] = c;
        }
      }
      nk += __popc(cb);
      __syncwarp();
    }
    __syncwarp();
    if constexpr (SPEC) {
      if (nk > NMAX) {
        pvalid = false;
        continue;  // abandoned (uniform): the symbolic kernel counts this row
      }
      n = nk;
    } else if (nk != n && lane == 0) {
      atomicOr(&info->error, kErrNumericCount);
    }
    // sort the n columns with their dense index; rank[] and the sorted columns
    const bool narrow = static_cast<unsigned>(kmax - kmin) < (1u << 25);
    for (int e = lane; e < n; e += G) {
      const int32_t c = cols[e];
      if (narrow) packed32[e] = (static_cast<uint32_t>(c - kmin) << 7) | static_cast<uint32_t>(e);
      else packed[e] = (static_cast<unsigned long long>(static_cast<uint32_t>(c)) << 32) | static_cast<uint32_t>(e);
    }
    __syncwarp();
    if (narrow) group_sort_inplace<G, E, uint32_t>(packed32, n, lane, kFull);
    else group_sort_inplace<G, E, unsigned long long>(packed, n, lane, kFull);
    __syncwarp();
    int32_t* ocp = SPEC ? sp.col + row * sp.cap : ccol + base;
    double* ovp = SPEC ? sp.val + row * sp.cap : cval + base;
    uint8_t* rank = sidx;
    for (int e = lane; e < n; e += G) {
      int32_t c;
      uint32_t ix;
      if (narrow) {
        const uint32_t v = packed32[e];
        c = kmin + static_cast<int32_t>(v >> 7);
        ix = v & 127u;
      } else {
        const unsigned long long v = packed[e];
        c = static_cast<int32_t>(v >> 32);
        ix = static_cast<uint32_t>(v) & 127u;
      }
      ocp[e] = c;
      ovp[e] = vals[ix];
      ocols[e] = c;
      rank[ix] = static_cast<uint8_t>(e);
    }
    __syncwarp();
    // product -> output position for the next row; map rows j >= na and lanes
    // past a B row's length point at the spare slot NMAX
    for (int j = 0; j < G; ++j) {
      const int lj = __shfl_sync(kFull, len, j);
      map[j * G + lane] = static_cast<uint16_t>(vals_sa + 8u * ((j < na && lane < lj) ? rank[map[j * G + lane]] : NMAX));
    }
    __syncwarp();
    if constexpr (SPEC) {
      if (lane == 0) {
        rpt[row] = n;
        sp.flag[row] = 1;
      }
    }
    pvalid = true;
    pna = na;
    pn = n;
    pk = k;
    plen = len;
    mb ^= 1;
    ++nfull;
    __syncwarp();
   }
  }
  if (lane == 0 && (nreuse | nfull)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&info->reuse_rows), static_cast<unsigned long long>(nreuse));
    atomicAdd(reinterpret_cast<unsigned long long*>(&info->full_rows), static_cast<unsigned long long>(nfull));
  }
}

// Symbolic phase of the structure-reuse route (A*A-shaped products with
// warp-sized A and B rows, e.g. 3-D stencils): nnz(C(i,:)) = nnz(C(i-1,:))
// whenever row i is flagged by k_reuse_flags (its structure is row i-1's
// shifted by one: kernels_reuse.cuh). Only unflagged rows count their distinct
// columns, with a 1024-slot table (a symbolic bin of <= 1024 products cannot
// fill it). No values, no sort: the numeric phase (k_num_reuse_multi) then
// writes C in place -- no speculative scratch, no copy.
constexpr int kSymReuseWarps = 8;
constexpr int kSymReuseT = 1024;
constexpr size_t kSymReuseWarpBytes = kSymReuseT * 4 + 2 * 32 * 16;
__global__ void __launch_bounds__(32 * kSymReuseWarps)
    k_sym_reuse(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, uint32_t scale, int rows_per_warp,
                const uint8_t* __restrict__ rflag, DevInfo* info) {
  // A warp takes runs of 32 consecutive rows of the bin, one row per lane: a
  // flagged row whose predecessor in the bin (lane - 1; lane 0: the previous
  // piece's last row) is row - 1 has that row's count; the others ("heads")
  // count their distinct columns, warp-cooperatively, and the counts are
  // copied forward lane to lane.
  constexpr int G = 32;
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = smem_raw + static_cast<size_t>(warp) * kSymReuseWarpBytes;
  int32_t* keys = reinterpret_cast<int32_t*>(wb);
  const uint32_t mult = scale * 0x9E3779B1u;
  // runs of R consecutive bin rows per warp, taken in pieces of min(R, 32);
  // the count carries over between the pieces. R follows the bin's size (read
  // on the device): 32*S rows (S <= 8) while every warp stays busy, shorter
  // runs for small bins. (rows_per_warp > 0 overrides.)
  int64_t R = rows_per_warp;
  if (R <= 0) {
    const int64_t warps = static_cast<int64_t>(gridDim.x) * kSymReuseWarps;
    R = 32 * max(1ll, min(8ll, static_cast<long long>(rl.count / (warps * 32))));
    while (R > 4 && rl.count < warps * R) R >>= 1;
  }
  bool cvalid = false;  // the previous piece's last row (warp-uniform)
  int64_t c_row = -2;
  long long c_n = 0;
  long long nreuse = 0, nfull = 0;
  const int64_t first = (static_cast<int64_t>(blockIdx.x) * kSymReuseWarps + warp) * R;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kSymReuseWarps * R;
  const int P = static_cast<int>(min(static_cast<int64_t>(G), R));  // rows per piece (R: a multiple of P)
  for (int64_t run0 = first; run0 < rl.count; run0 += (run0 - first) % R + P >= R ? stride - (R - P) : P) {
    if ((run0 - first) % R == 0) cvalid = false;  // a new run: its first row is a head
    const bool valid = lane < P && run0 + lane < rl.count;
    int64_t row = -1, a0 = 0;
    long long np = 0;
    int na = 0;
    bool fl = false;
    if (valid) {
      row = rl.row(run0 + lane);
      np = rpt[row];
      a0 = A.rpt[row];
      na = static_cast<int>(A.rpt[row + 1] - a0);
      fl = rflag[row] != 0;
    }
    // the predecessor in the bin: lane - 1, or the previous run's last row; a
    // flagged row whose predecessor is row - 1 has its count
    int64_t p_row = __shfl_up_sync(kFull, row, 1);
    bool p_ok = __shfl_up_sync(kFull, valid && np != 0, 1);
    if (lane == 0) {
      p_row = c_row;
      p_ok = cvalid;
    }
    const bool same = valid && np != 0 && p_ok && fl && p_row + 1 == row;
    const unsigned heads = __ballot_sync(kFull, valid && !same);
    long long n = 0;
    // heads: count distinct columns (a row without products: 0)
    for (unsigned hm = heads; hm;) {
      const int h = __ffs(hm) - 1;
      hm &= hm - 1u;
      const long long hnp = __shfl_sync(kFull, np, h);
      long long cnt_total = 0;
      if (hnp != 0) {
        const int64_t ha0 = __shfl_sync(kFull, a0, h);
        const int hna = __shfl_sync(kFull, na, h);
        const int tsz = static_cast<int>(min(static_cast<long long>(kSymReuseT),
                                             static_cast<long long>(1) << ceil_log2_ll(2 * hnp)));
        const int lg = max(2, 31 - __clz(tsz));
        const uint32_t hshift = 32u - static_cast<uint32_t>(lg), hmask = (1u << lg) - 1u;
        fill_empty<G>(keys, 1 << lg, lane);
        // the head row's entries: their B rows, loaded by the lanes at once
        int64_t hb0 = 0, hb1 = 0;
        if (lane < hna) {
          const int32_t k = A.col[ha0 + lane];
          hb0 = B.rpt[k];
          hb1 = B.rpt[k + 1];
        }
        __syncwarp();
        int cnt = 0;
        auto insert = [&](int32_t c) {
          uint32_t hh = (static_cast<uint32_t>(c) * mult) >> hshift;
          int32_t cur = keys[hh];
          while (cur != c) {
            if (cur == -1) {
              cur = atomicCAS(reinterpret_cast<int*>(keys + hh), -1, c);
              if (cur == -1) {
                ++cnt;
                break;
              }
            } else {
              hh = (hh + 1) & hmask;
              cur = *reinterpret_cast<volatile int32_t*>(keys + hh);
            }
          }
        };
        const int hlen = static_cast<int>(hb1 - hb0);
        if (__reduce_max_sync(kFull, static_cast<unsigned>(hlen)) <= static_cast<unsigned>(G) &&
            __shfl_sync(kFull, hb1, max(hna - 1, 0)) < (int64_t(1) << 31)) {
          // B rows of <= 32 entries (the route's rows): 8 entries' columns loaded
          // before any is inserted (one latency per 8 entries, not per entry)
          const int32_t hb = static_cast<int32_t>(hb0);
          for (int j0 = 0; j0 < hna; j0 += 8) {
            int32_t c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int j = (j0 + u) & 31;
              const int32_t bj = __shfl_sync(kFull, hb, j);
              const int lj = __shfl_sync(kFull, hlen, j);
              c[u] = (j0 + u < hna && lane < lj) ? B.col[bj + lane] : -1;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (c[u] >= 0) insert(c[u]);
          }
        } else {
          for (int j = 0; j < hna; ++j) {
            const int64_t q1 = __shfl_sync(kFull, hb1, j);
            for (int64_t q = __shfl_sync(kFull, hb0, j) + lane; q < q1; q += G) insert(B.col[q]);
          }
        }
        cnt_total = static_cast<long long>(__reduce_add_sync(kFull, static_cast<unsigned>(cnt)));
        __syncwarp();
        ++nfull;
      }
      if (lane == h) n = cnt_total;
    }
    // copy the counts forward: a row that passed takes the last head's count
    // before it (or, with no head before it, the previous run's last row's)
    int src = (heads >> lane) & 1u ? lane : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, src, o);
      if (lane >= o) src = max(src, y);
    }
    const long long from_head = __shfl_sync(kFull, n, max(src, 0));
    if (src < 0) n = c_n;
    else n = from_head;
    if (valid) {
      rpt[row] = n;
      if (same) ++nreuse;
    }
    // carry the run's last row
    const int last = static_cast<int>(min(static_cast<long long>(P), static_cast<long long>(rl.count - run0))) - 1;
    c_row = __shfl_sync(kFull, row, last);
    c_n = __shfl_sync(kFull, n, last);
    cvalid = __shfl_sync(kFull, valid && np != 0, last);
  }
  nreuse = static_cast<long long>(__reduce_add_sync(kFull, static_cast<unsigned>(nreuse)));
  if (lane == 0 && (nreuse | nfull)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&info->reuse_rows), static_cast<unsigned long long>(nreuse));
    atomicAdd(reinterpret_cast<unsigned long long*>(&info->full_rows), static_cast<unsigned long long>(nfull));
  }
}

// shift1[k] = 1 when B row k is B row k-1 shifted by one column (same length,
// every column one larger): the per-B-row precondition that lets k_num_reuse
// accept a row adjacent to its predecessor (d = 1) without comparing every
// product's column. Thread per row (a warp-per-32-rows variant with coalesced
// entry loads measured slower: 0.17 vs 0.12 ms on the 27-point stencil).
__global__ void __launch_bounds__(256)
    k_shift_flags(DevCsr B, uint8_t* __restrict__ shift1) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < B.rows; k += stride) {
    bool same = false;
    if (k > 0) {
      const int64_t r0 = B.rpt[k - 1], r1 = B.rpt[k], r2 = B.rpt[k + 1];
      const int64_t len = r2 - r1;
      same = len == r1 - r0;
      // 16 entries per round, their loads issued before any is compared (rows
      // of <= 32 entries: at most two rounds, the second not waiting on the first)
      bool ok = same;
      for (int64_t q0 = 0; same && q0 < len; q0 += 16) {
        int32_t c[16], cp[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const bool on = q0 + u < len;
          c[u] = on ? B.col[r1 + q0 + u] : 1;
          cp[u] = on ? B.col[r0 + q0 + u] : 0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) ok = ok & (c[u] == cp[u] + 1);
      }
      same = ok;
    }
    shift1[k] = same ? 1 : 0;
  }
}

// In-place bitonic sort of np (pow2) packed keys in shared memory by a block.
template <int THREADS>
__device__ __forceinline__ void block_bitonic_smem(unsigned long long* a, int np) {
  for (int k = 2; k <= np; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (np >> 1); i += THREADS) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo + j;
        const bool up = (lo & k) == 0;
        const unsigned long long x = a[lo], y = a[hi];
        if ((x > y) == up) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
  }
}

// Block kernel: one row per block iteration, table of T slots in shared
// memory, ordered steps with a block barrier per A entry.
// OVERLAY (the B200 tier for rows of up to 8192 nonzeros: T = 16384 slots,
// 128 KB of values + 64 KB of keys): the sort keys overlay the table's keys --
// the condense step reads every thread's slots into registers before the
// block-wide scan, so the packed (column, slot) keys can be written over them;
// 192 KB per block instead of 256 KB.
template <int T, int THREADS, int NMAX, bool OVERLAY = false>
__global__ void __launch_bounds__(THREADS)
    k_num_block(RowList rl_in, DevCsr A, DevCsr B, const int64_t* __restrict__ rpt,
                int32_t* __restrict__ ccol, double* __restrict__ cval, uint32_t scale,
                DevInfo* info) {
  static_assert(!OVERLAY || NMAX * 8 <= T * 4, "the sort keys must fit the table's keys");
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* vals = reinterpret_cast<double*>(smem_raw);
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(smem_raw + T * 8);
  int32_t* keys = reinterpret_cast<int32_t*>(smem_raw + T * 8 + (OVERLAY ? 0 : NMAX * 8));
  __shared__ long long s_red[32];
  constexpr int PER = T / THREADS;
  const Hash hs = make_hash(scale, log2_const<T>());
  for (int64_t idx = blockIdx.x; idx < rl.count; idx += gridDim.x) {
    const int64_t row = rl.row(idx);
    const int64_t base = rpt[row];
    const int n = static_cast<int>(rpt[row + 1] - base);
    if (n == 0) continue;
    for (int s = threadIdx.x; s < T; s += THREADS) {
      keys[s] = -1;
      vals[s] = 0.0;
    }
    __syncthreads();
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    for (int64_t p = a0; p < a1; ++p) {
      const int32_t k = A.col[p];
      const double av = A.val[p];
      const int64_t b1 = B.rpt[k + 1];
      for (int64_t q = B.rpt[k] + threadIdx.x; q < b1; q += THREADS) {
        const double x = __dmul_rn(av, B.val[q]);
        const uint32_t s = num_slot(keys, B.col[q], hs);
        vals[s] = __dadd_rn(vals[s], x);
      }
      __syncthreads();
    }
    // condense: each thread owns PER consecutive slots (read into registers
    // first: with OVERLAY the packed keys are written over the table's keys)
    int32_t kv[PER];
    int mine = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      kv[i] = keys[threadIdx.x * PER + i];
      mine += kv[i] != -1;
    }
    long long total;
    long long pos = block_exclusive_scan<THREADS>(mine, s_red, &total);
    if constexpr (OVERLAY) __syncthreads();  // every thread's slots read before any packed write
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int s = threadIdx.x * PER + i;
      if (kv[i] != -1)
        packed[pos++] = (static_cast<unsigned long long>(static_cast<uint32_t>(kv[i])) << 32) |
                        static_cast<uint32_t>(s);
    }
    if (threadIdx.x == 0 && total != n) atomicOr(&info->error, kErrNumericCount);
    int np = 1;
    while (np < n) np <<= 1;
    for (int e = n + threadIdx.x; e < np; e += THREADS) packed[e] = ~0ull;
    __syncthreads();
    block_bitonic_smem<THREADS>(packed, np);
    for (int e = threadIdx.x; e < n; e += THREADS) {
      const unsigned long long v = packed[e];
      ccol[base + e] = static_cast<int32_t>(v >> 32);
      cval[base + e] = vals[static_cast<uint32_t>(v)];
    }
    __syncthreads();
  }
}

// Heap tier (pipeline.cpp:396-410): rows past the largest shared tier.
// Table of bit_ceil(2*nnz) slots in a per-block region of a global pool,
// ordered steps, then the row's columns are ranked without a comparison
// sort: a bitmap over a window of the column range plus an exclusive popcount
// scan gives each entry its output position directly (columns are distinct).
constexpr int kGlobalThreads = 512;
__global__ void __launch_bounds__(kGlobalThreads)
    k_num_global(RowList rl_in, DevCsr A, DevCsr B, const int64_t* __restrict__ rpt,
                 int32_t* __restrict__ ccol, double* __restrict__ cval, uint32_t scale,
                 int32_t* __restrict__ pool_keys, double* __restrict__ pool_vals,
                 uint32_t* __restrict__ pool_bits, int64_t slots_per_block, int64_t words_per_block,
                 DevInfo* info) {
  const RowList rl = rl_in.resolved();
  __shared__ long long s_red[32];
  __shared__ int s_min, s_max;
  int32_t* keys = pool_keys + static_cast<int64_t>(blockIdx.x) * slots_per_block;
  double* vals = pool_vals + static_cast<int64_t>(blockIdx.x) * slots_per_block;
  uint32_t* bits = pool_bits + static_cast<int64_t>(blockIdx.x) * 2 * words_per_block;
  uint32_t* pref = bits + words_per_block;
  for (int64_t idx = blockIdx.x; idx < rl.count; idx += gridDim.x) {
    const int64_t row = rl.row(idx);
    const int64_t base = rpt[row];
    const int64_t n = rpt[row + 1] - base;
    if (n == 0) continue;
    int64_t t = 2;
    while (t < 2 * n) t <<= 1;
    if (t > slots_per_block) t = slots_per_block;
    int lg = 0;
    while ((1ll << lg) < t) ++lg;
    const Hash hs = make_hash(scale, lg);
    for (int64_t s = threadIdx.x; s < t; s += kGlobalThreads) {
      keys[s] = -1;
      vals[s] = 0.0;
    }
    if (threadIdx.x == 0) {
      s_min = 0x7fffffff;
      s_max = -1;
    }
    __syncthreads();
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    for (int64_t p = a0; p < a1; ++p) {
      const int32_t k = A.col[p];
      const double av = A.val[p];
      const int64_t b1 = B.rpt[k + 1];
      for (int64_t q = B.rpt[k] + threadIdx.x; q < b1; q += kGlobalThreads) {
        const double x = __dmul_rn(av, B.val[q]);
        const uint32_t s = num_slot(keys, B.col[q], hs);
        vals[s] = __dadd_rn(vals[s], x);
      }
      __syncthreads();
    }
    int lmin = 0x7fffffff, lmax = -1;
    for (int64_t s = threadIdx.x; s < t; s += kGlobalThreads) {
      const int32_t key = keys[s];
      if (key != -1) {
        lmin = min(lmin, key);
        lmax = max(lmax, key);
      }
    }
    atomicMin(&s_min, lmin);
    atomicMax(&s_max, lmax);
    __syncthreads();
    const int64_t kmin = s_min, kmax = s_max;
    const int64_t wbits = words_per_block * 32;
    int64_t written = 0;
    for (int64_t w0 = kmin; w0 <= kmax; w0 += wbits) {
      const int64_t span = min(wbits, kmax - w0 + 1);
      const int64_t nwords = (span + 31) / 32;
      for (int64_t w = threadIdx.x; w < nwords; w += kGlobalThreads) bits[w] = 0u;
      __syncthreads();
      for (int64_t s = threadIdx.x; s < t; s += kGlobalThreads) {
        const int32_t key = keys[s];
        if (key != -1 && key >= w0 && key < w0 + span) {
          const int64_t off = key - w0;
          atomicOr(&bits[off >> 5], 1u << (off & 31));
        }
      }
      __syncthreads();
      // exclusive popcount scan over nwords, each thread a contiguous chunk
      const int64_t per = (nwords + kGlobalThreads - 1) / kGlobalThreads;
      const int64_t w_lo = min(nwords, threadIdx.x * per), w_hi = min(nwords, w_lo + per);
      long long mine = 0;
      for (int64_t w = w_lo; w < w_hi; ++w) mine += __popc(bits[w]);
      long long wtotal;
      long long run = block_exclusive_scan<kGlobalThreads>(mine, s_red, &wtotal);
      for (int64_t w = w_lo; w < w_hi; ++w) {
        pref[w] = static_cast<uint32_t>(run);
        run += __popc(bits[w]);
      }
      __syncthreads();
      for (int64_t s = threadIdx.x; s < t; s += kGlobalThreads) {
        const int32_t key = keys[s];
        if (key != -1 && key >= w0 && key < w0 + span) {
          const int64_t off = key - w0;
          const uint32_t word = bits[off >> 5];
          const int64_t pos =
              written + pref[off >> 5] + __popc(word & ((1u << (off & 31)) - 1u));
          ccol[base + pos] = key;
          cval[base + pos] = vals[s];
        }
      }
      written += wtotal;
      __syncthreads();
    }
    if (threadIdx.x == 0 && written != n) atomicOr(&info->error, kErrNumericCount);
    __syncthreads();
  }
}

// Numeric phase, first launch: the rows finished speculatively in the symbolic
// phase are copied from the scratch into C. A warp takes 32 consecutive rows:
// flags and row pointers load coalesced, then the lanes copy two rows at a
// time with every load of both rows (<= kSpecCap entries each) issued before
// the first store -- 16 independent loads per lane in flight.
__global__ void __launch_bounds__(256)
    k_spec_copy(Spec sp, const int64_t* __restrict__ rpt, int64_t M, int32_t* __restrict__ ccol,
                double* __restrict__ cval) {
  constexpr int kIt = kSpecCap / 32;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int32_t* __restrict__ scol = sp.col;
  const double* __restrict__ sval = sp.val;
  for (int64_t r0 = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; r0 < M;
       r0 += warps * 32) {
    const int64_t r = r0 + lane;
    const bool mine = r < M && sp.flag[r] != 0;
    const int64_t base = mine ? rpt[r] : 0;
    const int n = mine ? static_cast<int>(rpt[r + 1] - base) : 0;
    unsigned todo = __ballot_sync(kFull, mine && n > 0);
    while (todo) {
      int64_t b[2], s0[2];
      int nn[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int l = todo ? __ffs(todo) - 1 : 0;
        const bool have = todo != 0;
        todo &= todo - 1u;
        b[k] = __shfl_sync(kFull, base, l);
        nn[k] = have ? __shfl_sync(kFull, n, l) : 0;
        s0[k] = (r0 + l) * kSpecCap;
      }
      int32_t c[2][kIt];
      double v[2][kIt];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < kIt; ++i) {
          const int e = lane + 32 * i;
          c[k][i] = e < nn[k] ? scol[s0[k] + e] : 0;
          v[k][i] = e < nn[k] ? sval[s0[k] + e] : 0.0;
        }
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int i = 0; i < kIt; ++i) {
          const int e = lane + 32 * i;
          if (e < nn[k]) {
            ccol[b[k] + e] = c[k][i];
            cval[b[k] + e] = v[k][i];
          }
        }
    }
  }
}

// Checksums of a device CSR (streamed products): warp per row, sum of values
// (fp64) and of (col + c0 + 1) * (row + r0 + 1) mod 2^64.
__global__ void __launch_bounds__(256)
    k_checksum(const int64_t* __restrict__ rpt, const int32_t* __restrict__ col, const double* __restrict__ val,
               int64_t rows, int64_t r0, int64_t c0, double* vsum, unsigned long long* hsum) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  double v = 0.0;
  unsigned long long h = 0;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    const unsigned long long rr = static_cast<unsigned long long>(r + r0 + 1);
    unsigned long long hc = 0;
    const int64_t e1 = rpt[r + 1];
    int64_t e = rpt[r] + lane;
    for (; e + 96 < e1; e += 128) {  // four independent loads in flight per lane
      const int32_t c0_ = col[e], c1_ = col[e + 32], c2_ = col[e + 64], c3_ = col[e + 96];
      const double v0 = val[e], v1 = val[e + 32], v2 = val[e + 64], v3 = val[e + 96];
      hc += static_cast<unsigned long long>(c0_) + c1_ + c2_ + c3_ + 4 * (c0 + 1);
      v += (v0 + v1) + (v2 + v3);
    }
    for (; e < e1; e += 32) {
      hc += static_cast<unsigned long long>(col[e] + c0 + 1);
      v += val[e];
    }
    h += hc * rr;
  }
  v = warp_sum(v);
  h = warp_sum(h);
  if (lane == 0) {
    atomicAdd(vsum, v);
    atomicAdd(hsum, h);
  }
}

}  // namespace spgemm_b200
