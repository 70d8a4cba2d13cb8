// kernels_heap.cuh -- the heaviest rows: symbolic bin 7 and the numeric heap
// tier (reference: the spill/heap paths, pipeline.cpp:315-348 and 396-410,
// hash_tables.cpp:113-123), re-designed around a shared-memory BITMAP of the
// output row's column set instead of a (global) hash table.
//
// One 1024-thread block per row, one block per SM (the bitmap takes 128 KB of
// the SM's shared memory). Columns are handled in windows of 2^20 (one window
// for every B with <= 1M columns).
//
//   symbolic   bit per product (atomicOr); the count is the number of bits the
//              row set. Exact, no probing, no table size to outgrow, so the
//              reference's spill recount is not needed -- the rows it would
//              have spilled (count > 0.8 * 24575) are still counted and
//              reported as spilled_rows.
//   numeric    pass A sets the bits again; a rank directory (uint16 prefix per
//              word within a 64-word superblock + uint32 superblock prefix)
//              gives every column its output position, so C.col is written
//              sorted straight from the bitmap (no comparison sort) and the
//              products of pass B land at their position. Pass B adds with
//              fp64 atomics into C.val (RED.ADD.F64): the result is within the
//              north-star 1e-12 tolerance but the summation order is not the
//              reference's. SpgemmOptions::ordered_heap selects the ordered
//              (bitwise) heap kernel k_num_global instead.
//
// Work distribution ("flattened" products). A row's A entries are taken in
// tiles of 1024; the tile's non-empty entries are compacted and prefix-summed
// by B row length, and warp w takes the w-th 1/32 of the tile's products --
// balanced however skewed the B rows are (R-MAT hubs). Within a warp, 32
// consecutive products per round: lane l's entry is found with a 5-step
// shuffle search over the next 32 entry starts.
#pragma once

#include "kernels.cuh"

namespace spgemm_b200 {

constexpr int kBigThreads = 1024;
constexpr int kBigWarps = kBigThreads / 32;
constexpr int kBigWindowLog = 20;
constexpr int64_t kBigWindow = int64_t(1) << kBigWindowLog;  // columns per bitmap window
constexpr int kBigWords = static_cast<int>(kBigWindow / 32);  // 32768 words = 128 KB
constexpr int kBigSuper = 64;                                  // words per rank superblock
constexpr int kBigWordsPerThread = kBigWords / kBigThreads;    // 32

// Staged tile of A entries (compacted: non-empty B rows only). Product
// offsets within a tile are 32-bit: a tile takes at most 1024 entries and
// stops early before its product count would reach 2^31.
struct BigTile {
  int32_t S[kBigThreads + 1];  // product prefix; S[n] = tile total
  int32_t b0[kBigThreads];     // B row start (32-bit index path)
  double av[kBigThreads];      // A value
  long long red[kBigWarps];
  int nce, ne;                 // compacted entries, A entries consumed
};

// The numeric kernel's bitmap and word prefixes are padded (one word / two
// halfwords per 32) so the rank pass, where thread t scans words [32t, 32t+32),
// is free of bank conflicts.
constexpr int kBigWordsPad = kBigWords + kBigWords / 32;
constexpr int kBigPrePad = kBigWords + 2 * (kBigWords / 32);
__device__ __forceinline__ uint32_t bm_idx(uint32_t w) { return w + (w >> 5); }
__device__ __forceinline__ uint32_t pre_idx(uint32_t w) { return w + 2 * (w >> 5); }

constexpr size_t kBigSymSmem = sizeof(uint32_t) * kBigWords + sizeof(BigTile);
constexpr size_t kBigNumSmem = sizeof(uint32_t) * kBigWordsPad + sizeof(uint16_t) * kBigPrePad +
                               sizeof(uint32_t) * (kBigWords / kBigSuper) + sizeof(BigTile);
static_assert(kBigNumSmem <= 227 * 1024, "heap-tier numeric block exceeds the opt-in shared memory");

// B's entries stream through L2 once per pass: loaded with an evict-first
// policy, so they do not push out the C.val lines of the rows in flight
// (which the ordered heap kernel read-modify-writes, evict-last).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int32_t ld_first(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_first(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// Walks every product of A row [a0, a1): visit(col, x, valid) is called by all
// 32 lanes of every warp once per round (valid = the lane holds a product).
// Round mapping: lane l of a round starting at product p0 belongs to entry
// jc + popc(M & bits<=l), where jc holds p0 and M has bit d set for every
// entry starting at p0+d (d in 1..31) -- one REDUX.OR per 32 products.
template <bool VALS, typename F>
__device__ __forceinline__ void big_walk(const DevCsr& A, const DevCsr& B, int64_t a0, int64_t a1, BigTile& t,
                                         F visit) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr long long kLimit = (1ll << 31) - 1;
  const uint64_t once = l2_evict_first_policy();
  for (int64_t e0 = a0; e0 < a1; e0 += t.ne) {
    const int ne = static_cast<int>(min(static_cast<int64_t>(kBigThreads), a1 - e0));
    long long len = 0;
    int32_t b0 = 0;
    double av = 0.0;
    if (tid < ne) {
      const int32_t k = A.col[e0 + tid];
      const int64_t r0 = B.rpt[k];
      len = B.rpt[k + 1] - r0;
      b0 = static_cast<int32_t>(r0);
      if constexpr (VALS) av = A.val[e0 + tid];
    }
    // one scan gives both the compacted index (low 11 bits) and the product prefix
    long long total;
    const long long ex = block_exclusive_scan<kBigThreads>((len << 11) | (len > 0 ? 1 : 0), t.red, &total);
    const long long s64 = ex >> 11;
    const bool in = tid < ne && s64 + len <= kLimit;  // a prefix of the tile's entries
    const int ne_eff = __syncthreads_count(in);
    const int ci = static_cast<int>(ex & 2047);
    if (in && len > 0) {
      t.S[ci] = static_cast<int32_t>(s64);
      t.b0[ci] = b0;
      t.av[ci] = av;
    }
    if (tid == ne_eff - 1) {
      t.nce = ci + (len > 0 ? 1 : 0);
      t.S[t.nce] = static_cast<int32_t>(s64 + len);
      t.ne = ne_eff;
    }
    __syncthreads();
    const int nce = t.nce;
    const int P = t.S[nce];
    const int pw0 = static_cast<int>(static_cast<long long>(P) * warp / kBigWarps);
    const int pw1 = static_cast<int>(static_cast<long long>(P) * (warp + 1) / kBigWarps);
    if (pw0 < pw1) {
      // jc = the entry holding product pw0: largest j with S[j] <= pw0
      int lo = 0, hi = nce - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (t.S[mid] <= pw0) lo = mid;
        else hi = mid - 1;
      }
      int jc = lo;
      int p0 = pw0;
      while (p0 < pw1) {
        // Long run: the next >= 32 products all belong to entry jc (most of the
        // product mass of skewed matrices comes from long B rows) -- no entry
        // search, U rounds of loads in flight.
        const int send = t.S[jc + 1];
        if (send - p0 >= 32) {
          const int stop = min(send, pw1);
          const int32_t bj = t.b0[jc] - t.S[jc];
          const double a = VALS ? t.av[jc] : 0.0;
          constexpr int U = 4;
          for (; p0 + 32 * U <= stop; p0 += 32 * U) {
            int32_t c[U];
            double bv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              c[u] = ld_first(B.col + bj + p0 + 32 * u + lane, once);
              if constexpr (VALS) bv[u] = ld_first(B.val + bj + p0 + 32 * u + lane, once);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) visit(c[u], VALS ? __dmul_rn(a, bv[u]) : 0.0, true);
          }
          for (; p0 + 32 <= stop; p0 += 32) {
            const int32_t at = bj + p0 + lane;
            visit(ld_first(B.col + at, once), VALS ? __dmul_rn(a, ld_first(B.val + at, once)) : 0.0, true);
          }
          if (p0 >= pw1) break;
          if (p0 == send) {
            ++jc;
            continue;
          }
        }
        // General round: lane l belongs to entry jc + popc(M & bits<=l).
        const int je = jc + 1 + lane;
        const int d = je <= nce ? t.S[je] - p0 : 64;  // >= lane + 1
        const unsigned M = __reduce_or_sync(kFull, d < 32 ? (1u << d) : 0u);
        const int j = jc + __popc(M & ((2u << lane) - 1u));
        const int p = p0 + lane;
        const bool valid = p < pw1;
        int32_t col = -1;
        double x = 0.0;
        if (valid) {
          const int32_t at = t.b0[j] + (p - t.S[j]);
          col = ld_first(B.col + at, once);
          if constexpr (VALS) x = __dmul_rn(t.av[j], ld_first(B.val + at, once));
        }
        visit(col, x, valid);
        // next round starts at p0+32: the entry holding it
        jc += __popc(M) + (__any_sync(kFull, d == 32) ? 1 : 0);
        p0 += 32;
      }
    }
    __syncthreads();
  }
}

// Symbolic, bin 7: rl lists the rows; the count of row i replaces its nprod
// in rpt. Rows counting more than `thresh` (the reference's spill threshold)
// are counted in info->spill_count.
__global__ void __launch_bounds__(kBigThreads, 1)
    k_big_sym(RowList rl_in, DevCsr A, DevCsr B, int64_t* __restrict__ rpt, DevInfo* info, int thresh) {
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);
  BigTile& t = *reinterpret_cast<BigTile*>(smem_raw + sizeof(uint32_t) * kBigWords);
  const int tid = threadIdx.x;
  for (int64_t idx = blockIdx.x; idx < rl.count; idx += gridDim.x) {
    const int64_t row = rl.row(idx);
    if (rpt[row] == 0) continue;  // no products (pipeline.cpp:368-371)
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    long long cnt = 0;
    for (int64_t wc0 = 0; wc0 < B.cols; wc0 += kBigWindow) {
      const int nwords = static_cast<int>((min(kBigWindow, B.cols - wc0) + 31) >> 5);
      uint4* b4 = reinterpret_cast<uint4*>(bm);
      for (int s = tid; s < (nwords + 3) >> 2; s += kBigThreads) b4[s] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
      const int32_t c0 = static_cast<int32_t>(wc0);
      big_walk<false>(A, B, a0, a1, t, [&](int32_t col, double, bool valid) {
        const uint32_t off = static_cast<uint32_t>(col - c0);
        if (valid && off < static_cast<uint32_t>(kBigWindow)) {
          const uint32_t bit = 1u << (off & 31u);  // (symbolic: unpadded bitmap)
          cnt += (atomicOr(bm + (off >> 5), bit) & bit) == 0u;
        }
      });
    }
    const long long total = block_sum_ll<kBigThreads>(cnt, t.red);
    if (tid == 0) {
      rpt[row] = total;
      if (total > thresh) atomicAdd(&info->spill_count, 1ull);
    }
    __syncthreads();
  }
}

// C.val of the rows in flight is zeroed and then hit by atomic adds from the
// whole row; both go out with an evict-last L2 policy so the lines stay
// on chip between the two while the B gathers stream through L2.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
#ifdef SPGEMM_ABLATE_NOKEEP
  *p = v;
#else
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#endif
}
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_keep(double* p, double v, uint64_t pol) {
#ifdef SPGEMM_ABLATE_NOKEEP
  atomicAdd(p, v);
#else
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#endif
}

// Numeric heap tier (see the header comment).
__global__ void __launch_bounds__(kBigThreads, 1)
    k_big_num(RowList rl_in, DevCsr A, DevCsr B, const int64_t* __restrict__ rpt, int32_t* __restrict__ ccol,
              double* __restrict__ cval, DevInfo* info) {
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);
  uint16_t* pre = reinterpret_cast<uint16_t*>(smem_raw + sizeof(uint32_t) * kBigWordsPad);
  uint32_t* sup =
      reinterpret_cast<uint32_t*>(smem_raw + sizeof(uint32_t) * kBigWordsPad + sizeof(uint16_t) * kBigPrePad);
  BigTile& t = *reinterpret_cast<BigTile*>(smem_raw + sizeof(uint32_t) * kBigWordsPad +
                                           sizeof(uint16_t) * kBigPrePad + sizeof(uint32_t) * (kBigWords / kBigSuper));
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t keep = l2_evict_last_policy();
  for (int64_t idx = blockIdx.x; idx < rl.count; idx += gridDim.x) {
    const int64_t row = rl.row(idx);
    const int64_t base = rpt[row];
    const int64_t n = rpt[row + 1] - base;
    if (n == 0) continue;
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    int64_t woff = 0;  // entries of the row in earlier windows
    for (int64_t wc0 = 0; wc0 < B.cols; wc0 += kBigWindow) {
      uint4* b4 = reinterpret_cast<uint4*>(bm);  // whole (padded) bitmap: the rank pass reads all of it
      for (int s = tid; s < kBigWordsPad / 4; s += kBigThreads) b4[s] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
      const int32_t c0 = static_cast<int32_t>(wc0);
      // ---- pass A: the window's column set
      big_walk<false>(A, B, a0, a1, t, [&](int32_t col, double, bool valid) {
        const uint32_t off = static_cast<uint32_t>(col - c0);
        if (valid && off < static_cast<uint32_t>(kBigWindow)) atomicOr(bm + bm_idx(off >> 5), 1u << (off & 31u));
      });
      // ---- rank directory; C.col written from the bitmap, C.val zeroed
      const int w0 = tid * kBigWordsPerThread;  // 32 words: half a superblock
      int mine = 0;
#pragma unroll 8
      for (int i = 0; i < kBigWordsPerThread; ++i) mine += __popc(bm[bm_idx(w0 + i)]);
      long long wtot;
      const long long g = block_exclusive_scan<kBigThreads>(mine, t.red, &wtot);
      const long long sbase = __shfl_sync(kFull, g, lane & ~1);  // prefix before the superblock
      if ((tid & 1) == 0) sup[tid >> 1] = static_cast<uint32_t>(g);
      int run = static_cast<int>(g - sbase);
      for (int i = 0; i < kBigWordsPerThread; ++i) {
        const int w = w0 + i;
        pre[pre_idx(w)] = static_cast<uint16_t>(run);
        run += __popc(bm[bm_idx(w)]);
      }
      __syncthreads();
      // C.col straight from the bitmap, word-major (consecutive threads take
      // consecutive words, so a warp's stores cover one contiguous span);
      // C.val of the window zeroed with coalesced stores.
      for (int w = tid; w < kBigWords; w += kBigThreads) {
        uint32_t m = bm[bm_idx(w)];
        if (m) {
          int64_t pos = woff + sup[w / kBigSuper] + pre[pre_idx(w)];
          do {
            const int b = __ffs(m) - 1;
            m &= m - 1u;
#ifndef SPGEMM_ABLATE_OUT  // diagnostic builds only (tools/build_ablation.sh)
            ccol[base + pos] = c0 + w * 32 + b;
#endif
            ++pos;
          } while (m);
        }
      }
      for (int64_t e = tid; e < wtot; e += kBigThreads) st_keep(cval + base + woff + e, 0.0, keep);
      __syncthreads();  // rank directory + zeroed C.val visible to the block
      // ---- pass B: products accumulate at their rank
      double* crow = cval + base + woff;
#ifndef SPGEMM_ABLATE_PASSB
      big_walk<true>(A, B, a0, a1, t, [&](int32_t col, double x, bool valid) {
        const uint32_t off = static_cast<uint32_t>(col - c0);
        if (valid && off < static_cast<uint32_t>(kBigWindow)) {
          const uint32_t w = off >> 5;
          const uint32_t r = sup[w / kBigSuper] + pre[pre_idx(w)] + __popc(bm[bm_idx(w)] & ((1u << (off & 31u)) - 1u));
#ifndef SPGEMM_ABLATE_RED
          red_add_keep(crow + r, x, keep);
#else
          if (x == 1.2345e-300) crow[r] = x;
#endif
        }
      });
#endif
      woff += wtot;
    }
    if (tid == 0 && woff != n) atomicOr(&info->error, kErrNumericCount);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Ordered heap tier (deterministic=true, the default): the same bitmap + rank
// directory as k_big_num, but pass B keeps the reference's per-column
// summation order, ((0 + a[i,k0]*b[k0,c]) + a[i,k1]*b[k1,c]) + ... in A-row
// order (hash_tables.cpp:182-193), so C is bitwise the reference's.
//
// Order needs one owner per output column. B's columns are split once per
// product into kPanels column panels balanced by B's column counts
// (k_col_hist + k_panel_bounds), and every B row's panel boundaries are stored
// (k_panel_split: poff[k*(kPanels+1) + p] = first entry of row k in panel p).
// Warp w of the row's block owns panel w: it walks the whole A row in order,
// 32 entries at a time, takes only its panel's slice of each B row (two loads
// per entry, no search), flattens the slices into rounds of 32 consecutive
// products (A order, then B order) and adds each product into C.val at its
// rank with a plain read-modify-write. Within a round, products of one entry
// have distinct columns; when a round spans several entries, lanes holding the
// same column (__match_any_sync) fold in lane order -- which is A order -- the
// group's first lane starting from C.val and each next lane adding to its
// predecessor's sum. Rounds are separated by __syncwarp, and no other warp
// ever touches the panel's columns, so every column is folded sequentially in
// A order. No atomics, no zeroing race: pass A zeroes C.val before the block
// barrier that precedes pass B.
constexpr int kPanels = kBigWarps;  // one column panel per warp
constexpr int kHistBuckets = 4096;

// Histogram of B's columns over kHistBuckets equal-width buckets.
__global__ void __launch_bounds__(256)
    k_col_hist(const int32_t* __restrict__ col, int64_t nnz, int64_t bucket_w,
               unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[kHistBuckets];
  for (int i = threadIdx.x; i < kHistBuckets; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz; e += stride)
    atomicAdd(&h[min(static_cast<int64_t>(kHistBuckets - 1), col[e] / bucket_w)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBuckets; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(h[i]));
}

// Panel p starts at the first bucket boundary where the cumulative count
// reaches p/kPanels of B's nonzeros (one block).
__global__ void __launch_bounds__(1024)
    k_panel_bounds(const unsigned long long* __restrict__ hist, int64_t bucket_w, int64_t ncols,
                   int32_t* __restrict__ colb) {
  __shared__ long long red[32];
  constexpr int PER = kHistBuckets / 1024;
  long long mine = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) mine += static_cast<long long>(hist[threadIdx.x * PER + i]);
  long long total;
  long long run = block_exclusive_scan<1024>(mine, red, &total);
  if (threadIdx.x == 0) {
    colb[0] = 0;
    colb[kPanels] = static_cast<int32_t>(min(ncols, static_cast<int64_t>(0x7fffffff)));
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int b = threadIdx.x * PER + i;
    const long long before = run;
    run += static_cast<long long>(hist[b]);
    // panel p (1..P-1) begins at bucket b when the cumulative count crosses p*total/P within it
    for (int p = 1; p < kPanels; ++p) {
      const long long target = total * p / kPanels;
      if (before < target && run >= target) colb[p] = static_cast<int32_t>(min(ncols, (b + 1) * bucket_w));
      if (total == 0 && b == 0) colb[p] = static_cast<int32_t>(min(ncols, p * (ncols / kPanels)));
    }
  }
}

// poff[k*(kPanels+1) + p] = first entry of B row k with column >= colb[p]
// (warp per row, lane p binary-searches boundary p; lane 0 = row start).
__global__ void __launch_bounds__(256)
    k_panel_split(DevCsr B, const int32_t* __restrict__ colb, int32_t* __restrict__ poff) {
  const int lane = threadIdx.x & 31;
  const int32_t bound = colb[lane];
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; k < B.rows; k += warps) {
    const int64_t r0 = B.rpt[k], r1 = B.rpt[k + 1];
    int64_t lo = r0, hi = r1;  // first index with col >= bound
    if (lane == 0) hi = r0;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (B.col[mid] < bound) lo = mid + 1;
      else hi = mid;
    }
    int32_t* out = poff + k * (kPanels + 1);
    out[lane] = static_cast<int32_t>(lo);
    if (lane == 0) out[kPanels] = static_cast<int32_t>(r1);
  }
}

__global__ void __launch_bounds__(kBigThreads, 1)
    k_big_num_ord(RowList rl_in, DevCsr A, DevCsr B, const int64_t* __restrict__ rpt, int32_t* __restrict__ ccol,
                  double* __restrict__ cval, const int32_t* __restrict__ poff, DevInfo* info) {
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);
  uint16_t* pre = reinterpret_cast<uint16_t*>(smem_raw + sizeof(uint32_t) * kBigWordsPad);
  uint32_t* sup =
      reinterpret_cast<uint32_t*>(smem_raw + sizeof(uint32_t) * kBigWordsPad + sizeof(uint16_t) * kBigPrePad);
  BigTile& t = *reinterpret_cast<BigTile*>(smem_raw + sizeof(uint32_t) * kBigWordsPad +
                                           sizeof(uint16_t) * kBigPrePad + sizeof(uint32_t) * (kBigWords / kBigSuper));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t keep = l2_evict_last_policy();  // the rows' C.val stays in L2 between its RMWs
  const uint64_t once = l2_evict_first_policy();  // B's entries stream through
  for (int64_t idx = blockIdx.x; idx < rl.count; idx += gridDim.x) {
    const int64_t row = rl.row(idx);
    const int64_t base = rpt[row];
    const int64_t n = rpt[row + 1] - base;
    if (n == 0) continue;
    const int64_t a0 = A.rpt[row], a1 = A.rpt[row + 1];
    int64_t woff = 0;
    for (int64_t wc0 = 0; wc0 < B.cols; wc0 += kBigWindow) {
      uint4* b4 = reinterpret_cast<uint4*>(bm);
      for (int s = tid; s < kBigWordsPad / 4; s += kBigThreads) b4[s] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
      const int32_t c0 = static_cast<int32_t>(wc0);
      // ---- pass A: the window's column set (as k_big_num)
      big_walk<false>(A, B, a0, a1, t, [&](int32_t col, double, bool valid) {
        const uint32_t off = static_cast<uint32_t>(col - c0);
        if (valid && off < static_cast<uint32_t>(kBigWindow)) atomicOr(bm + bm_idx(off >> 5), 1u << (off & 31u));
      });
      // ---- rank directory; C.col from the bitmap; C.val zeroed
      const int w0 = tid * kBigWordsPerThread;
      int mine = 0;
#pragma unroll 8
      for (int i = 0; i < kBigWordsPerThread; ++i) mine += __popc(bm[bm_idx(w0 + i)]);
      long long wtot;
      const long long g = block_exclusive_scan<kBigThreads>(mine, t.red, &wtot);
      const long long sbase = __shfl_sync(kFull, g, lane & ~1);
      if ((tid & 1) == 0) sup[tid >> 1] = static_cast<uint32_t>(g);
      int run = static_cast<int>(g - sbase);
      for (int i = 0; i < kBigWordsPerThread; ++i) {
        const int w = w0 + i;
        pre[pre_idx(w)] = static_cast<uint16_t>(run);
        run += __popc(bm[bm_idx(w)]);
      }
      __syncthreads();
      for (int w = tid; w < kBigWords; w += kBigThreads) {
        uint32_t m = bm[bm_idx(w)];
        if (m) {
          int64_t pos = woff + sup[w / kBigSuper] + pre[pre_idx(w)];
          do {
            const int b = __ffs(m) - 1;
            m &= m - 1u;
            ccol[base + pos] = c0 + w * 32 + b;
            ++pos;
          } while (m);
        }
      }
      double* crow = cval + base + woff;
      for (int64_t e = tid; e < wtot; e += kBigThreads) st_keep(crow + e, 0.0, keep);
      __syncthreads();  // rank directory + zeroed C.val visible to the block
      // ---- pass B (ordered): warp `warp` owns column panel `warp`. One A
      // entry at a time (its slice's columns are distinct, so the lanes never
      // share a rank); up to U rounds of one entry are in flight at once.
      const int32_t* pcol = poff + warp;
      for (int64_t e0 = a0; e0 < a1; e0 += 32) {
        const int64_t j = e0 + lane;
        int32_t s = 0;
        int len = 0;
        double av = 0.0;
        if (j < a1) {
          const int64_t k = A.col[j];
          s = pcol[k * (kPanels + 1)];
          len = pcol[k * (kPanels + 1) + 1] - s;
          av = A.val[j];
        }
        unsigned todo = __ballot_sync(kFull, len > 0);
        while (todo) {
          const int src = __ffs(todo) - 1;
          todo &= todo - 1u;
          const int32_t sj = __shfl_sync(kFull, s, src);
          const int lj = __shfl_sync(kFull, len, src);
          const double aj = __shfl_sync(kFull, av, src);
          constexpr int U = 4;
          for (int qb = 0; qb < lj; qb += 32 * U) {
            uint32_t r[U];
            double x[U];
            bool in[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int q = qb + 32 * u + lane;
              int32_t col = 0;
              double bv = 0.0;
              if (q < lj) {
                col = ld_first(B.col + sj + q, once);
                bv = ld_first(B.val + sj + q, once);
              }
              const uint32_t off = static_cast<uint32_t>(col - c0);
              in[u] = q < lj && off < static_cast<uint32_t>(kBigWindow);
              x[u] = __dmul_rn(aj, bv);
              r[u] = 0;
              if (in[u]) {
                const uint32_t w = off >> 5;
                r[u] = sup[w / kBigSuper] + pre[pre_idx(w)] + __popc(bm[bm_idx(w)] & ((1u << (off & 31u)) - 1u));
              }
            }
            double cur[U];
#pragma unroll
            for (int u = 0; u < U; ++u) cur[u] = in[u] ? ld_keep(crow + r[u], keep) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (in[u]) st_keep(crow + r[u], __dadd_rn(cur[u], x[u]), keep);
          }
          __syncwarp();  // this entry's updates before the next entry's
        }
      }
      woff += wtot;
      __syncthreads();
    }
    if (tid == 0 && woff != n) atomicOr(&info->error, kErrNumericCount);
    __syncthreads();
  }
}

}  // namespace spgemm_b200
