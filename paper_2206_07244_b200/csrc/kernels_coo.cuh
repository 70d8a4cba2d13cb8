// kernels_coo.cuh -- csr_from_coo on the device (the
// ingestion side of the path): triples in input order -> CSR with each row's
// columns sorted and duplicates summed in input order, the reference's
// semantics (csr.cpp:12-72: the first duplicate's value as is, then += the
// next ones in file order).
//
// Two stable counting sorts (LSD: by column, then by row) give the entries in
// (row, column, input index) order. A stable pass: per-key counts (atomics,
// order-free), an exclusive scan of the counts (k_scan), and a scatter in tile
// order -- each 1024-entry tile sorts its (key, local index) pairs in shared
// memory, then, chained behind the previous tile (dynamic tile ids, so no
// tile waits on one that has not started), reserves each key run's slots from
// the key's cursor. Runs of equal (row, column) are then folded sequentially
// by their first entry, and compacted with a scan of the run heads; the row
// pointers come from the per-row head counts.
#pragma once

#include "kernels.cuh"

namespace spgemm_b200 {

constexpr int kCooTile = 1024;
constexpr int kCooThreads = 256;
constexpr int kCooItems = kCooTile / kCooThreads;  // 4

// Entries outside the shape: the smallest offending index (for the message).
__global__ void __launch_bounds__(256)
    k_coo_check(const int64_t* __restrict__ row, const int64_t* __restrict__ col, int64_t n, int64_t rows,
                int64_t cols, unsigned long long* __restrict__ bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride) {
    if (static_cast<uint64_t>(row[e]) >= static_cast<uint64_t>(rows) ||
        static_cast<uint64_t>(col[e]) >= static_cast<uint64_t>(cols))
      atomicMin(bad, static_cast<unsigned long long>(e));
  }
}

__global__ void __launch_bounds__(256)
    k_coo_count(const int64_t* __restrict__ key, int64_t n, unsigned long long* __restrict__ cnt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride)
    atomicAdd(&cnt[key[e]], 1ull);
}

// One stable counting-sort pass: perm_out[cursor[key] + rank] = entry, where
// the entries are visited in perm_in order (identity when null) and rank
// counts the earlier entries (in that order) with the same key. cursor holds
// the exclusive scan of the key counts on entry and is advanced tile by tile.
__global__ void __launch_bounds__(kCooThreads)
    k_coo_scatter(const int64_t* __restrict__ key, const uint32_t* __restrict__ perm_in, int64_t n,
                  long long* __restrict__ cursor, int* __restrict__ done, int* __restrict__ tile_counter,
                  uint32_t* __restrict__ perm_out) {
  __shared__ unsigned long long s_key[kCooTile];  // (key << 10) | local index, sorted
  __shared__ uint32_t s_ent[kCooTile];            // entry of each local index
  __shared__ int s_head[kCooTile];                // position of the run head of each sorted position
  __shared__ long long s_base[kCooTile];          // cursor value reserved by each run head
  __shared__ int s_tile;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t t0 = static_cast<int64_t>(tile) * kCooTile;
#pragma unroll
  for (int u = 0; u < kCooItems; ++u) {
    const int li = tid * kCooItems + u;
    const int64_t i = t0 + li;
    if (i < n) {
      const uint32_t e = perm_in ? perm_in[i] : static_cast<uint32_t>(i);
      s_ent[li] = e;
      s_key[li] = (static_cast<unsigned long long>(key[e]) << 10) | static_cast<unsigned long long>(li);
    } else {
      s_key[li] = ~0ull;
    }
  }
  __syncthreads();
  block_bitonic_smem<kCooThreads>(s_key, kCooTile);
  // run heads and, per position, its run head (an inclusive max scan)
  int hv[kCooItems];
  int local_max = -1;
#pragma unroll
  for (int u = 0; u < kCooItems; ++u) {
    const int s = tid * kCooItems + u;
    const bool valid = s_key[s] != ~0ull;
    const bool head = valid && (s == 0 || (s_key[s] >> 10) != (s_key[s - 1] >> 10));
    local_max = max(local_max, head ? s : -1);
    hv[u] = local_max;
  }
  // exclusive max over the threads before this one
  __shared__ int s_wmax[kCooThreads / 32];
  const int lane = tid & 31, warp = tid >> 5;
  int x = local_max;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x = max(x, y);
  }
  if (lane == 31) s_wmax[warp] = x;
  __syncthreads();
  int before = __shfl_up_sync(kFull, x, 1);
  if (lane == 0) before = -1;
  for (int w = 0; w < warp; ++w) before = max(before, s_wmax[w]);
#pragma unroll
  for (int u = 0; u < kCooItems; ++u) s_head[tid * kCooItems + u] = max(before, hv[u]);
  __syncthreads();
  // wait for the previous tile's reservations, then reserve this tile's runs
  if (tid == 0 && tile > 0) {
    while (atomicAdd(done + tile - 1, 0) == 0) {
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kCooItems; ++u) {
    const int s = tid * kCooItems + u;
    if (s_key[s] != ~0ull && s_head[s] == s) {
      int e = s + 1;  // run end
      while (e < kCooTile && s_key[e] != ~0ull && (s_key[e] >> 10) == (s_key[s] >> 10)) ++e;
      const int64_t k = static_cast<int64_t>(s_key[s] >> 10);
      const long long b = __ldcg(cursor + k);  // (written by earlier tiles on other SMs: not from L1)
      s_base[s] = b;
      __stcg(cursor + k, b + (e - s));
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) atomicExch(done + tile, 1);
#pragma unroll
  for (int u = 0; u < kCooItems; ++u) {
    const int s = tid * kCooItems + u;
    if (s_key[s] != ~0ull) {
      const int h = s_head[s];
      perm_out[s_base[h] + (s - h)] = s_ent[s_key[s] & 1023ull];
    }
  }
}

// Run heads of the (row, column)-sorted entries: head[p] = 1 when entry p
// starts a new (row, column); rowcnt[row] counts the heads (distinct columns).
__global__ void __launch_bounds__(256)
    k_coo_heads(const int64_t* __restrict__ row, const int64_t* __restrict__ col, const uint32_t* __restrict__ perm,
                int64_t n, int64_t* __restrict__ head, unsigned long long* __restrict__ rowcnt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += stride) {
    const uint32_t e = perm[p];
    bool h = p == 0;
    if (!h) {
      const uint32_t f = perm[p - 1];
      h = row[e] != row[f] || col[e] != col[f];
    }
    head[p] = h ? 1 : 0;
    if (h) atomicAdd(&rowcnt[row[e]], 1ull);
  }
}

// Each run head folds its run in input order (the run is stable-sorted) and
// writes C.col/C.val at its compacted index.
__global__ void __launch_bounds__(256)
    k_coo_fold(const int64_t* __restrict__ row, const int64_t* __restrict__ col, const double* __restrict__ val,
               const uint32_t* __restrict__ perm, int64_t n, const int64_t* __restrict__ head_at,
               int32_t* __restrict__ ccol, double* __restrict__ cval) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += stride) {
    const int64_t at = head_at[p];
    const bool h = head_at[p + 1] != at;  // (exclusive scan of the head flags)
    if (!h) continue;
    const uint32_t e = perm[p];
    double v = val[e];
    for (int64_t q = p + 1; q < n; ++q) {
      const uint32_t f = perm[q];
      if (row[f] != row[e] || col[f] != col[e]) break;
      v += val[f];
    }
    ccol[at] = static_cast<int32_t>(col[e]);
    cval[at] = v;
  }
}

}  // namespace spgemm_b200
