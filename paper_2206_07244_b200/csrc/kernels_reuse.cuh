// kernels_reuse.cuh -- per-row reuse flags and the multi-row structure-reuse
// numeric kernel (the reuse route: C = A*A-shaped products of regular
// matrices whose A and B rows have <= 32 entries -- 3-D stencils, FEM).
//
// Row i's output structure is row i-1's shifted by one column exactly when A
// row i is A row i-1 shifted by one (same length, every column + 1) and every
// B row k it references is B row k-1 shifted by one (shift1[k], k_shift_flags):
// then the products group into columns the same way, in the same sorted order.
// k_reuse_flags evaluates that test once per row (flag[i]); the symbolic
// kernel copies counts along flagged rows and the numeric kernel below folds
// flagged rows through the predecessor's product -> output map.
//
// k_num_reuse_multi. One warp per run of up to 32 consecutive bin rows. A row
// that is not flagged (a chain head: boundary rows of a grid, the run's first
// row) takes the full path: dense-index column table, sort, C(i,:), and the
// map "product (j, q) -> accumulator of its output" for the next row (or, when
// the warp's previous row has the same shape at another shift, the exact
// per-product column check). Flagged rows are folded M at a time through that
// map: their A rows are consecutive in A (A.val contiguous), their B rows k+r
// are consecutive in B (B row k + r starts r*len after B row k), so the group's
// metadata is one row's; step j adds a[r][j] * B(k_j + r, q) into
// accumulator buffer r at map[j][q] for all M rows, one A entry per step, in
// A-row order from +0.0 -- bitwise the reference (hash_tables.cpp:179-201,
// reference.cpp:21-27). The M read-modify-write chains are independent, so
// the shared-memory latency of one chain (ld -> add -> st -> next ld) is
// hidden by the other M-1; the next batch's B values are loaded while this
// batch folds. The kernel is bound by the L1 data pipe (ncu: ~90% of peak,
// two thirds of it the accumulators' shared loads and stores), so the layout
// minimises shared wavefronts: accumulator slots skewed per 25-position plane
// (multi_slot: fewer bank conflicts), lanes without a product predicated off,
// and each position's first product stored without a read (no zeroing).
// (k_num_reuse folds one row at a time: its single chain left the warp
// stalled on shared memory; ncu.)
#pragma once

namespace spgemm_b200 {

// flag[i] = 1 when row i's structure is row i-1's shifted by one (see above);
// rows with more than 32 entries or without entries are never flagged. The
// A-row shift comes from shift1 itself when A and B are one matrix.
__global__ void __launch_bounds__(256)
    k_reuse_flags(DevCsr A, const uint8_t* __restrict__ shift1, uint8_t* __restrict__ flag, int a_is_b) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < A.rows; i += stride) {
    bool ok = false;
    if (i > 0) {
      const int64_t r0 = A.rpt[i - 1], r1 = A.rpt[i], r2 = A.rpt[i + 1];
      const int na = static_cast<int>(r2 - r1);
      ok = na == r1 - r0 && na > 0 && na <= 32 && (!a_is_b || shift1[i] != 0);
      // batches of 8 entries: their loads issued before any is tested
      for (int q0 = 0; ok && q0 < na; q0 += 8) {
        int32_t c[8], cp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool on = q0 + u < na;
          c[u] = on ? A.col[r1 + q0 + u] : 0;
          cp[u] = on && !a_is_b ? A.col[r0 + q0 + u] : c[u] - 1;
        }
        // the 8 flag gathers issued together (no short-circuit between them)
        uint8_t sf[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) sf[u] = q0 + u < na ? shift1[c[u]] : uint8_t{1};
        bool f = true;
#pragma unroll
        for (int u = 0; u < 8; ++u) f = f & (q0 + u >= na || c[u] == cp[u] + 1) & (sf[u] != 0);
        ok = f;
      }
    }
    flag[i] = ok ? 1 : 0;
  }
}

#ifndef SPGEMM_MULTI_MINB
#define SPGEMM_MULTI_MINB 6  // resident blocks per SM
#endif
constexpr int kMultiWarps = 4;
constexpr int kMultiM = 4;               // flagged rows folded together
#ifndef SPGEMM_MULTI_U
#define SPGEMM_MULTI_U 2
#endif
constexpr int kMultiU = SPGEMM_MULTI_U;  // steps per batch of B loads (two batches in flight)
constexpr uint32_t kMultiVS = 152 * 8;  // one accumulator buffer: slots multi_slot(0..127) + spare (151)
constexpr int kMultiSpare = 151;
// Accumulator slot of output position p. 64-bit shared accesses are served per
// half-warp: 16 lanes whose slots share a bank pair (slot mod 16) cost an extra
// wavefront. Output positions of a 3-D stencil product come in planes of 25
// (5 x 5 for radius 2), and a step's 27 products then collide mod 16 (2
// wavefronts per half-warp); skewing every plane by 4 slots leaves 3
// wavefronts per warp access instead of 4 (tools: DESIGN §6). Any permutation
// is exact; this one only changes bank conflicts.
__device__ __forceinline__ int multi_slot(int p) { return p + 4 * (p / 25); }
static_assert(127 + 4 * (127 / 25) < kMultiSpare, "slots below the spare");
constexpr size_t kMultiWarpBytes = kMultiM * kMultiVS + 128 * 4 + 32 * 8 + kMultiM * 32 * 8 + 32 * 32 * 2;  // 8704
static_assert(kMultiWarps * kMultiWarpBytes + 1024 < 65536, "the map holds 16-bit shared addresses");
static_assert(kMultiVS % 16 == 0 && kMultiWarpBytes % 16 == 0, "16-byte aligned accumulator buffers");
static_assert(32 % kMultiU == 0 && kMultiU % 2 == 0, "U: even, divides the warp width");

__global__ void __launch_bounds__(32 * kMultiWarps, SPGEMM_MULTI_MINB)
    k_num_reuse_multi(RowList rl_in, DevCsr A, DevCsr B, const int64_t* __restrict__ rpt,
                      int32_t* __restrict__ ccol, double* __restrict__ cval, uint32_t scale, DevInfo* info, Spec sp,
                      int rows_per_warp, const uint8_t* __restrict__ flag) {
  constexpr int G = 32, NMAX = 128, T = 256, E = 4, M = kMultiM, U = kMultiU;
  constexpr int VD = kMultiVS / 8;  // doubles per accumulator buffer
  const RowList rl = rl_in.resolved();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = smem_raw + static_cast<size_t>(warp) * kMultiWarpBytes;
  double* vals = reinterpret_cast<double*>(wb);  // [M][VD]
  // the full path's table, rank and claim order overlay accumulator buffers 1..M-1
  int32_t* keys = reinterpret_cast<int32_t*>(wb + kMultiVS);  // [T]; after the walk: sort keys
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(keys);
  uint32_t* packed32 = reinterpret_cast<uint32_t*>(keys);
  uint8_t* sidx = wb + kMultiVS + T * 4;                              // [T] dense index per slot; then rank
  int32_t* cols = reinterpret_cast<int32_t*>(wb + kMultiVS + T * 5);  // [NMAX] claim order
  static_assert(kMultiVS + T * 5 + NMAX * 4 <= kMultiM * kMultiVS, "overlay");
  unsigned char* pw = wb + M * kMultiVS;
  int32_t* ocols = reinterpret_cast<int32_t*>(pw);                  // [NMAX] last row's output columns
  uint2* meta = reinterpret_cast<uint2*>(pw + NMAX * 4);             // [32] (B row start, length) of entry j
  double* avs = reinterpret_cast<double*>(pw + NMAX * 4 + 32 * 8);   // [M][32] A values of the group's rows
  uint16_t* map = reinterpret_cast<uint16_t*>(pw + NMAX * 4 + 32 * 8 + M * 32 * 8);  // [32][32]
  const uint32_t vals_sa = static_cast<uint32_t>(__cvta_generic_to_shared(vals));
  const char* bvl = reinterpret_cast<const char*>(B.val + lane);
  const uint16_t* mapl = map + lane;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t mult = scale * 0x9E3779B1u;

  // the warp's previous row (its map and ocols are valid when pvalid); lane j
  // holds entry j's column and B-row start
  bool pvalid = false;
  int pna = 0, pn = 0;
  int32_t pk = 0, pb0 = 0;
  int plen = 0;
  unsigned nreuse = 0, nfull = 0;
  int64_t R = rows_per_warp;
  if (R <= 0) {
    const int64_t warps = static_cast<int64_t>(gridDim.x) * kMultiWarps;
    R = kReuseRows;
    while (R > 1 && rl.count < warps * R) R >>= 1;
  }
  const int64_t first = (static_cast<int64_t>(blockIdx.x) * kMultiWarps + warp) * R;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kMultiWarps * R;
  for (int64_t run0 = first; run0 < rl.count; run0 += stride) {
    // the run's rows, one per lane: id, C offset and nnz, A-row bounds, flag
    int64_t lrow = -1, lbase = 0, la0 = 0;
    int ln = 0, lna = 0;
    bool need = false, lflag = false;
    if (lane < R && run0 + lane < rl.count) {
      lrow = rl.row(run0 + lane);
      lbase = rpt[lrow];
      ln = static_cast<int>(rpt[lrow + 1] - lbase);
      need = !sp.done(lrow) && ln > 0;
      if (need) {
        la0 = A.rpt[lrow];
        lna = static_cast<int>(min(A.rpt[lrow + 1] - la0, static_cast<int64_t>(G + 1)));
        lflag = flag[lrow] != 0;
      }
    }
    // a flagged row folds through its predecessor's map when that predecessor
    // is the previous lane's row (the warp processes it just before)
    const int64_t up_row = __shfl_up_sync(kFull, lrow, 1);
    const bool up_need = __shfl_up_sync(kFull, need, 1);
    unsigned todo = __ballot_sync(kFull, need);
    const unsigned chain = __ballot_sync(kFull, need && lflag && lane > 0 && up_need && up_row + 1 == lrow);
    while (todo) {
      const int src = __ffs(todo) - 1;
      const int64_t base = __shfl_sync(kFull, lbase, src);
      const int n = __shfl_sync(kFull, ln, src);
      const int64_t a0 = __shfl_sync(kFull, la0, src);
      const int na = __shfl_sync(kFull, lna, src);
      if (((chain >> src) & 1u) && pvalid) {
        // ---- M flagged rows at once: rows src .. src+m-1 (consecutive)
        const unsigned brk = ~(chain >> src);  // the first zero bit ends the group
        const int m = min(M, brk ? __ffs(brk) - 1 : 32 - src);
        todo &= ~(((1u << m) - 1u) << src);
        // entry j of row src (its B row start; row src + r's is r*len further)
        int32_t k = 0, b0 = 0;
        int len = 0;
        if (lane < na) {
          k = A.col[a0 + lane];
          const int64_t r0 = B.rpt[k];
          len = static_cast<int>(B.rpt[k + 1] - r0);
          b0 = static_cast<int32_t>(r0);
        }
        meta[lane] = make_uint2(static_cast<uint32_t>(b0), static_cast<uint32_t>(len));
        // the group's A values: its rows are consecutive in A, na entries each
#pragma unroll
        for (int r = 0; r < M; ++r) avs[r * 32 + lane] = (r < m && lane < na) ? A.val[a0 + r * na + lane] : 0.0;
        // (no zeroing: a position's first product in A order -- bit 0 of its map
        // entry -- is stored as 0.0 + x without reading the accumulator)
        // B values of U steps x M rows; the next batch's loads are issued
        // before this batch's folds (software pipeline, two register sets)
        auto load = [&](int j0, double (&bv)[U][M], bool (&on_)[U]) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint2 bl = meta[j0 + u];  // rows j >= na: length 0
            const bool on = lane < static_cast<int>(bl.y);
            on_[u] = on;
#pragma unroll
            for (int r = 0; r < M; ++r)
              bv[u][r] = ldg_f64_if(bvl + static_cast<size_t>(bl.x + r * bl.y) * 8u, on && r < m);
          }
        };
        auto fold = [&](int j0, const double (&bv)[U][M], const bool (&on)[U]) {
          uint32_t am[U];  // the steps' map entries, loaded ahead of the chains
#pragma unroll
          for (int u = 0; u < U; ++u) am[u] = mapl[(j0 + u) * G];
          double x[U][M];
#pragma unroll
          for (int r = 0; r < M; ++r) {
#pragma unroll
            for (int u = 0; u < U; u += 2) {
              const double2 a2 = *reinterpret_cast<const double2*>(avs + r * 32 + j0 + u);
              x[u][r] = __dmul_rn(a2.x, bv[u][r]);
              x[u + 1][r] = __dmul_rn(a2.y, bv[u + 1][r]);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            // lanes without a product (lane >= len, j >= na) are predicated off
            // (no shared access: a common spare slot would add a wavefront).
            // The volatile shared accesses stay in program order: the M
            // buffers' loads of step u, then their stores -- the M chains
            // overlap, and step u's stores precede step u+1's loads
            const uint32_t a = am[u] & ~1u;
            const bool rd = on[u] && (am[u] & 1u) == 0u;  // not the position's first product
            double acc[M];
#pragma unroll
            for (int r = 0; r < M; ++r) acc[r] = lds_f64_if(a + r * kMultiVS, rd);  // 0.0 when not read
#pragma unroll
            for (int r = 0; r < M; ++r) sts_f64_if(a + r * kMultiVS, __dadd_rn(acc[r], x[u][r]), on[u]);
          }
        };
        double bA[U][M], bB[U][M];
        bool oA[U], oB[U];
        load(0, bA, oA);
#pragma unroll 1
        for (int j0 = 0; j0 < na; j0 += 2 * U) {
          if (j0 + U < na) load(j0 + U, bB, oB);
          fold(j0, bA, oA);
          if (j0 + U >= na) break;
          if (j0 + 2 * U < na) load(j0 + 2 * U, bA, oA);
          fold(j0 + U, bB, oB);
        }
        __syncwarp();
        // C rows: the previous row's columns + r + 1, buffer r's values
        int64_t rb[M];
#pragma unroll
        for (int r = 0; r < M; ++r) rb[r] = __shfl_sync(kFull, lbase, min(src + r, 31));
        for (int e = lane; e < n; e += G) {
          const int32_t c0 = ocols[e];
#pragma unroll
          for (int r = 0; r < M; ++r) {
            if (r < m) {
              ccol[rb[r] + e] = c0 + r + 1;
              cval[rb[r] + e] = vals[r * VD + multi_slot(e)];
            }
          }
          ocols[e] = c0 + m;
        }
        __syncwarp();
        pk = k + (m - 1);
        pb0 = b0 + (m - 1) * len;
        plen = len;
        pna = na;
        pn = n;
        nreuse += m;
        continue;
      }
      todo &= todo - 1u;
      // ---- one row: the exact check against the warp's previous row, or the full path
      int32_t k = 0, b0 = 0;
      int len = 0;
      double av = 0.0;
      if (lane < na) {
        k = A.col[a0 + lane];
        av = A.val[a0 + lane];
        const int64_t r0 = B.rpt[k];
        len = static_cast<int>(B.rpt[k + 1] - r0);
        b0 = static_cast<int32_t>(r0);
      }
      if (na > G || __reduce_max_sync(kFull, static_cast<unsigned>(len)) > static_cast<unsigned>(G)) {
        if (lane == 0) atomicOr(&info->error, kErrNumericCount);  // outside the route's precondition
        pvalid = false;
        continue;
      }
      meta[lane] = make_uint2(static_cast<uint32_t>(b0), static_cast<uint32_t>(len));
      avs[lane] = av;
      __syncwarp();
      int32_t* ocp = ccol + base;
      double* ovp = cval + base;
      const int32_t d = __shfl_sync(kFull, k, 0) - __shfl_sync(kFull, pk, 0);
      bool reused =
          pvalid && na == pna && n == pn && __all_sync(kFull, lane >= na || (len == plen && k - pk == d));
      if (reused) {
        // same shape at shift d: check every product's column while folding
        bool ok = true;
        for (int j = 0; j < na; ++j) {
          const int32_t pbj = __shfl_sync(kFull, pb0, j);
          const uint2 mj = meta[j];
          if (lane < static_cast<int>(mj.y)) {
            const int32_t c = B.col[mj.x + lane];
            const int32_t cp = B.col[pbj + lane];
            const double x = __dmul_rn(avs[j], B.val[mj.x + lane]);
            ok = ok && c - cp == d;
            const uint32_t a = map[j * G + lane];
            const uint32_t aa = a & ~1u;
            sts_f64(aa, __dadd_rn((a & 1u) ? 0.0 : lds_f64(aa), x));
          }
          __syncwarp();
          if (!__all_sync(kFull, ok)) break;  // structure differs: the full path recomputes
        }
        reused = __all_sync(kFull, ok);
        __syncwarp();
      }
      if (reused) {
        for (int e = lane; e < n; e += G) {
          const int32_t c = ocols[e] + d;
          ocols[e] = c;
          ocp[e] = c;
          ovp[e] = vals[multi_slot(e)];
        }
        ++nreuse;
      } else {
        // ---- full path: dense-index column table, sort, map for the next rows
        int32_t kmin = 0x7fffffff, kmax = -1;
        if (lane < na && len > 0) {
          kmin = B.col[b0];
          kmax = B.col[b0 + len - 1];
        }
        kmin = static_cast<int32_t>(__reduce_min_sync(kFull, static_cast<unsigned>(kmin)));
        kmax = static_cast<int32_t>(__reduce_max_sync(kFull, static_cast<unsigned>(kmax + 1))) - 1;
        const int lg = min(log2_const<T>(), max(2, ceil_log2_ll(2 * static_cast<long long>(n))));
        const uint32_t hshift = 32u - static_cast<uint32_t>(lg), hmask = (1u << lg) - 1u;
        fill_empty<G>(keys, 1 << lg, lane);
        __syncwarp();
        int nk = 0;
        for (int j = 0; j < na; ++j) {
          const uint2 mj = meta[j];
          const bool on = lane < static_cast<int>(mj.y);
          const int32_t c = on ? B.col[mj.x + lane] : -1;
          const double x = on ? __dmul_rn(avs[j], B.val[mj.x + lane]) : 0.0;
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
          const unsigned cbits = __ballot_sync(kFull, fresh);
          if (nk + __popc(cbits) > NMAX) {  // more columns than the symbolic count allows
            nk = NMAX + 1;
            break;
          }
          if (c >= 0) {
            const int ix = fresh ? nk + __popc(cbits & lt) : sidx[h];
            const double prev = fresh ? 0.0 : vals[ix];
            vals[ix] = __dadd_rn(prev, x);
            map[j * G + lane] = static_cast<uint16_t>(ix);
            if (fresh) {
              sidx[h] = static_cast<uint8_t>(ix);
              cols[ix] = c;
            }
          }
          nk += __popc(cbits);
          __syncwarp();
        }
        __syncwarp();
        int nn = n;
        if (nk != n) {
          if (lane == 0) atomicOr(&info->error, kErrNumericCount);
          nn = min(n, min(nk, NMAX));
        }
        const bool narrow = static_cast<unsigned>(kmax - kmin) < (1u << 25);
        for (int e = lane; e < nn; e += G) {
          const int32_t c = cols[e];
          if (narrow) packed32[e] = (static_cast<uint32_t>(c - kmin) << 7) | static_cast<uint32_t>(e);
          else packed[e] = (static_cast<unsigned long long>(static_cast<uint32_t>(c)) << 32) | static_cast<uint32_t>(e);
        }
        __syncwarp();
        if (narrow) group_sort_inplace<G, E, uint32_t>(packed32, nn, lane, kFull);
        else group_sort_inplace<G, E, unsigned long long>(packed, nn, lane, kFull);
        __syncwarp();
        uint8_t* rank = sidx;
        for (int e = lane; e < nn; e += G) {
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
        // product -> its output's accumulator address (buffer 0) for the next
        // rows; map rows j >= na and lanes past a B row's length: the spare slot
        // bit 0: the product is its position's first in A order (the claim-order
        // columns are consumed: their bytes mark the positions seen)
        uint8_t* seen = reinterpret_cast<uint8_t*>(cols);
        for (int e = lane; e < NMAX; e += G) seen[e] = 0;
        __syncwarp();
        for (int j = 0; j < G; ++j) {
          const int lj = __shfl_sync(kFull, len, j);
          uint32_t m = vals_sa + 8u * kMultiSpare;
          if (j < na && lane < lj) {
            const int pos = rank[map[j * G + lane]];
            m = vals_sa + 8u * multi_slot(pos) + (seen[pos] ? 0u : 1u);
            seen[pos] = 1;  // (a step's positions are distinct)
          }
          map[j * G + lane] = static_cast<uint16_t>(m);
          __syncwarp();
        }
        ++nfull;
      }
      pvalid = true;
      pk = k;
      pb0 = b0;
      plen = len;
      pna = na;
      pn = n;
    }
  }
  nreuse = __reduce_add_sync(kFull, lane == 0 ? nreuse : 0u);
  nfull = __reduce_add_sync(kFull, lane == 0 ? nfull : 0u);
  if (lane == 0 && (nreuse | nfull)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&info->reuse_rows), static_cast<unsigned long long>(nreuse));
    atomicAdd(reinterpret_cast<unsigned long long*>(&info->full_rows), static_cast<unsigned long long>(nfull));
  }
}

}  // namespace spgemm_b200
