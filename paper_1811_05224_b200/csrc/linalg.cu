// linalg.cu — bandwidth-bound FP64 kernels of the solve:
//   * packed block-lower-triangular GEMV (row panels, fixed chunks, warp-shuffle reductions,
//     deterministic two-level sum; no tensor cores: a single right-hand side is not a contraction)
//   * mass matrices: apply, lumped scaling, cyclic-tridiagonal solves (one system per time step)
//   * Krylov vector kernels (block dot products, updates) with fixed reduction order
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"
#include "special.cuh"

namespace stb {

// doubles per work item (32 KB); chunk sizes 2K-16K and unroll 2/4/8 measured within 1% on C3
// (6.73-6.83 TB/s), unroll 8 at 4K best
constexpr int GEMV_CH_DEFAULT = 4096;
constexpr int GEMV_UNROLL = 8;
static int gemv_ch() { return GEMV_CH_DEFAULT; }
constexpr int GEMV_WARPS = 8;

using GSeg = bem_matrix_s::GemvSeg;

// one warp per work item (row i of a panel, chunk c); items enumerated in memory order
template <int UNR>
__global__ void __launch_bounds__(GEMV_WARPS * 32) k_gemv(const double* __restrict__ A,
                                                         const GSeg* __restrict__ segs, int nseg,
                                                         long long n_items, int ng,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ partial, int GEMV_CH) {
  const int lane = threadIdx.x & 31;
  const long long warp0 = (long long)blockIdx.x * GEMV_WARPS + (threadIdx.x >> 5);
  const long long nwarp = (long long)gridDim.x * GEMV_WARPS;
  int sidx = 0;
  for (long long it = warp0; it < n_items; it += nwarp) {
    // locate the segment (items are monotone per warp: linear search forward from last)
    if (it < segs[sidx].item0) sidx = 0;
    while (sidx + 1 < nseg && segs[sidx + 1].item0 <= it) ++sidx;
    const GSeg S = segs[sidx];
    const long long local = it - S.item0;
    const int i = (int)(local / S.nch), c = (int)(local % S.nch);
    const long long col0 = (long long)c * GEMV_CH;
    const int len = (int)min((long long)GEMV_CH, S.len - col0);
    const double* __restrict__ row = A + S.off + (long long)i * S.ld + col0;
    const double* __restrict__ xx = x + S.xoff + col0;
    double acc0 = 0.0, acc1 = 0.0;
    // rows are 32-byte aligned (padded stride, aligned panel offsets) and x offsets are even
    // (b0 * ng + c * GEMV_CH, ng even; odd ng falls back to scalar x loads): A and x as double2
    const int nv = len / 2;
    const double2* __restrict__ row2 = reinterpret_cast<const double2*>(row);
    int k = lane;
    if ((((size_t)xx) & 15) == 0) {
      const double2* __restrict__ x2 = reinterpret_cast<const double2*>(xx);
#pragma unroll UNR
      for (; k < nv; k += 32) {
        const double2 av = __ldcs(row2 + k);   // streamed once: evict-first
        const double2 xv = __ldg(x2 + k);
        acc0 = fma(av.x, xv.x, acc0);
        acc1 = fma(av.y, xv.y, acc1);
      }
    } else {
#pragma unroll 4
      for (; k < nv; k += 32) {
        const double2 av = __ldcs(row2 + k);
        acc0 = fma(av.x, __ldg(xx + 2 * k), acc0);
        acc1 = fma(av.y, __ldg(xx + 2 * k + 1), acc1);
      }
    }
    if ((len & 1) && lane == 0) acc0 = fma(__ldcs(row + len - 1), __ldg(xx + len - 1), acc0);
    double acc = acc0 + acc1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) partial[S.pbase + (long long)i * S.pstride + c] = acc;
  }
}

// ---------------------------------------------------------------- symmetric packed blocks
// reduce-scatter of 32 per-lane values over the warp: lane r returns sum over lanes of v[r]
__device__ __forceinline__ double reduce_scatter32(double (&v)[32], int lane) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int r = 0; r < h; ++r) {
      const double keep = up ? v[r + h] : v[r];
      const double send = up ? v[r] : v[r + h];
      v[r] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

// SYMV of the packed block-lower-triangular matrix: one CTA per (a, b) block, its upper-triangle
// tiles dealt to the warps; an off-diagonal tile T = V_ab[ti, tj] contributes T x_b[tj] to
// y_a[ti] (row sums: a warp reduce-scatter) and T^T x_b[ti] to y_a[tj] (column sums, lane-local);
// each warp accumulates into its own shared-memory copy of y_a, summed in fixed order into one
// partial per (row, b) (deterministic).  Every stored double is read once from HBM.
constexpr int SYMV_WARPS = 4;
// The row reduction is fused: the partials of block (a, b) go to partial[rpbase[a] + b' ng + i]
// (b' = the block's index in its row); the CTA that completes a row (device-scope counter per row,
// reset by it) sums the row's partials in b' order -- fixed, so the result is deterministic -- and
// writes y_a = alpha sum + beta y_a.
__global__ void __launch_bounds__(SYMV_WARPS * 32) k_gemv_sym(const double* __restrict__ A,
                                                             const GSeg* __restrict__ segs, int nseg,
                                                             long long n_items, int ng, long long blk,
                                                             const double* __restrict__ x,
                                                             double* __restrict__ partial,
                                                             const long long* __restrict__ rpbase,
                                                             const int* __restrict__ rpstride,
                                                             int* __restrict__ rowcnt, double alpha,
                                                             double beta, double* __restrict__ y) {
  __shared__ int s_last;
  extern __shared__ double sm[];
  const int nt = sym_nt(ng), L = nt * SYM_TS, ntp = nt * (nt + 1) / 2;
  double* xs = sm;
  double* ys = sm + L;
  double* ds = ys + SYMV_WARPS * L;                    // per-warp diagonal-tile scratch (SYM_TD each)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* yw = ys + w * L;
  for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[mid].item0 <= it) lo = mid; else hi = mid - 1;
    }
    const GSeg S = segs[lo];
    const int bl = (int)(it - S.item0);               // b - b0
    const double* __restrict__ blkp = A + S.off + (long long)bl * blk;
    const double* __restrict__ xb = x + S.xoff + (long long)bl * ng;
    __syncthreads();                                   // the previous item's y is written out
    for (int k = threadIdx.x; k < L; k += blockDim.x) xs[k] = k < ng ? xb[k] : 0.0;
    for (int k = threadIdx.x; k < SYMV_WARPS * L; k += blockDim.x) ys[k] = 0.0;
    __syncthreads();
    int ti = 0, tj = w;                                // tile t = w in row-major upper order
    while (tj >= nt && ti < nt) { tj -= nt - ti - 1; ++ti; }   // w >= ntp: ti reaches nt, no tile
    for (int t = w; t < ntp; t += SYMV_WARPS) {
      const double* __restrict__ tp = blkp + sym_tile_offset(ti, tj, nt);
      const bool cok = tj * SYM_TS + lane < ng;
      double v[32];
      double s = 0.0;
      if (ti != tj) {
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = (cok && ti * SYM_TS + r < ng) ? __ldcs(tp + r * SYM_TS + lane) : 0.0;
        // T^T x_b[ti] -> y_a[tj] (column sums)
#pragma unroll
        for (int r = 0; r < 32; ++r) s = fma(v[r], xs[ti * SYM_TS + r], s);
      } else {
        // diagonal tile, upper triangle stored (row r: columns r..31): read as 17 full-warp
        // coalesced loads into the warp's shared scratch (32 masked row loads would issue as many
        // load instructions as a full tile for half the bytes), then row by row.  The row sums below
        // give sum_{c >= r} T[r][c] x[c]; the strictly upper part transposed adds sum_{r < c} T[r][c] x[r]
        double* dsm = ds + w * SYM_TD;
#pragma unroll
        for (int k = 0; k < (SYM_TD + 31) / 32; ++k)
          if (k * 32 + lane < SYM_TD) dsm[k * 32 + lane] = __ldcs(tp + k * 32 + lane);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r)
          v[r] = (cok && r <= lane && ti * SYM_TS + r < ng) ? dsm[sym_row_base(r, true) + lane] : 0.0;
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) s = fma(r < lane ? v[r] : 0.0, xs[ti * SYM_TS + r], s);
      }
      yw[tj * SYM_TS + lane] += s;
      const double xj = xs[tj * SYM_TS + lane];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] *= xj;
      yw[ti * SYM_TS + lane] += reduce_scatter32(v, lane);
      tj += SYMV_WARPS;                                 // advance to tile t + SYMV_WARPS
      while (tj >= nt && ti < nt) { tj -= nt - ti - 1; ++ti; }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < ng; k += blockDim.x) {
      double yv = 0.0;
#pragma unroll
      for (int ww = 0; ww < SYMV_WARPS; ++ww) yv += ys[ww * L + k];
      partial[S.pbase + (long long)bl * ng + k] = yv;
    }
    __threadfence();                                   // this block's partials, device-wide
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(rowcnt + S.a, 1) == rpstride[S.a] - 1;
    __syncthreads();
    if (s_last) {                                      // the row is complete: reduce it
      __threadfence();
      const double* __restrict__ pr = partial + rpbase[S.a];
      const int nb = rpstride[S.a];
      for (int k = threadIdx.x; k < ng; k += blockDim.x) {
        double sum = 0.0;
        for (int j = 0; j < nb; ++j) sum += __ldcg(pr + (long long)j * ng + k);
        double* yp = y + (long long)S.a * ng + k;
        *yp = (beta == 0.0) ? alpha * sum : fma(alpha, sum, beta * *yp);
      }
      if (threadIdx.x == 0) rowcnt[S.a] = 0;
    }
  }
}

// rows without any owned block (multi-GPU): y = beta y (the fused SYMV reduction never visits them)
__global__ void k_empty_rows(const int* __restrict__ pstride, int ng, int nt, double beta, double* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)ng * nt || pstride[r / ng] != 0) return;
  y[r] = beta == 0.0 ? 0.0 : beta * y[r];
}

// y[a*ng + i] = alpha * sum_k partial[row_pbase[a] + i*stride + k] + beta * y
__global__ void k_gemv_reduce(const double* __restrict__ partial, const long long* __restrict__ pbase,
                              const int* __restrict__ pstride, int ng, int nt, double alpha,
                              double beta, double* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)ng * nt) return;
  const int a = (int)(r / ng), i = (int)(r % ng);
  const int st = pstride[a];
  const double* p = partial + pbase[a] + (long long)i * st;
  double s = 0.0;
  for (int k = 0; k < st; ++k) s += p[k];
  y[r] = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * y[r]);
}

bem_status gemv_setup(bem_matrix* A) {
  const bem_mesh* m = A->mesh;
  const int ng = m->ng, nt = m->nt;
  // partial layout per test step a: all blocks of the block row containing a, in block order
  A->row_pbase.assign(nt, 0);
  A->row_pstride.assign(nt, 0);
  std::vector<std::vector<std::pair<int, int>>> blk_of_a(nt);  // (block index, nch)
  for (size_t bi = 0; bi < m->blocks.size(); ++bi) {
    const Block& b = m->blocks[bi];
    for (int a = b.a0; a < b.a1; ++a) {
      long long len = (long long)panel_nb(a, b.b0, b.b1) * ng;
      if (len <= 0) continue;
      // full storage: chunks of GEMV_CH columns; sym: one partial per trial block b
      int nch = A->sym ? panel_nb(a, b.b0, b.b1) : (int)((len + gemv_ch() - 1) / gemv_ch());
      blk_of_a[a].push_back({(int)bi, nch});
    }
  }
  long long pb = 0;
  for (int a = 0; a < nt; ++a) {
    int st = 0;
    for (auto& pr : blk_of_a[a]) st += pr.second;
    A->row_pbase[a] = pb;
    A->row_pstride[a] = st;
    pb += (long long)st * ng;
  }
  A->n_partials = pb;
  A->empty_rows = false;
  for (int a = 0; a < nt; ++a) A->empty_rows |= A->row_pstride[a] == 0;
  // segments in memory order (block, a)
  A->segs.clear();
  long long item = 0;
  for (size_t bi = 0; bi < m->blocks.size(); ++bi) {
    const Block& b = m->blocks[bi];
    for (int a = b.a0; a < b.a1; ++a) {
      long long len = (long long)panel_nb(a, b.b0, b.b1) * ng;
      if (len <= 0) continue;
      int nch = A->sym ? panel_nb(a, b.b0, b.b1) : (int)((len + gemv_ch() - 1) / gemv_ch());
      int cbase = 0;
      for (auto& pr : blk_of_a[a]) {
        if (pr.first == (int)bi) break;
        cbase += pr.second;
      }
      GSeg s;
      s.item0 = item;
      s.off = A->poff[A->poff_base[bi] + (a - b.a0)];
      s.ld = pad4(len);
      s.len = len;
      s.xoff = (long long)b.b0 * ng;
      // full storage: partial[pbase + i * pstride + chunk]; sym: partial[pbase + b * ng + i]
      s.pbase = A->row_pbase[a] + (A->sym ? (long long)cbase * ng : cbase);
      s.nch = nch;
      s.pstride = A->row_pstride[a];
      s.a = a;
      s.pad = 0;
      A->segs.push_back(s);
      item += A->sym ? (long long)nch : (long long)ng * nch;   // sym: one item per (a, b) block
    }
  }
  A->n_items = item;
  cudaError_t e;
  const cudaStream_t st = A->stream;
  size_t nseg = std::max<size_t>(1, A->segs.size());
  if ((e = cudaMallocAsync((void**)&A->d_segs, sizeof(GSeg) * nseg, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  if ((e = cudaMemcpyAsync(A->d_segs, A->segs.data(), sizeof(GSeg) * A->segs.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  A->partials_bytes = sizeof(double) * std::max<long long>(1, A->n_partials);
  if ((e = storage_acquire(m->device, A->partials_bytes, st, (void**)&A->d_partials)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  if ((e = cudaMallocAsync((void**)&A->d_row_pbase, sizeof(long long) * nt, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  if ((e = cudaMallocAsync((void**)&A->d_row_pstride, sizeof(int) * nt, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  if ((e = cudaMemcpyAsync(A->d_row_pbase, A->row_pbase.data(), sizeof(long long) * nt, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  if ((e = cudaMemcpyAsync(A->d_row_pstride, A->row_pstride.data(), sizeof(int) * nt, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  if (m->comm) {   // distributed mode (any communicator, also one rank)
    if ((e = cudaMallocAsync((void**)&A->d_ysum, sizeof(double) * (size_t)ng * nt, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  }
  if (A->sym) {
    if ((e = cudaMallocAsync((void**)&A->d_rowcnt, sizeof(int) * nt, st)) != cudaSuccess ||
        (e = cudaMemsetAsync(A->d_rowcnt, 0, sizeof(int) * nt, st)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  }
  if (A->sym && comm_overlaps(m) && nt >= 2) {
    // row chunks for the overlapped all-reduce: segments of test steps [row0[c], row0[c+1]) in
    // memory order, items renumbered per chunk
    const int nch = std::min(bem_matrix_s::COMM_CHUNKS, nt);
    std::vector<GSeg> ch;
    for (int c = 0; c < nch; ++c) {
      A->chunk_row0[c] = (int)((long long)nt * c / nch);
      A->chunk_row0[c + 1] = (int)((long long)nt * (c + 1) / nch);
      A->chunk_seg0[c] = (int)ch.size();
      long long it = 0;
      for (const GSeg& g : A->segs) {
        if (g.a < A->chunk_row0[c] || g.a >= A->chunk_row0[c + 1]) continue;
        GSeg x = g;
        x.item0 = it;
        it += x.nch;   // sym: one item per (a, b) block
        ch.push_back(x);
      }
      A->chunk_items[c] = it;
    }
    A->chunk_seg0[nch] = (int)ch.size();
    A->nchunks = nch;
    if ((e = cudaMallocAsync((void**)&A->d_segs_ch, sizeof(GSeg) * std::max<size_t>(1, ch.size()), st)) != cudaSuccess ||
        (ch.size() && (e = cudaMemcpyAsync(A->d_segs_ch, ch.data(), sizeof(GSeg) * ch.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess))
      return cuda_fail(e, "gemv_setup");
    for (int c = 0; c < nch; ++c)
      if ((e = cudaEventCreateWithFlags(&A->chunk_ev[c], cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e, "gemv_setup");
  }
  return BEM_OK;
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// persistent grid: exactly the CTAs that are resident at once (a second partial wave of a
// grid-stride kernel would run at reduced occupancy)
static int g_gemv_ctas_per_sm = 0;
static int gemv_ctas_per_sm() {
  if (!g_gemv_ctas_per_sm) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemv<GEMV_UNROLL>, GEMV_WARPS * 32, 0) != cudaSuccess || n <= 0) n = 4;
    g_gemv_ctas_per_sm = n;
  }
  return g_gemv_ctas_per_sm;
}

bem_status gemv_launch(const bem_matrix* A, double a, const double* x, double b, double* y,
                       cudaStream_t st) {
  if (A->toeplitz) return toeplitz_gemv(A, a, x, b, y, st);
  const bem_mesh* m = A->mesh;
  const long long n = (long long)m->ng * m->nt;
  if (A->n_items > 0 && A->sym) {
    const size_t smem = sizeof(double) * ((1 + SYMV_WARPS) * sym_nt(m->ng) * SYM_TS + SYMV_WARPS * SYM_TD);
    // x, per-warp y and diagonal scratch exceed the default 48 KB beyond N_Gamma ~ 900: opt in
    static size_t smem_set = 48 * 1024;
    if (smem > smem_set) {
      if (cudaFuncSetAttribute(k_gemv_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "bem_matvec: shared memory for this N_Gamma");
      smem_set = smem;
    }
    const long long blocks = std::min<long long>(A->n_items, 1LL << 30);
    // fused row reduction: into y (or the distributed partial sum ysum)
    const bool dist = m->comm != nullptr;
    if (dist && A->nchunks > 1) {
      // multi-GPU with NCCL: row chunk c's all-reduce (on the communicator's stream) overlaps the
      // GEMV of chunk c + 1; rows without owned blocks are zeroed first
      if (A->empty_rows) {
        k_empty_rows<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A->d_row_pstride, m->ng, m->nt, 0.0, A->d_ysum);
        count_launch();
      }
      for (int c = 0; c < A->nchunks; ++c) {
        const int s0 = A->chunk_seg0[c], ns = A->chunk_seg0[c + 1] - s0;
        if (A->chunk_items[c] > 0) {
          k_gemv_sym<<<(unsigned)std::min<long long>(A->chunk_items[c], 1LL << 30), SYMV_WARPS * 32, smem, st>>>(
              A->data, A->d_segs_ch + s0, ns, A->chunk_items[c], m->ng, A->blk_elems, x, A->d_partials, A->d_row_pbase,
              A->d_row_pstride, A->d_rowcnt, 1.0, 0.0, A->d_ysum);
          count_launch();
        }
        cudaEventRecord(A->chunk_ev[c], st);
        const long long r0 = (long long)A->chunk_row0[c] * m->ng, nr = (long long)(A->chunk_row0[c + 1] - A->chunk_row0[c]) * m->ng;
        bem_status s = allreduce_sum_async(m, A->d_ysum + r0, nr, st, A->chunk_ev[c]);
        if (s != BEM_OK) return s;
      }
      bem_status s = comm_join(m, st);
      if (s != BEM_OK) return s;
      vec_axpby(y, a, A->d_ysum, b, n, st);
      cudaError_t e = cudaGetLastError();
      return e == cudaSuccess ? BEM_OK : cuda_fail(e, "bem_matvec");
    }
    k_gemv_sym<<<(unsigned)blocks, SYMV_WARPS * 32, smem, st>>>(A->data, A->d_segs, (int)A->segs.size(), A->n_items, m->ng, A->blk_elems, x, A->d_partials,
                                                                A->d_row_pbase, A->d_row_pstride, A->d_rowcnt,
                                                                dist ? 1.0 : a, dist ? 0.0 : b, dist ? A->d_ysum : y);
    count_launch();
    if (A->empty_rows) {
      k_empty_rows<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A->d_row_pstride, m->ng, m->nt, dist ? 0.0 : b, dist ? A->d_ysum : y);
      count_launch();
    }
    if (dist) {
      bem_status s = allreduce_sum(m, A->d_ysum, n, st);
      if (s != BEM_OK) return s;
      vec_axpby(y, a, A->d_ysum, b, n, st);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BEM_OK : cuda_fail(e, "bem_matvec");
  } else if (A->n_items > 0) {
    long long blocks = std::min<long long>((A->n_items + GEMV_WARPS - 1) / GEMV_WARPS,
                                           (long long)num_sms() * gemv_ctas_per_sm());
    k_gemv<GEMV_UNROLL><<<(unsigned)blocks, GEMV_WARPS * 32, 0, st>>>(A->data, A->d_segs, (int)A->segs.size(), A->n_items, m->ng, x, A->d_partials, gemv_ch());
    count_launch();
  }
  if (m->comm) {   // distributed mode (any communicator, also one rank)
    // partial y over the owned blocks, summed over ranks (NCCL all-reduce = reduce-scatter +
    // all-gather), then y = a * ysum + b * y
    k_gemv_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A->d_partials, A->d_row_pbase, A->d_row_pstride, m->ng, m->nt, 1.0, 0.0, A->d_ysum);
    count_launch();
    bem_status s = allreduce_sum(m, A->d_ysum, n, st);
    if (s != BEM_OK) return s;
    vec_axpby(y, a, A->d_ysum, b, n, st);
  } else {
    k_gemv_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A->d_partials, A->d_row_pbase, A->d_row_pstride, m->ng, m->nt, a, b, y);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "bem_matvec");
}


// ---------------------------------------------------------------- block-Toeplitz variant
// Uniform time steps: A(a, b) = T_{a-b}.  Y[i, a] = sum_{d <= a} sum_j T_d[i, j] X[j, a - d] with
// X[j, b] = x[b ng + j]: one GEMM over the stacked contraction index k = d ng + j (SURVEY 8(f) row
// f3) — a genuine contraction (many right-hand sides through the Toeplitz shift).  CTA tile
// 128 rows i x 128 columns a, K split into lag ranges (fixed partial slots, reduced in fixed order).
// The multiply runs on the FP64 tensor cores (DMMA m8n8k4): their peak is only ~9% above the DFMA
// peak on B200 (37.1 vs 34.1 TFLOP/s, profiles/r01_fp64_peak.txt, r01_dmma_peak.txt) but one
// DMMA does 256 FMAs per warp from 2 operand registers per lane, so the tile loop is no longer
// bound by shared-memory operand loads and issue slots as the 8 x 8 DFMA register tile was.
// a tiles of 64 columns: the lags d > a of a tile's last lag chunk (the triangle, computed on
// zero-filled x) cost TA^2 / 2 per tile, 1/5 of the C4 products at TA = 128, 1/9 at 64.
// 8 warps as 4 (i) x 2 (a), warp tile 32 x 32 = 4 x 4 DMMA tiles, 32 accumulators per lane.
// Shared tiles row-major [i or a][k] with row stride 18 doubles (144 B): the 16-byte fragment loads
// of a quarter warp hit 8 distinct bank quads.  Global -> shared by cp.async (zero-filled outside
// the matrix) in a 3-stage pipeline: the tiles of the next two K steps are in flight while the
// current one is multiplied.
constexpr int TZ_TI = 128, TZ_TA = 64, TZ_TK = 16, TZ_LDK = TZ_TK + 2, TZ_STAGES = 3, TZ_UI = 4, TZ_VA = 4;
constexpr size_t TZ_SMEM = sizeof(double) * TZ_STAGES * (TZ_TI + TZ_TA) * TZ_LDK;
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" :: "r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N)); }
// Work units (1-D grid): a-tile at (in order), then chunk of dpz lags within the tile's lag range
// [0, min(nt, a0 + 128)) (lags beyond the tile's last column contribute nothing), then i-tile: all
// units but a tile's last chunk cost the same, and the host sizes dpz for whole waves of the SMs.
__global__ void __launch_bounds__(256, 2) k_toeplitz_mm(const double* __restrict__ T, long long ldT_d,
                                                    int ldT, const double* __restrict__ x, int ng, int nt,
                                                    int dpz, double* __restrict__ part) {
  extern __shared__ __align__(16) double tz_sm[];
  // stage s: Ts = tz_sm + s * 2 * TI * LDK  ([ii][jj] = T_d[i0 + ii][j0 + jj]),
  //          Xs = Ts + TI * LDK            ([aa][jj] = X[j0 + jj][a0 + aa - d] = x[(a0 + aa - d) ng + j0 + jj])
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = (warp & 3) * (8 * TZ_UI), wa = (warp >> 2) * (8 * TZ_VA), fr = lane & 3, fc = lane >> 2;
  const int nti = (ng + TZ_TI - 1) / TZ_TI;
  int r = blockIdx.x, at = 0;
  for (;; ++at) {
    const int cnt = nti * ((min(nt, (at + 1) * TZ_TA) + dpz - 1) / dpz);
    if (r < cnt) break;
    r -= cnt;
  }
  const int chunk = r / nti, i0 = (r % nti) * TZ_TI, a0 = at * TZ_TA;
  const int d0 = chunk * dpz, d1 = min(min(nt, d0 + dpz), a0 + TZ_TA);   // d > a: nothing
  const int nj = (ng + TZ_TK - 1) / TZ_TK;
  const int nsteps = max(0, d1 - d0) * nj;
  double acc[TZ_UI][TZ_VA][2];
#pragma unroll
  for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
    for (int v = 0; v < TZ_VA; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
  auto issue = [&](int step) {
    double* Ts = tz_sm + (step % TZ_STAGES) * ((TZ_TI + TZ_TA) * TZ_LDK);
    double* Xs = Ts + TZ_TI * TZ_LDK;
    const int d = d0 + step / nj, j0 = (step % nj) * TZ_TK;
#pragma unroll
    for (int q = 0; q < 4; ++q) {            // T: 128 rows x 8 chunks of 16 bytes
      const int e = tid + q * 256, ii = e >> 3, jj = (e & 7) * 2;
      const int i = i0 + ii, j = j0 + jj;
      const int bytes = (i < ng && j < ng) ? (j + 1 < ng ? 16 : 8) : 0;
      const double* src = T + (long long)d * ldT_d + (long long)min(i, ng - 1) * ldT + (bytes ? j : 0);
      cp_async16(Ts + ii * TZ_LDK + jj, src, bytes);
    }
#pragma unroll
    for (int q = 0; q < TZ_TA * 16 / 256; ++q) {  // X: TA columns x 16 doubles (rows of x need not be 16-B aligned)
      const int e = tid + q * 256, aa = e >> 4, jj = e & 15;
      const int b = a0 + aa - d, j = j0 + jj;
      const bool ok = j < ng && b >= 0 && b < nt;
      cp_async8(Xs + aa * TZ_LDK + jj, x + (ok ? (long long)b * ng + j : 0), ok ? 8 : 0);
    }
  };
#pragma unroll
  for (int sgi = 0; sgi < TZ_STAGES - 1; ++sgi) {
    if (sgi < nsteps) issue(sgi);
    cp_async_commit();
  }
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<TZ_STAGES - 2>();
    __syncthreads();                         // stage step % STAGES complete for all threads; the
                                             // stage refilled below was last read in step - 1
    if (step + TZ_STAGES - 1 < nsteps) issue(step + TZ_STAGES - 1);
    cp_async_commit();
    const double* Ts = tz_sm + (step % TZ_STAGES) * ((TZ_TI + TZ_TA) * TZ_LDK);
    const double* Xs = Ts + TZ_TI * TZ_LDK;
    // k order inside the stage: product s of lane (fc, fr) takes k = 4 fr + s (the sum over the 16
    // k of the stage is the same), so a lane's fragments of two products are one 16-byte load
#pragma unroll
    for (int h = 0; h < TZ_TK / 8; ++h) {
      double2 af[TZ_UI], bf[TZ_VA];
#pragma unroll
      for (int u = 0; u < TZ_UI; ++u) af[u] = *reinterpret_cast<const double2*>(Ts + (wi + 8 * u + fc) * TZ_LDK + 4 * fr + 2 * h);
#pragma unroll
      for (int v = 0; v < TZ_VA; ++v) bf[v] = *reinterpret_cast<const double2*>(Xs + (wa + 8 * v + fc) * TZ_LDK + 4 * fr + 2 * h);
#pragma unroll
      for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
        for (int v = 0; v < TZ_VA; ++v) dmma_8x8x4(acc[u][v], af[u].x, bf[v].x);
#pragma unroll
      for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
        for (int v = 0; v < TZ_VA; ++v) dmma_8x8x4(acc[u][v], af[u].y, bf[v].y);
    }
  }
  cp_async_wait<0>();
  // partial Y tile of this lag range: part[z][a][i]; lane holds D[fc][2 fr + e] of each tile
  const long long n = (long long)nt * ng;
#pragma unroll
  for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
    for (int v = 0; v < TZ_VA; ++v)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + wi + 8 * u + fc, a = a0 + wa + 8 * v + 2 * fr + e;
        if (i < ng && a < nt) part[(long long)chunk * n + (long long)a * ng + i] = acc[u][v][e];
      }
}
// TMA version (sm_100a Tensor Memory Accelerator): the T and X tiles of a K step are fetched by
// two cp.async.bulk.tensor copies issued by one thread, completion signalled on the stage's
// mbarrier (expect_tx of the tile bytes; out-of-range rows / columns and the causal x columns
// b < 0 are zero-filled by the TMA unit), 128-byte swizzled in shared memory so that the DMMA
// fragment loads (8 rows x 16 B per quarter warp) stay conflict-free without row padding.  Same
// tiles, work units, warp layout and k order as k_toeplitz_mm.
// Tile shapes (TI x TA, pipeline depth NS): 128 x 64 (4 stages) or 256 x 32 (3 stages; halves the
// zero triangle of each a-tile's last lag chunk, TA^2 / 2 per tile, at twice the T-tile traffic
// from L2).  8 warps of 32 x 32: TI / 32 in i, TA / 32 in a.
template <int TI, int TA, int NS>
struct TzShape {
  static constexpr int stage = (TI + TA) * TZ_TK;                   // doubles per stage
  static constexpr size_t smem = sizeof(double) * NS * stage + 1024 + 128;
};
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(bar), "r"(parity) : "memory");
}
// element (r, k) of a swizzled tile of 16-double rows: the 16-byte chunk k / 2 XOR (r mod 8)
__device__ __forceinline__ const double2* swz(const double* base, int r, int k) {
  return reinterpret_cast<const double2*>(base + r * TZ_TK + ((((k >> 1) ^ (r & 7))) << 1));
}
// one K step (16 deep) of a warp's 32 x 32 tile, the 8-column tiles v >= V0 (V0 = 0: all; skipping
// the causal triangle's zero tiles with V0 > 0 per lag measured slower)
template <int V0>
__device__ __forceinline__ void tz_mma(double (&acc)[TZ_UI][TZ_VA][2], const double* Ts, const double* Xs, int wi,
                                       int wa, int fr, int fc) {
#pragma unroll
  for (int h = 0; h < TZ_TK / 8; ++h) {
    double2 af[TZ_UI], bf[TZ_VA];
#pragma unroll
    for (int u = 0; u < TZ_UI; ++u) af[u] = *swz(Ts, wi + 8 * u + fc, 4 * fr + 2 * h);
#pragma unroll
    for (int v = V0; v < TZ_VA; ++v) bf[v] = *swz(Xs, wa + 8 * v + fc, 4 * fr + 2 * h);
#pragma unroll
    for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
      for (int v = V0; v < TZ_VA; ++v) dmma_8x8x4(acc[u][v], af[u].x, bf[v].x);
#pragma unroll
    for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
      for (int v = V0; v < TZ_VA; ++v) dmma_8x8x4(acc[u][v], af[u].y, bf[v].y);
  }
}
template <int TI, int TA, int NS>
__global__ void __launch_bounds__(256, 2) k_toeplitz_tma(const __grid_constant__ CUtensorMap tmT,
                                                     const __grid_constant__ CUtensorMap tmX, int ng, int nt,
                                                     int dpz, double* __restrict__ part) {
  constexpr int TZ_TSTAGES = NS, TZ_TSTAGE = TzShape<TI, TA, NS>::stage, NWI = TI / 32;
  static_assert(NWI * (TA / 32) == 8, "8 warps of 32 x 32");
  extern __shared__ __align__(16) unsigned char tz_raw[];
  // 1024-byte aligned stages (the swizzle pattern repeats every 8 rows of 128 B)
  double* tz = reinterpret_cast<double*>((reinterpret_cast<size_t>(tz_raw) + 1023) & ~size_t(1023));
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(tz + TZ_TSTAGES * TZ_TSTAGE);   // full
  unsigned long long* ebar = bar + TZ_TSTAGES;                                                  // empty
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = (warp % NWI) * (8 * TZ_UI), wa = (warp / NWI) * (8 * TZ_VA), fr = lane & 3, fc = lane >> 2;
  const int nti = (ng + TI - 1) / TI;
  int r = blockIdx.x, at = 0;
  for (;; ++at) {
    const int cnt = nti * ((min(nt, (at + 1) * TA) + dpz - 1) / dpz);
    if (r < cnt) break;
    r -= cnt;
  }
  const int chunk = r / nti, i0 = (r % nti) * TI, a0 = at * TA;
  const int d0 = chunk * dpz, d1 = min(min(nt, d0 + dpz), a0 + TA);
  const int nj = (ng + TZ_TK - 1) / TZ_TK;
  const int nsteps = max(0, d1 - d0) * nj;
  if (tid == 0) {
    for (int s = 0; s < TZ_TSTAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" :: "r"(smem_u32(ebar + s)));   // one arrival per warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int step) {   // thread 0
    const int s = step % TZ_TSTAGES;
    double* Ts = tz + s * TZ_TSTAGE;
    double* Xs = Ts + TI * TZ_TK;
    const int d = d0 + step / nj, j0 = (step % nj) * TZ_TK;
    const unsigned b = smem_u32(bar + s);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"((unsigned)(sizeof(double) * TZ_TSTAGE)) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 :: "r"(smem_u32(Ts)), "l"(reinterpret_cast<unsigned long long>(&tmT)), "r"(j0), "r"(i0), "r"(d), "r"(b)
                 : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(Xs)), "l"(reinterpret_cast<unsigned long long>(&tmX)), "r"(j0), "r"(a0 - d), "r"(b)
                 : "memory");
  };
  double acc[TZ_UI][TZ_VA][2];
#pragma unroll
  for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
    for (int v = 0; v < TZ_VA; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
  // producer / consumer ring without block barriers: stage s holds step k (k mod S = s); a warp
  // waits on full[s], multiplies, and its lane 0 arrives on empty[s]; thread 0 refills stage s with
  // step k + S once all eight warps arrived
  if (tid == 0)
    for (int k = 0; k < TZ_TSTAGES && k < nsteps; ++k) issue(k);
  for (int step = 0; step < nsteps; ++step) {
    const int st_ = step % TZ_TSTAGES;
    const unsigned ph = (unsigned)((step / TZ_TSTAGES) & 1);
    mbar_wait(smem_u32(bar + st_), ph);
    const double* Ts = tz + st_ * TZ_TSTAGE;
    tz_mma<0>(acc, Ts, Ts + TI * TZ_TK, wi, wa, fr, fc);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(ebar + st_)) : "memory");
    if (tid == 0 && step + TZ_TSTAGES < nsteps) {
      mbar_wait(smem_u32(ebar + st_), ph);                            // all warps are done with stage st_
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before async writes
      issue(step + TZ_TSTAGES);
    }
  }
  const long long n = (long long)nt * ng;
#pragma unroll
  for (int u = 0; u < TZ_UI; ++u)
#pragma unroll
    for (int v = 0; v < TZ_VA; ++v)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + wi + 8 * u + fc, a = a0 + wa + 8 * v + 2 * fr + e;
        if (i < ng && a < nt) part[(long long)chunk * n + (long long)a * ng + i] = acc[u][v][e];
      }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    cudaGetLastError();
  }
  return fn;
}

__global__ void k_toeplitz_reduce(const double* __restrict__ part, int nsplit, long long n, double alpha,
                                  double beta, double* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (int z = 0; z < nsplit; ++z) s += part[(long long)z * n + r];
  y[r] = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * y[r]);
}

// one TMA tile shape's launch: tensor maps, occupancy, lag chunk, units (false: not applicable)
struct TzLaunch {
  int ti, ta, ns, ctas;
  size_t smem;
  void (*kern)(CUtensorMap, CUtensorMap, int, int, int, double*);
};
template <int TI, int TA, int NS>
static TzLaunch tz_launch() {
  static int ctas = 0;
  const size_t smem = TzShape<TI, TA, NS>::smem;
  if (!ctas) {
    cudaFuncSetAttribute(k_toeplitz_tma<TI, TA, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, k_toeplitz_tma<TI, TA, NS>, 256, smem) != cudaSuccess || ctas < 1) ctas = 1;
  }
  return TzLaunch{TI, TA, NS, ctas, smem,
                  reinterpret_cast<void (*)(CUtensorMap, CUtensorMap, int, int, int, double*)>(k_toeplitz_tma<TI, TA, NS>)};
}

bem_status toeplitz_gemv(const bem_matrix* A, double a, const double* x, double b, double* y,
                         cudaStream_t st) {
  const bem_mesh* m = A->mesh;
  const int ng = m->ng, nt = m->nt;
  const long long n = (long long)ng * nt;
  static bool attr = false;
  static int tz_ctas = 1;
  if (!attr) {
    cudaFuncSetAttribute(k_toeplitz_mm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TZ_SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tz_ctas, k_toeplitz_mm, 256, TZ_SMEM) != cudaSuccess || tz_ctas < 1) tz_ctas = 1;
    attr = true;
  }
  const long long ldT_d = A->poff.size() > 1 ? A->poff[1] - A->poff[0] : 0;
  // TMA path: tensor maps of T (j, i, d) and of this product's x (j, b); the strides must be
  // multiples of 16 bytes (N_Gamma even) and x 16-byte aligned -- otherwise the cp.async kernel
  static const bool no_tma = getenv("BEM_TOEPLITZ_NO_TMA") != nullptr;
  static const int shape = getenv("BEM_TZ_SHAPE") ? atoi(getenv("BEM_TZ_SHAPE")) : 1;
  EncodeTiledFn enc = no_tma ? nullptr : encode_tiled();
  bool tma = enc && ng % 2 == 0 && ((size_t)x & 15) == 0 && ldT_d > 0 && nt > 1;
  TzLaunch L{TZ_TI, TZ_TA, TZ_STAGES, tz_ctas, TZ_SMEM, nullptr};
  if (tma) L = shape == 0 ? tz_launch<128, 64, 4>() : (shape == 2 ? tz_launch<256, 32, 4>() : tz_launch<256, 32, 3>());
  CUtensorMap tmT, tmX;
  if (tma) {
    const cuuint64_t gT[3] = {(cuuint64_t)ng, (cuuint64_t)ng, (cuuint64_t)nt};
    const cuuint64_t sT[2] = {(cuuint64_t)pad4(ng) * 8, (cuuint64_t)ldT_d * 8};
    const cuuint32_t bT[3] = {TZ_TK, (cuuint32_t)L.ti, 1}, one3[3] = {1, 1, 1};
    const cuuint64_t gX[2] = {(cuuint64_t)ng, (cuuint64_t)nt};
    const cuuint64_t sX[1] = {(cuuint64_t)ng * 8};
    const cuuint32_t bX[2] = {TZ_TK, (cuuint32_t)L.ta}, one2[2] = {1, 1};
    tma = enc(&tmT, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)A->data, gT, sT, bT, one3, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
          enc(&tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)x, gX, sX, bX, one2, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (!tma) L = TzLaunch{TZ_TI, TZ_TA, TZ_STAGES, tz_ctas, TZ_SMEM, nullptr};   // the cp.async kernel
  // lag chunk dpz: minimise the busiest SM's time, (units per SM) x (dpz + 4), where two co-resident
  // units share the SM's FP64 tensor pipe at ~1.15x the throughput of one (C4 measured)
  const int nti = (ng + L.ti - 1) / L.ti, nta = (nt + L.ta - 1) / L.ta, sms = num_sms();
  auto units = [&](int dz) {
    long long u = 0;
    for (int at = 0; at < nta; ++at) u += (long long)nti * ((std::min(nt, (at + 1) * L.ta) + dz - 1) / dz);
    return u;
  };
  int dpz = nt;
  double best = 1e300;
  for (int dz = std::min(nt, 8); dz <= nt; ++dz) {
    const long long u = units(dz);
    const long long per_sm = (u + sms - 1) / sms;
    const double cost = (double)per_sm * (dz + 4) / (per_sm >= 2 && L.ctas >= 2 ? 1.15 : 1.0);   // + 4: fill / epilogue
    if (cost < best) best = cost, dpz = dz;
  }
  const long long nunits = units(dpz);
  const int nsplit = (nt + dpz - 1) / dpz;
  double* part = nullptr;
  const size_t bytes = sizeof(double) * n * nsplit;
  cudaError_t e = storage_acquire(m->device, bytes, st, (void**)&part);
  if (e != cudaSuccess) return cuda_fail(e, "toeplitz product");
  e = cudaMemsetAsync(part, 0, bytes, st);   // lag ranges beyond a tile's columns leave their slots zero
  if (tma) {
    L.kern<<<(unsigned)nunits, 256, L.smem, st>>>(tmT, tmX, ng, nt, dpz, part);
  } else {
    k_toeplitz_mm<<<(unsigned)nunits, 256, TZ_SMEM, st>>>(A->data, ldT_d, (int)pad4(ng), x, ng, nt, dpz, part);
  }
  k_toeplitz_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nsplit, n, a, b, y);
  count_launch(2);
  storage_release(m->device, part, bytes, st);
  e = cudaGetLastError();
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "toeplitz product");
}

// ------------------------------------------------------------------ mass matrices
// primal (eq. 4): M[(a,i),(a,i)] = M[(a,i),(a,i+1)] = h_t(a) h_i / 2
// dual (Thm 1):   lower h_{l-1} v-/4, diag h_l (2 + v- + v+)/4, upper h_{l+1} v+/4 (times h_t(a))
// lumped: row sums of the dual mass
__global__ void k_mass_fill(int kind, const Seg* __restrict__ seg, const Dual* __restrict__ dual,
                            const double* __restrict__ t, int ng, int nt, double* lo, double* di,
                            double* up) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)ng * nt) return;
  const int a = (int)(r / ng), l = (int)(r % ng);
  const double ht = t[a + 1] - t[a];
  const double hm = seg[(l - 1 + ng) % ng].h, h0 = seg[l].h, hp = seg[(l + 1) % ng].h;
  if (kind == BEM_MASS_PRIMAL) {
    lo[r] = 0.0;
    di[r] = 0.5 * ht * h0;
    up[r] = 0.5 * ht * h0;
  } else {
    const double vm = dual[l].vm, vp = dual[l].vp;
    const double L = ht * hm * vm * 0.25, D = ht * h0 * (2.0 + vm + vp) * 0.25, U = ht * hp * vp * 0.25;
    if (kind == BEM_MASS_DUAL) {
      lo[r] = L; di[r] = D; up[r] = U;
    } else {
      lo[r] = 0.0; di[r] = (L + D) + U; up[r] = 0.0;
    }
  }
}

__global__ void k_cyclic_factor(const double* __restrict__ lo, const double* __restrict__ di,
                                const double* __restrict__ up, int ng, int nt, int staged, double* __restrict__ fac);

bem_status mass_setup(bem_matrix* M, int kind) {
  const bem_mesh* m = M->mesh;
  const long long n = (long long)m->ng * m->nt;
  M->mass_kind = kind;
  cudaError_t e;
  const cudaStream_t st = M->stream;
  mesh_wait(m, st);
  if ((e = cudaMallocAsync((void**)&M->d_lo, sizeof(double) * n, st)) != cudaSuccess ||
      (e = cudaMallocAsync((void**)&M->d_di, sizeof(double) * n, st)) != cudaSuccess ||
      (e = cudaMallocAsync((void**)&M->d_up, sizeof(double) * n, st)) != cudaSuccess ||
      (e = cudaMallocAsync((void**)&M->d_work, sizeof(double) * 2 * (4 * n + 2LL * m->nt), st)) != cudaSuccess)
    return cuda_fail(e, "bem_assemble_M");
  k_mass_fill<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(kind, m->d_seg, m->d_dual, m->d_t, m->ng, m->nt, M->d_lo, M->d_di, M->d_up);
  count_launch();
  if (kind == BEM_MASS_DUAL) {   // factorisation for both transpose flags, once per matrix
    static int fmax_smem = -1;
    if (fmax_smem < 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&fmax_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) fmax_smem = 48 * 1024;
      cudaFuncSetAttribute(k_cyclic_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, fmax_smem);
    }
    const size_t fsmem = sizeof(double) * 7 * (size_t)m->ng;
    const int fstaged = fsmem <= (size_t)fmax_smem;
    k_cyclic_factor<<<2 * m->nt, 32, fstaged ? fsmem : 0, st>>>(M->d_lo, M->d_di, M->d_up, m->ng, m->nt, fstaged,
                                                                M->d_work);
    count_launch();
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "bem_assemble_M");
}

__global__ void k_mass_apply(const double* __restrict__ lo, const double* __restrict__ di,
                             const double* __restrict__ up, int ng, int nt, double a,
                             const double* __restrict__ x, double b, double* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)ng * nt) return;
  const int i = (int)(r % ng);
  const long long base = r - i;
  const double v = lo[r] * x[base + (i - 1 + ng) % ng] + di[r] * x[r] + up[r] * x[base + (i + 1) % ng];
  y[r] = (b == 0.0) ? a * v : fma(a, v, b * y[r]);
}

bem_status mass_apply(const bem_matrix* M, double a, const double* x, double b, double* y,
                      cudaStream_t st) {
  const bem_mesh* m = M->mesh;
  const long long n = (long long)m->ng * m->nt;
  k_mass_apply<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(M->d_lo, M->d_di, M->d_up, m->ng, m->nt, a, x, b, y);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "mass_apply");
}

// cyclic tridiagonal solve per time step (Sherman-Morrison around the Thomas algorithm).
// Row l of the (transposed) system: sub s_l at column l-1, diag d_l, super p_l at column l+1.
// Cyclic tridiagonal dual mass (one system of N_Gamma unknowns per time step): the
// factorisation does not depend on the right-hand side, so it is computed once per matrix and
// transpose flag (k_cyclic_factor: Thomas on the first / last diagonal modified system plus the
// Sherman-Morrison vector z), and a solve is a forward / backward substitution with precomputed
// multipliers: one warp per time step stages x and the factors in shared memory (coalesced) and
// scales x by the pivots' inverses; the two recurrences -- one FMA per element each,
// v_l = x_l inv_l - (sl_l inv_l) v_{l-1} and v_l = yy_l - cp_l v_{l+1} -- run as warp scans of
// affine maps (below); the warp writes y = yy - fact z.
// factor layout per (transpose t, step a): [sl inv, inv, cp, zz] x ng, then 2 scalars (alpha/gam, den)
// one warp per (transpose, step): the three diagonals staged in shared memory with coalesced
// loads, lane 0 runs the recurrences out of shared memory (a thread per step reading global
// memory waited on an L2 round trip per element: C5 0.36 ms per factorisation), the warp writes
// the factors; staged = 0 (N_Gamma beyond the shared-memory limit): the same from global memory
__global__ void __launch_bounds__(32) k_cyclic_factor(const double* __restrict__ lo, const double* __restrict__ di,
                                                     const double* __restrict__ up, int ng, int nt, int staged,
                                                     double* __restrict__ fac) {
  extern __shared__ double fsm[];   // lo, di, up, sl, inv, cp, zz (7 ng) when staged
  const int id = blockIdx.x, lane = threadIdx.x;
  const int transpose = id / nt, a = id % nt;
  const long long base = (long long)a * ng;
  double* F = fac + (long long)id * (4LL * ng + 2);
  const double* Lo = staged ? fsm : lo + base;
  const double* Di = staged ? fsm + ng : di + base;
  const double* Up = staged ? fsm + 2 * ng : up + base;
  double* sl = staged ? fsm + 3 * ng : F;
  double* inv = staged ? fsm + 4 * ng : F + ng;
  double* cp = staged ? fsm + 5 * ng : F + 2 * ng;
  double* zz = staged ? fsm + 6 * ng : F + 3 * ng;
  if (staged) {
    for (int l = lane; l < ng; l += 32) {
      fsm[l] = lo[base + l];
      fsm[ng + l] = di[base + l];
      fsm[2 * ng + l] = up[base + l];
    }
  }
  __syncwarp();
  if (lane == 0) {
    auto sub = [&](int l) -> double { return transpose ? Up[(l - 1 + ng) % ng] : Lo[l]; };
    auto sup = [&](int l) -> double { return transpose ? Lo[(l + 1) % ng] : Up[l]; };
    const double alpha_c = sub(0);      // row 0, column ng-1
    const double beta_c = sup(ng - 1);  // row ng-1, column 0
    const double gam = -Di[0];
    double den = Di[0] - gam;
    sl[0] = 0.0;
    inv[0] = 1.0 / den;
    cp[0] = sup(0) * inv[0];
    zz[0] = gam * inv[0];
    for (int l = 1; l < ng; ++l) {
      double bl = Di[l];
      if (l == ng - 1) bl -= alpha_c * beta_c / gam;
      const double sv = sub(l);
      den = bl - sv * cp[l - 1];
      inv[l] = 1.0 / den;
      sl[l] = sv * inv[l];
      cp[l] = (l < ng - 1) ? sup(l) * inv[l] : 0.0;
      const double ul = (l == ng - 1) ? beta_c : 0.0;
      zz[l] = (ul - sv * zz[l - 1]) * inv[l];
    }
    for (int l = ng - 2; l >= 0; --l) zz[l] -= cp[l] * zz[l + 1];
    F[4 * ng] = alpha_c / gam;
    F[4 * ng + 1] = 1.0 + zz[0] + (alpha_c / gam) * zz[ng - 1];
  }
  __syncwarp();
  if (staged)
    for (int l = lane; l < 4 * ng; l += 32) F[l] = fsm[3 * ng + l];
}

// staged: x and the factors in shared memory (4 ng doubles); otherwise (N_Gamma beyond the
// shared-memory limit) the recurrences run on y and the factors in global memory
__global__ void __launch_bounds__(32) k_cyclic_solve(const double* __restrict__ fac, int ng, int nt,
                                                    int transpose, int staged, const double* x,
                                                    double* y) {
  extern __shared__ double sm[];   // x / yy, sl, inv, cp  (4 ng)
  const int a = blockIdx.x, lane = threadIdx.x;
  const long long base = (long long)a * ng;
  const double* F = fac + ((long long)transpose * nt + a) * (4LL * ng + 2);
  double* yy = staged ? sm : y + base;
  const double* sl = staged ? sm + ng : F;
  const double* inv = staged ? sm + 2 * ng : F + ng;
  const double* cp = staged ? sm + 3 * ng : F + 2 * ng;
  if (staged) {
    for (int l = lane; l < ng; l += 32) {
      yy[l] = x[base + l] * F[ng + l];
      sm[ng + l] = F[l];
      sm[3 * ng + l] = F[2 * ng + l];
    }
  } else {
    for (int l = lane; l < ng; l += 32) yy[l] = x[base + l] * inv[l];
  }
  __syncwarp();
  // the two first-order recurrences v_l = yy_l - c_l v_(l-1/l+1) as warp scans of affine maps:
  // lane j composes the maps of its chunk (v -> A v + B), an exclusive shuffle scan composes the
  // chunks before it, and the lane runs its chunk from the incoming value (the dependent chain is
  // 2 x chunk + 5 steps instead of ng: FP64 FMA latency bound, C5 32 -> 16 us per solve)
  const int nfw = ng - 1, chk = (nfw + 31) / 32;
  auto sweep = [&](const double* coef, int dir) {
    // element k of the sweep (k = 0 .. ng - 2): index 1 + k forward, ng - 2 - k backward
    const int k0 = min(nfw, lane * chk), k1 = min(nfw, k0 + chk);
    double A = 1.0, Bv = 0.0;
    for (int k = k0; k < k1; ++k) {
      const int l = dir > 0 ? 1 + k : ng - 2 - k;
      A = -coef[l] * A;
      Bv = fma(-coef[l], Bv, yy[l]);
    }
    // exclusive scan: compose the maps of lanes < lane (in order), identity for lane 0
    double eA = __shfl_up_sync(0xffffffffu, A, 1), eB = __shfl_up_sync(0xffffffffu, Bv, 1);
    if (lane == 0) { eA = 1.0; eB = 0.0; }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double pA = __shfl_up_sync(0xffffffffu, eA, d), pB = __shfl_up_sync(0xffffffffu, eB, d);
      if (lane >= d) {   // (this prefix) after (the earlier prefix): v -> eA (pA v + pB) + eB
        eB = fma(eA, pB, eB);
        eA = eA * pA;
      }
    }
    const double v0 = dir > 0 ? yy[0] : yy[ng - 1];
    double v = fma(eA, v0, eB);
    __syncwarp();
    for (int k = k0; k < k1; ++k) {
      const int l = dir > 0 ? 1 + k : ng - 2 - k;
      v = fma(-coef[l], v, yy[l]);
      yy[l] = v;
    }
    __syncwarp();
  };
  sweep(sl, 1);
  sweep(cp, -1);
  __syncwarp();
  const double fact = (yy[0] + F[4 * ng] * yy[ng - 1]) / F[4 * ng + 1];
  __syncwarp();
  for (int l = lane; l < ng; l += 32) y[base + l] = yy[l] - fact * F[3 * ng + l];
}

__global__ void k_diag_solve(const double* __restrict__ di, long long n, const double* __restrict__ x,
                             double* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = x[r] / di[r];
}

bem_status mass_solve(const bem_matrix* M, int transpose, const double* x, double* y,
                      cudaStream_t st) {
  const bem_mesh* m = M->mesh;
  const long long n = (long long)m->ng * m->nt;
  if (M->mass_kind == BEM_MASS_DUAL_LUMPED) {
    k_diag_solve<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(M->d_di, n, x, y);
  } else {
    // shared staging up to the opt-in limit (N_Gamma <= 7264 at 227 KB), global memory beyond
    static int smem_max = -1;
    if (smem_max < 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) smem_max = 48 * 1024;
      cudaFuncSetAttribute(k_cyclic_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    }
    const size_t smem = sizeof(double) * 4 * (size_t)m->ng;
    const int staged = smem <= (size_t)smem_max;
    k_cyclic_solve<<<m->nt, 32, staged ? smem : 0, st>>>(M->d_work, m->ng, m->nt, transpose ? 1 : 0, staged, x, y);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "mass_solve");
}

// ------------------------------------------------------------------ vector kernels
// out[j] = sum_n Q[j*ldq + n] w[n] for j < k: one CTA per j, fixed-order tree reduction
// out[j] = <Q_j, w> for j < k: 2-D grid (vector j, chunk c) writes partials, k_dots_sum adds the
// chunks in fixed order (deterministic; enough CTAs to stream the k+1 vectors at HBM speed)
constexpr int DOT_CHUNK = 8192;
constexpr int DOT_MAXCH = 1024;
__global__ void k_dots(const double* __restrict__ Q, long long ldq, const double* __restrict__ w,
                       long long n, long long chunk, double* __restrict__ part) {
  __shared__ double red[8];
  const int j = blockIdx.x, c = blockIdx.y;
  const double* q = Q + (long long)j * ldq;
  const long long r0 = (long long)c * chunk, r1 = min(n, r0 + chunk);
  double s = 0.0;
  for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) s = fma(q[r], w[r], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    part[(long long)j * gridDim.y + c] = t;
  }
}
__global__ void k_dots_sum(const double* __restrict__ part, int nch, int k, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int c = 0; c < nch; ++c) s += part[(long long)j * nch + c];
  out[j] = s;
}
// per host thread and device (concurrent solves on several threads each own theirs), freed when
// the thread exits
struct DotScratch {
  double* p[64] = {nullptr};
  size_t n[64] = {0};
  ~DotScratch() {
    for (int d = 0; d < 64; ++d)
      if (p[d]) cudaFree(p[d]);
    cudaGetLastError();
  }
};
static thread_local DotScratch g_dot;
void vec_dots(const double* Q, long long ldq, int k, const double* w, long long n, double* out,
              cudaStream_t st) {
  const int nch = (int)std::max<long long>(1, std::min<long long>(DOT_MAXCH, (n + DOT_CHUNK - 1) / DOT_CHUNK));
  const long long chunk = (n + nch - 1) / nch;
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  const size_t need = (size_t)k * nch;
  if (need > g_dot.n[dev]) {
    // per-device scratch, grows rarely (largest k seen); stream-ordered free / allocation
    if (g_dot.p[dev]) cudaFreeAsync(g_dot.p[dev], st);
    g_dot.n[dev] = std::max<size_t>(need, 64 * 1024);
    cudaMallocAsync((void**)&g_dot.p[dev], sizeof(double) * g_dot.n[dev], st);
  }
  dim3 grid(k, nch);
  k_dots<<<grid, 256, 0, st>>>(Q, ldq, w, n, chunk, g_dot.p[dev]);
  k_dots_sum<<<(k + 127) / 128, 128, 0, st>>>(g_dot.p[dev], nch, k, out);
  count_launch(2);
}

// w[n] -= sum_j h[j] Q[j][n]
__global__ void k_update(double* __restrict__ w, const double* __restrict__ Q, long long ldq, int k,
                         const double* __restrict__ h, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (int j = 0; j < k; ++j) s = fma(h[j], Q[(long long)j * ldq + r], s);
  w[r] -= s;
}
void vec_update(double* w, const double* Q, long long ldq, int k, const double* h, long long n,
                cudaStream_t st) {
  k_update<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, Q, ldq, k, h, n);
  count_launch();
}
// out[n] = sum_j coef[j] Q[j][n]
__global__ void k_combine(double* __restrict__ out, const double* __restrict__ Q, long long ldq,
                          int k, const double* __restrict__ coef, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  for (int j = 0; j < k; ++j) s = fma(coef[j], Q[(long long)j * ldq + r], s);
  out[r] = s;
}
void vec_combine(double* out, const double* Q, long long ldq, int k, const double* coef, long long n,
                 cudaStream_t st) {
  k_combine<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, Q, ldq, k, coef, n);
  count_launch();
}
__global__ void k_scale(double* __restrict__ y, const double* __restrict__ x, double s, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = s * x[r];
}
void vec_scale(double* y, const double* x, double s, long long n, cudaStream_t st) {
  k_scale<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, x, s, n);
  count_launch();
}
// y = x / sqrt(*nrm2) (the next Arnoldi vector, scaled on the device so that the host need not
// read the norm first); left untouched on breakdown (sqrt(*nrm2) <= 1e-300)
__global__ void k_scale_rnorm(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ nrm2,
                              long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const double h = sqrt(*nrm2);
  if (r < n && h > 1e-300) y[r] = (1.0 / h) * x[r];
}
void vec_scale_rnorm(double* y, const double* x, const double* nrm2_dev, long long n, cudaStream_t st) {
  k_scale_rnorm<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, x, nrm2_dev, n);
  count_launch();
}
__global__ void k_axpby(double* __restrict__ y, double a, const double* __restrict__ x, double b, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = (b == 0.0) ? a * x[r] : fma(a, x[r], b * y[r]);
}
void vec_axpby(double* y, double a, const double* x, double b, long long n, cudaStream_t st) {
  k_axpby<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, a, x, b, n);
  count_launch();
}
__global__ void k_mul(double* __restrict__ y, const double* __restrict__ d, const double* __restrict__ x, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = d[r] * x[r];
}
void vec_mul(double* y, const double* d, const double* x, long long n, cudaStream_t st) {
  k_mul<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(y, d, x, n);
  count_launch();
}

// ------------------------------------------------------------------ special-function probe
__global__ void k_special(int which, long long n, const double* __restrict__ x, double* __restrict__ out) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double v = x[r];
  double o;
  if (which == 0) o = dev_e1(v);
  else if (which == 1) o = dev_ein(v);
  else if (which == 2) o = dev_hfun(v);
  else o = dev_psi(v);
  out[r] = o;
}
bem_status eval_special(int which, long long n, const double* x, double* out, cudaStream_t st) {
  if (n <= 0) return BEM_OK;
  k_special<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(which, n, x, out);
  count_launch();
  cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "bem_eval_special");
}

}  // namespace stb

namespace stb {
// live FP64 rate (bem_diag_fp64_rate): 8 independent DFMA chains per thread, 256 threads, 8 CTAs
// per SM -- the denominator of the assembly roofline measured in the thermal / power state of the
// moment (the bulk kernels run under the board power cap)
__global__ void __launch_bounds__(256) k_dfma_rate(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;   // keeps the chains alive
}
bem_status diag_fp64_rate(double seconds, double* tflops) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaError_t e = cudaMalloc((void**)&d, sizeof(double));
  if (e != cudaSuccess) return cuda_fail(e, "bem_diag_fp64_rate");
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int grid = nsm * 8, tpb = 256, iters = 2000;
  const double flops = 2.0 * grid * tpb * (double)iters * 16 * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // back to back for `seconds`; the rate of the second half (the sustained clock)
  double total = 0.0, t_half = 0.0, fl_half = 0.0;
  while (total < seconds) {
    cudaEventRecord(e0, st);
    for (int r = 0; r < 4; ++r) k_dfma_rate<<<grid, tpb, 0, st>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1, st);
    if ((e = cudaEventSynchronize(e1)) != cudaSuccess) break;
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms <= 0.0f) break;
    total += 1e-3 * ms;
    if (total >= 0.5 * seconds) { t_half += 1e-3 * ms; fl_half += 4.0 * flops; }
  }
  count_launch();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(d);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bem_diag_fp64_rate");
  *tflops = t_half > 0.0 ? fl_half / t_half / 1e12 : 0.0;
  return BEM_OK;
}
__global__ void k_gather(const double* __restrict__ data, const long long* __restrict__ offs, long long n,
                         double* __restrict__ out) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) out[r] = offs[r] >= 0 ? data[offs[r]] : 0.0;
}
bem_status gather_entries(const double* data, const long long* offs, long long n, double* out, cudaStream_t st) {
  if (n <= 0) return BEM_OK;
  k_gather<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(data, offs, n, out);
  count_launch();
  cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? BEM_OK : cuda_fail(e, "gather_entries");
}
}  // namespace stb
