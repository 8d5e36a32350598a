// Shared device-side definitions: slab geometry, device state, reductions.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace topo {

// ---------------------------------------------------------------------------
// Slab geometry.  One slab = elements [ex0, ex1)
// along x; nodes [ex0, ex0+nown) are owned (the last slab also owns ix=nelx).
//
// Node arrays, per component c (SoA), x slowest:
//   idx = c*ncomp + ixl*nplane + (iz+1)*NY + (iy+1),  ixl = ix - ex0 + 1
// ixl = 0 and ixl = nown+1 are ghost planes (neighbour slab or zero outside
// the domain); y and z carry one zero pad node on each side, so every node's
// 26 neighbours are addressable without bounds checks.
//
// Element arrays: idx = exl*eplane + (ez+1)*EY + (ey+1), exl = ex - ex0 + H,
// H >= max(1, R) halo planes each side (R = filter radius in elements); one
// zero pad element on each side in y and z.  Out-of-domain entries are 0.
// ---------------------------------------------------------------------------
struct Geo {
  int nelx, nely, nelz;
  int ex0, ex1, nex;       // owned elements [ex0, ex1), nex = ex1 - ex0
  int nown;                // owned node planes
  int NY, NZ, NXL;         // node pitches: NY >= nely+3 (mult. of 4), NZ = nelz+3, NXL = nown+2
  long long nplane;        // NY*NZ
  long long ncomp;         // NXL*nplane
  int H;                   // element halo planes
  int EY, EZ, NEXL;        // EY >= nely+2 (mult. of 4), EZ = nelz+2, NEXL = nex + 2H
  long long eplane;        // EY*EZ
  long long nelloc;        // NEXL*eplane
};

__host__ __device__ inline long long node_idx(const Geo& g, int ix, int iy, int iz) {
  return (long long)(ix - g.ex0 + 1) * g.nplane + (long long)(iz + 1) * g.NY + (iy + 1);
}
__host__ __device__ inline long long elem_idx(const Geo& g, int ex, int ey, int ez) {
  return (long long)(ex - g.ex0 + g.H) * g.eplane + (long long)(ez + 1) * g.EY + (ey + 1);
}

// Device-resident scalar state of one slab (PCG + OC + scratch sums).
// Programmatic dependent launch (sm_90+): every kernel of this library starts with
// pdl_enter().  launch_dependents lets a kernel launched after it with the
// programmatic-serialization attribute (LAUNCH: TOPO_PDL) be scheduled as soon
// as every CTA of this one has started; wait blocks until the preceding grid has
// completed and its memory is visible -- so reads of its outputs stay ordered.
// Both are no-ops when the kernel was not launched that way.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

struct DevState {
  // PCG
  double rz;        // r^T M^{-1} r of the current residual
  double pq;        // p^T K p
  double alpha, beta;
  double rr;        // ||r||^2 (free DOFs)
  double bb;        // ||f_free||^2
  double tol2;      // cg_rtol^2
  long long it;     // iterations done in this solve
  long long max_it;
  int done;         // 1 -> PCG kernels are no-ops
  int status;       // 0 ok, 2 ENOCONV, 3 EBREAKDOWN
  int fresh;        // 1 -> next p-update uses beta = 0 (start / restart)
  int pending;      // 1 -> u lacks alpha_prev * p (applied by the next odd update or a flush)
  int solo;         // TOPO_DIST_SOLO timing runs: no convergence / breakdown exit (max_it iterations)
  double alpha_prev;
  // OC bisection
  double l1, l2, lmid, target, vol, oc_tol;
  int oc_active, oc_pass;
  double oc_frozen;    // OC after compaction: volume of the elements frozen at a clamp bound
  double oc_lin;       // ... sum of dv~ A over the elements unclamped for every remaining lambda
  int oc_glo, oc_ghi;  // OC phase-1 grid search: last k with V(lmax 2^-k) <= target, first known > (0: none)
  double oc_gvhi;      // ... V at k = oc_ghi
  long long oc_nact;   // ... and the number of active (compacted) elements
  // landing zone of per-slab partial sums (allreduced across slabs)
  double sums[8];
};

constexpr int kBlock = 256;          // threads per block of the streaming kernels
constexpr unsigned char kVoid = 1, kSolid = 2;   // passive mask values (topo.h; reading R27)
constexpr int kMaxGridBlocks = 148 * 16;

// ---------------------------------------------------------------------------
// Deterministic grid reduction: block partials -> last block sums them in
// index order.  Returns true in every thread of the last block; `out[k]`
// (shared) then holds the grid totals.
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ void warp_sum(double (&v)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

__device__ __forceinline__ int flat_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
__device__ __forceinline__ int flat_nthreads() { return blockDim.x * blockDim.y * blockDim.z; }
__device__ __forceinline__ unsigned flat_bid() { return blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); }
__device__ __forceinline__ unsigned flat_nblocks() { return gridDim.x * gridDim.y * gridDim.z; }

template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double (*sh)[32]) {
  const int tid = flat_tid();
  const int lane = tid & 31, wid = tid >> 5, nw = flat_nthreads() >> 5;
  warp_sum<K>(v);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k][wid] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = (lane < nw) ? sh[k][lane] : 0.0;
  warp_sum<K>(v);   // every warp now holds the block total
}

// Max-reduction variant for a single value.
__device__ __forceinline__ double block_max(double v, double* sh) {
  const int tid = flat_tid();
  const int lane = tid & 31, wid = tid >> 5, nw = flat_nthreads() >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  v = (lane < nw) ? sh[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic grid reduction over a 1-3D grid of 1-3D blocks (blocks are a
// multiple of 32 threads).  `partials` holds K*nblocks doubles; `counter`
// must be 0 on entry and is reset by the last block.  The last KMAX of the K
// values are max-reduced, the others summed.  Returns true in every thread of
// the last block; `out_sh[k]` (shared) then holds the totals.
template <int K, int KMAX = 0>
__device__ bool grid_reduce(double (&v)[K], double* partials, unsigned int* counter,
                            double* out_sh) {
  __shared__ double sh[K > 0 ? K : 1][32];
  __shared__ bool am_last;
  const int tid = flat_tid(), nth = flat_nthreads();
  const unsigned bid = flat_bid(), nb = flat_nblocks();
  double vs[K];
#pragma unroll
  for (int k = 0; k < K; ++k) vs[k] = v[k];
  {
    double t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = (k < K - KMAX) ? vs[k] : 0.0;
    block_sum<K>(t, sh);
#pragma unroll
    for (int k = 0; k < K - KMAX; ++k) vs[k] = t[k];
  }
#pragma unroll
  for (int k = K - KMAX; k < K; ++k) vs[k] = block_max(vs[k], &sh[0][0]);
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) partials[(size_t)k * nb + bid] = vs[k];
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    am_last = (prev == nb - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  // each thread folds its partials with 4 independent accumulators so the L2
  // loads are in flight together (a dependent chain of ~10 L2 round trips per
  // value otherwise dominates the tail of short kernels); fixed order
  double t[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool mx = k >= K - KMAX;
    const double id = mx ? -1.0e300 : 0.0;
    double a4[4] = {id, id, id, id};
    for (unsigned b = tid; b < nb; b += 4 * nth) {
      double pv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned bj = b + j * nth;
        pv[j] = bj < nb ? __ldcg(&partials[(size_t)k * nb + bj]) : id;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) a4[j] = mx ? fmax(a4[j], pv[j]) : a4[j] + pv[j];
    }
    t[k] = mx ? fmax(fmax(a4[0], a4[1]), fmax(a4[2], a4[3])) : (a4[0] + a4[1]) + (a4[2] + a4[3]);
  }
  {
    double s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = (k < K - KMAX) ? t[k] : 0.0;
    block_sum<K>(s, sh);
#pragma unroll
    for (int k = 0; k < K - KMAX; ++k) t[k] = s[k];
  }
#pragma unroll
  for (int k = K - KMAX; k < K; ++k) t[k] = block_max(t[k], &sh[0][0]);
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) out_sh[k] = t[k];
    *counter = 0u;
  }
  __syncthreads();
  return true;
}

}  // namespace topo
