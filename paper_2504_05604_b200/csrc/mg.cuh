// Geometric multigrid preconditioner kernels (DESIGN.md
// readings M1-M6).  fp64, deterministic (every output written by one thread,
// fixed summation order; no atomics).
//
// Level 0 is the fine slab (W = 1, layout of common.cuh); levels l >= 1 use the
// same padded node layout: node (ix,iy,iz) at ((ix+1)*NZ + iz+1)*NY + iy+1,
// components SoA with stride ncomp, zero pads / ghost planes.  Element
// matrices of stored levels are SoA: K[(r*24 + s) * nel + e], e = (ex*nz +
// ez)*ny + ey, r,s local DOFs in SPEC S:45 corner order.
//
// Transfer (M2): P = trilinear interpolation, per axis fine node 2j <- coarse j,
// 2j+1 <- (j, j+1) with weights 1/2; restriction = P^T.  Coarse operators
// (M3): Galerkin P^T K P.  Smoother (M5): damped Jacobi.  Coarsest (M6):
// explicit inverse by Gauss-Jordan (SPD, no pivoting), applied as a dense
// matvec.
#pragma once
#include "common.cuh"
#include "matvec_wht.cuh"

namespace topo {

struct LvGeo {
  int nx, ny, nz;         // elements per axis
  int NY;                 // y pitch (nodes)
  long long nplane;       // NY * NZ
  long long ncomp;        // component stride
  // node planes [xa, xb] a launch computes (distributed levels, x-slabs: a rank's
  // owned planes; default: all, xb = -1 -> nx).  nodes() counts the range and
  // lv_decode offsets into it, so every node-parallel kernel is range-aware;
  // the layout (n(), ncomp, nel()) stays the whole level's.
  int xa = 0, xb = -1;
  __host__ __device__ long long n(int ix, int iy, int iz) const {
    return (long long)(ix + 1) * nplane + (long long)(iz + 1) * NY + (iy + 1);
  }
  __host__ __device__ int xlast() const { return xb < 0 ? nx : xb; }
  __host__ __device__ bool full() const { return xa == 0 && xlast() == nx; }
  __host__ __device__ long long nodes() const { return (long long)(xlast() - xa + 1) * (ny + 1) * (nz + 1); }
  __host__ __device__ long long nel() const { return (long long)nx * ny * nz; }
  // element planes adjacent to the node range: [max(xa - 1, 0), min(xlast, nx - 1)]
  __host__ __device__ long long el_lo() const { return (long long)(xa > 0 ? xa - 1 : 0) * ny * nz; }
  __host__ __device__ long long el_hi() const { return (long long)(xlast() < nx ? xlast() + 1 : nx) * ny * nz; }
  // per-component index range of the node planes (the whole component, pads
  // included, for the full range)
  __host__ __device__ long long v_lo() const { return full() ? 0 : (long long)(xa + 1) * nplane; }
  __host__ __device__ long long v_hi() const { return full() ? ncomp : (long long)(xlast() + 2) * nplane; }
};

// node k of the (nx+1)(ny+1)(nz+1) enumeration (of the range [xa, xb]), iy
// fastest (coalesced); 32-bit arithmetic (init validates node counts < 2^31)
__device__ __forceinline__ void lv_decode(const LvGeo& L, long long k, int& ix, int& iy, int& iz) {
  const unsigned kk = (unsigned)k, ny1 = (unsigned)(L.ny + 1), nz1 = (unsigned)(L.nz + 1);
  const unsigned t = kk / ny1;
  iy = (int)(kk - t * ny1);
  const unsigned u = t / nz1;
  iz = (int)(t - u * nz1);
  ix = (int)u + L.xa;
}
// element e of a vector-range loop over 3 components: index of the k-th entry
__device__ __forceinline__ long long lv_vidx(const LvGeo& L, long long k) {
  const long long w = L.v_hi() - L.v_lo();
  const long long c = k / w;
  return c * L.ncomp + L.v_lo() + (k - c * w);
}

__constant__ double c_mg_diag8[8 * 24];       // diag of M_c (level-1 Galerkin from fine E)
__constant__ signed char c_mg_nzA[8][8][8];   // child c, parent corner R -> child corners A with w != 0
__constant__ double c_mg_nzW[8][8][8];
__constant__ int c_mg_nzN[8][8];
__constant__ unsigned short c_mg_upair[300];  // upper triangle (r <= s) of a 24x24 element matrix: r*24+s

__host__ __device__ constexpr int mg_lidx(int a, int b, int c) { return 4 * c + (b ? (a ? 2 : 3) : (a ? 1 : 0)); }
__device__ __forceinline__ int corner_dx(int a) { return (a == 1 || a == 2 || a == 5 || a == 6) ? 1 : 0; }
__device__ __forceinline__ int corner_dy(int a) { return (a == 2 || a == 3 || a == 6 || a == 7) ? 1 : 0; }
__device__ __forceinline__ int corner_dz(int a) { return a >= 4 ? 1 : 0; }

#define MG_GATE(st) \
  if ((st) && (st)->done) return;

// ---------------------------------------------------------------------------
// Restriction  bC = mask_C( P^T mask_F(v) ),  v = bF - qF (kResid) or bF.
// Thread per coarse node; gathers the 3x3x3 fine neighbourhood of node 2j.
// ---------------------------------------------------------------------------
template <bool kResid, typename TF, typename TC>
__global__ void __launch_bounds__(kBlock)
k_mg_restrict(LvGeo F, LvGeo Cg, const TF* __restrict__ bF, const TF* __restrict__ qF,
              const uint8_t* __restrict__ fixF, const uint8_t* __restrict__ fixC, TC* __restrict__ bC,
              const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  const long long tot = Cg.nodes();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int jx, jy, jz;
    lv_decode(Cg, k, jx, jy, jz);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int dz = -1; dz <= 1; ++dz) {
      const int iz = 2 * jz + dz;
      if (iz < 0 || iz > F.nz) continue;
      const double wz = dz ? 0.5 : 1.0;
      for (int dx = -1; dx <= 1; ++dx) {
        const int ix = 2 * jx + dx;
        if (ix < 0 || ix > F.nx) continue;
        const double wxz = wz * (dx ? 0.5 : 1.0);
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
          const int iy = 2 * jy + dy;
          if (iy < 0 || iy > F.ny) continue;
          const double w = wxz * (dy ? 0.5 : 1.0);
          const long long i = F.n(ix, iy, iz);
          const uint8_t fm = fixF[i];
          double v0 = (double)bF[i], v1 = (double)bF[i + F.ncomp], v2 = (double)bF[i + 2 * F.ncomp];
          if (kResid) {
            v0 -= qF[i];
            v1 -= qF[i + F.ncomp];
            v2 -= qF[i + 2 * F.ncomp];
          }
          if (!(fm & 1)) s0 = fma(w, v0, s0);
          if (!(fm & 2)) s1 = fma(w, v1, s1);
          if (!(fm & 4)) s2 = fma(w, v2, s2);
        }
      }
    }
    const long long j = Cg.n(jx, jy, jz);
    const uint8_t fc = fixC[j];
    bC[j] = (TC)((fc & 1) ? 0.0 : s0);
    bC[j + Cg.ncomp] = (TC)((fc & 2) ? 0.0 : s1);
    bC[j + 2 * Cg.ncomp] = (TC)((fc & 4) ? 0.0 : s2);
  }
}

// Level-0 restriction of a masked residual (the pre-smoothing matvec's
// epilogue output), x-marching: thread per coarse (jy, jz) column and x-chunk;
// each fine plane is restricted in y-z once (9 gathers, coalesced in y) and
// shared by the two coarse planes it feeds (weights 1/2, 1, 1/2 along x), so
// the fine vector streams through HBM once.  Same sums as k_mg_restrict<false>
// (fp64, fixed order) up to the order of the x-terms.
//
// x-slabs (W > 1): res holds the fine planes [xa, xb) (global x; local plane 0
// at global x0) of one slab; planes outside contribute 0, the coarse planes
// j0 .. j0 + gridDim.y * cx_chunk - 1 that these planes reach are written, and
// with `accum` added to bC (zeroed first), so the sum over slabs -- in slab
// order (loopback) or by an allreduce (NCCL) -- is the restriction of the whole
// residual.  Single slab: x0 = 0, [xa, xb) = [0, nx], j0 = 0, accum = 0.
template <typename TF, typename TC>
__global__ void __launch_bounds__(128)
k_mg_restrict0(LvGeo F, LvGeo Cg, int cx_chunk, const TF* __restrict__ res, const uint8_t* __restrict__ fixC,
               TC* __restrict__ bC, const DevState* st, int x0, int xa, int xb, int j0, int jend, int accum) {
  pdl_enter();
  MG_GATE(st);
  const unsigned col = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned ny1 = Cg.ny + 1;
  if (col >= ny1 * (unsigned)(Cg.nz + 1)) return;
  const int jy = (int)(col % ny1), jz = (int)(col / ny1);
  const int ja = j0 + blockIdx.y * cx_chunk, jb = min(ja + cx_chunk, jend);
  if (ja >= jb) return;
  auto gyz = [&](int i, double g[3]) {     // y-z restriction of fine plane i at (jy, jz)
    g[0] = g[1] = g[2] = 0.0;
    if (i < xa || i >= xb) return;
    i -= x0;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
      const int iz = 2 * jz + dz;
      if (iz < 0 || iz > F.nz) continue;
      const double wz = dz ? 0.5 : 1.0;
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy) {
        const int iy = 2 * jy + dy;
        if (iy < 0 || iy > F.ny) continue;
        const double w = wz * (dy ? 0.5 : 1.0);
        const long long n = F.n(i, iy, iz);
        g[0] = fma(w, (double)res[n], g[0]);
        g[1] = fma(w, (double)res[n + F.ncomp], g[1]);
        g[2] = fma(w, (double)res[n + 2 * F.ncomp], g[2]);
      }
    }
  };
  double gp[3];
  gyz(2 * ja - 1, gp);
  for (int jx = ja; jx < jb; ++jx) {
    double ge[3], go[3];
    gyz(2 * jx, ge);
    gyz(2 * jx + 1, go);
    const long long j = Cg.n(jx, jy, jz);
    const uint8_t fc = fixC[j];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = fma(0.5, gp[c], fma(0.5, go[c], ge[c]));
      const long long o = j + c * Cg.ncomp;
      if (accum) {
        if (!((fc >> c) & 1)) bC[o] = (TC)((double)bC[o] + v);
      } else {
        bC[o] = (TC)(((fc >> c) & 1) ? 0.0 : v);
      }
      gp[c] = go[c];
    }
  }
}

// ---------------------------------------------------------------------------
// Prolongation  xF (+)= mask_F( P eC ).  Thread per fine node (<= 8 sources).
// ---------------------------------------------------------------------------
// (xin != nullptr: out of place, xF = xin + P eC)
template <bool kAdd, typename TC, typename TF>
__global__ void __launch_bounds__(kBlock)
k_mg_prolong(LvGeo F, LvGeo Cg, const TC* __restrict__ eC, const uint8_t* __restrict__ fixF,
             TF* __restrict__ xF, const DevState* st, const TF* __restrict__ xin = nullptr) {
  pdl_enter();
  MG_GATE(st);
  const long long tot = F.nodes();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(F, k, ix, iy, iz);
    const int jx = ix >> 1, jy = iy >> 1, jz = iz >> 1;
    const int nx = (ix & 1) + 1, ny = (iy & 1) + 1, nz = (iz & 1) + 1;
    const double w = (nx == 2 ? 0.5 : 1.0) * (ny == 2 ? 0.5 : 1.0) * (nz == 2 ? 0.5 : 1.0);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int a = 0; a < nz; ++a)
      for (int b = 0; b < nx; ++b)
        for (int c = 0; c < ny; ++c) {
          const long long j = Cg.n(jx + b, jy + c, jz + a);
          s0 += (double)eC[j];
          s1 += (double)eC[j + Cg.ncomp];
          s2 += (double)eC[j + 2 * Cg.ncomp];
        }
    const long long i = F.n(ix, iy, iz);
    const uint8_t fm = fixF[i];
    const double v[3] = {(fm & 1) ? 0.0 : w * s0, (fm & 2) ? 0.0 : w * s1, (fm & 4) ? 0.0 : w * s2};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long o = i + c * F.ncomp;
      xF[o] = (TF)(kAdd ? (double)(xin ? xin[o] : xF[o]) + v[c] : v[c]);
    }
  }
}

// Level 0 after the coarse correction (nu = 1): z = mask(w D^-1 r + P x1).  The
// first sweep z0 = w D^-1 r is recomputed from r instead of being stored by the
// pre-smoothing matvec (reads r and D^-1: 32 B/node instead of a z round trip).
// x-marching: thread per fine (iy, iz) column and x-chunk; the y-z
// interpolation of a coarse plane is formed once and used by the 2-3 fine planes
// that lie next to it; fine streams are coalesced in y.
// x-slabs: the fine planes [pa, pb) (global x; a slab's owned planes plus its
// ghost planes, local plane 0 at global x0) are written; chunks start at the even
// plane pa & ~1.  Single slab: x0 = 0, [pa, pb) = [0, nx].
// TZo: type of z (float with mg_fp32: the post-smoothing matvec rounds its
// input to the fp32 operator's precision anyway, so storing z in fp32 changes
// no result and halves its write and its TMA read).
template <typename TC, typename TZo = double, typename TR = double>
__global__ void __launch_bounds__(128)
k_mg_prolong0(LvGeo F, LvGeo Cg, int fx_chunk, const TR* __restrict__ r, const double* __restrict__ invd,
              const double* __restrict__ omp, const TC* __restrict__ eC, const uint8_t* __restrict__ fixF,
              TZo* __restrict__ z, const DevState* st, int x0, int pa, int pb) {
  pdl_enter();
  MG_GATE(st);
  const unsigned col = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned ny1 = F.ny + 1;
  if (col >= ny1 * (unsigned)(F.nz + 1)) return;
  const int iy = (int)(col % ny1), iz = (int)(col / ny1);
  const int ia = (pa & ~1) + blockIdx.y * fx_chunk, ib = min(ia + fx_chunk, pb);
  if (ia >= ib) return;
  const double omega = *omp;
  const int jy = iy >> 1, jz = iz >> 1, oy = iy & 1, oz = iz & 1;
  const double wy1 = oy ? 0.5 : 0.0, wy0 = 1.0 - wy1, wz1 = oz ? 0.5 : 0.0, wz0 = 1.0 - wz1;
  auto gyz = [&](int cx, double g[3]) {   // y-z interpolation of coarse plane cx at (iy, iz)
    const long long a = Cg.n(cx, jy, jz);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const TC* e = eC + a + c * Cg.ncomp;
      g[c] = fma(wz0, fma(wy0, (double)e[0], wy1 * (double)e[oy]),
                 wz1 * fma(wy0, (double)e[oz * Cg.NY], wy1 * (double)e[oz * Cg.NY + oy]));
    }
  };
  // planes in (even, odd) pairs: both read coarse plane c = i/2, the odd one also
  // c+1; all loads of a pair are issued before its stores (two planes in flight)
  double g0[3], g1[3];
  gyz(ia >> 1, g0);
  for (int i = ia; i < ib; i += 2) {
    const int c = i >> 1;
    const bool even_ok = i >= pa;             // only the first pair of a slab can start below pa
    const bool odd_ok = i + 1 < ib;
    gyz(c + 1, g1);
    const long long n0 = F.n(i - x0, iy, iz), n1 = n0 + F.nplane;
    double r0[3], r1[3];
    const uint8_t f0 = even_ok ? fixF[n0] : (uint8_t)7, f1 = odd_ok ? fixF[n1] : (uint8_t)7;
    const double d0 = even_ok ? invd[n0] : 0.0, d1 = odd_ok ? invd[n1] : 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      r0[k] = even_ok ? (double)r[n0 + k * F.ncomp] : 0.0;
      r1[k] = odd_ok ? (double)r[n1 + k * F.ncomp] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (even_ok) z[n0 + k * F.ncomp] = (TZo)(((f0 >> k) & 1) ? 0.0 : fma(omega * d0, r0[k], g0[k]));
      if (odd_ok) z[n1 + k * F.ncomp] = (TZo)(((f1 >> k) & 1) ? 0.0 : fma(omega * d1, r1[k], 0.5 * (g0[k] + g1[k])));
      g0[k] = g1[k];
    }
  }
}

// ---------------------------------------------------------------------------
// Damped Jacobi (M5) on one level.  q = A x comes from the operator kernel
// (unmasked at level 0, masked at coarse levels; masking happens here).
// The weight w_l = theta / lam_l lives in device memory (set by the setup's
// power steps, k_mg_rayleigh).
//   MODE 0: x = w D^-1 b                      (first sweep from x = 0)
//   MODE 1: x = x + w D^-1 (b - q)
//   MODE 2: MODE 1 and rho = b . x_new (PCG: b = r, x = z = V(r)); the last
//           block sets beta = rho / rho_old (0 on a fresh start), rz = rho.
// kNodeD: D^-1 is one scalar per node (level 0: KE_ii constant), else per DOF.
// ---------------------------------------------------------------------------
template <int MODE, bool kNodeD, typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_jacobi(LvGeo L, const T* __restrict__ b, const T* __restrict__ q,
            const T* __restrict__ invd, const uint8_t* __restrict__ fix, const double* __restrict__ omp,
            T* __restrict__ x, DevState* st, int gate, double* partials, unsigned int* counter) {
  pdl_enter();
  if (gate && st->done) return;
  const double omega = *omp;
  const long long tot = L.nodes();
  double dot = 0.0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    const long long i = L.n(ix, iy, iz);
    const uint8_t fm = fix[i];
    const double dn = kNodeD ? (double)invd[i] : 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long o = i + c * L.ncomp;
      const double d = kNodeD ? dn : (double)invd[o];
      const double bv = (double)b[o];
      double xn;
      if ((fm >> c) & 1) xn = 0.0;
      else if (MODE == 0) xn = omega * d * bv;
      else xn = fma(omega * d, bv - (double)q[o], (double)x[o]);
      x[o] = (T)xn;
      if (MODE == 2) dot = fma(bv, xn, dot);
    }
  }
  if (MODE == 2) {
    __shared__ double tot_sh[1];
    double v[1] = {dot};
    if (grid_reduce<1>(v, partials, counter, tot_sh) && threadIdx.x == 0) {
      const double rho = tot_sh[0];
      if (!(rho > 0.0) || !isfinite(rho)) {
        st->status = 3;
        st->done = 1;
      } else {
        st->beta = st->fresh ? 0.0 : rho / st->rz;
        st->rz = rho;
      }
    }
  }
}

// Small coarse levels: the same restriction with a WARP per coarse node (lane
// d < 27 takes fine neighbour d of the 3x3x3 box), partial sums combined by a
// fixed shuffle tree -- the thread-per-node loop is a 27-step latency chain
// with a handful of blocks on the deep levels (9-11 us per launch).
template <bool kResid, typename TF, typename TC>
__global__ void __launch_bounds__(kBlock)
k_mg_restrict_w(LvGeo F, LvGeo Cg, const TF* __restrict__ bF, const TF* __restrict__ qF,
                const uint8_t* __restrict__ fixF, const uint8_t* __restrict__ fixC, TC* __restrict__ bC,
                const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  const long long tot = Cg.nodes();
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int dx = lane < 27 ? lane / 9 - 1 : 0, dz = lane < 27 ? (lane / 3) % 3 - 1 : 0, dy = lane < 27 ? lane % 3 - 1 : 0;
  const double w = lane < 27 ? (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0) : 0.0;
  for (long long k = w0; k < tot; k += nw) {
    int jx, jy, jz;
    lv_decode(Cg, k, jx, jy, jz);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    const int ix = 2 * jx + dx, iy = 2 * jy + dy, iz = 2 * jz + dz;
    if (lane < 27 && ix >= 0 && ix <= F.nx && iy >= 0 && iy <= F.ny && iz >= 0 && iz <= F.nz) {
      const long long i = F.n(ix, iy, iz);
      const uint8_t fm = fixF[i];
      double v0 = (double)bF[i], v1 = (double)bF[i + F.ncomp], v2 = (double)bF[i + 2 * F.ncomp];
      if (kResid) {
        v0 -= qF[i];
        v1 -= qF[i + F.ncomp];
        v2 -= qF[i + 2 * F.ncomp];
      }
      s0 = (fm & 1) ? 0.0 : w * v0;
      s1 = (fm & 2) ? 0.0 : w * v1;
      s2 = (fm & 4) ? 0.0 : w * v2;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      const long long j = Cg.n(jx, jy, jz);
      const uint8_t fc = fixC[j];
      bC[j] = (TC)((fc & 1) ? 0.0 : s0);
      bC[j + Cg.ncomp] = (TC)((fc & 2) ? 0.0 : s1);
      bC[j + 2 * Cg.ncomp] = (TC)((fc & 4) ? 0.0 : s2);
    }
  }
}

// ---------------------------------------------------------------------------
// K-cycle (reading M8; Notay & Vassilevski 2008): a coarse level l is solved by
// two flexible-CG steps preconditioned by its own cycle B_l:
//   x1 = B(b); t = A x1; rho1 = x1.t, a1 = x1.b; kx = x1, kv = t     (k_kc_dot1)
//   b <- r2 = b - (a1/rho1) kv                                         (k_kc_r2)
//   x2 = B(r2); t = A x2; g = x2.kv, bb = x2.t, a2 = x2.r2             (k_kc_dot2)
//   rho2 = bb - g^2/rho1;  c2 = a2/rho2, c1 = a1/rho1 - g c2/rho1 (rho2 <= 0: c2 = 0)
//   x = c1 kx + c2 x2                                                  (k_kc_combine)
// The vectors are whole padded level buffers (pads and fixed DOFs hold 0 in x,
// t and b), reduced in fp64 in a fixed order.  kc[0..3] = rho1, a1, c1, c2.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_kc_dot1(LvGeo L, const T* __restrict__ x, const T* __restrict__ t, const T* __restrict__ b,
          T* __restrict__ kx, T* __restrict__ kv, double* __restrict__ kc, const DevState* gst,
          double* partials, unsigned int* counter, DevState* slab_out = nullptr) {
  pdl_enter();
  MG_GATE(gst);
  double xt = 0.0, xb = 0.0;
  const long long n = 3 * (L.v_hi() - L.v_lo());
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const long long i = lv_vidx(L, k);
    const T xv = x[i], tv = t[i];
    kx[i] = xv;
    kv[i] = tv;
    xt = fma((double)xv, (double)tv, xt);
    xb = fma((double)xv, (double)b[i], xb);
  }
  __shared__ double tot[2];
  double v[2] = {xt, xb};
  if (grid_reduce<2>(v, partials, counter, tot) && threadIdx.x == 0) {
    if (slab_out) {   // x-slab partial: allreduced, then k_kc_finish1
      slab_out->sums[0] = tot[0];
      slab_out->sums[1] = tot[1];
      return;
    }
    kc[0] = tot[0];
    kc[1] = tot[1];
  }
}
__global__ void k_kc_finish1(const DevState* st, double* __restrict__ kc, const DevState* gst) {
  pdl_enter();
  MG_GATE(gst);
  kc[0] = st->sums[0];
  kc[1] = st->sums[1];
}
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_kc_r2(LvGeo L, T* __restrict__ b, const T* __restrict__ kv, const double* __restrict__ kc, const DevState* gst) {
  pdl_enter();
  MG_GATE(gst);
  const double s = kc[0] > 0.0 ? kc[1] / kc[0] : 0.0;
  const long long n = 3 * (L.v_hi() - L.v_lo());
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const long long i = lv_vidx(L, k);
    b[i] = (T)fma(-s, (double)kv[i], (double)b[i]);
  }
}
__device__ __forceinline__ void kc_coeffs(double* kc, double g, double bb, double a2) {
  const double rho1 = kc[0], a1 = kc[1];
  if (!(rho1 > 0.0) || !isfinite(rho1)) {     // B_l(b) = 0 (b = 0): no correction
    kc[2] = 0.0;
    kc[3] = 0.0;
    return;
  }
  const double rho2 = bb - g * g / rho1;
  const double c2 = (rho2 > 0.0 && isfinite(rho2)) ? a2 / rho2 : 0.0;
  kc[2] = a1 / rho1 - g * c2 / rho1;
  kc[3] = c2;
}
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_kc_dot2(LvGeo L, const T* __restrict__ x, const T* __restrict__ t, const T* __restrict__ b,
          const T* __restrict__ kv, double* __restrict__ kc, const DevState* gst, double* partials,
          unsigned int* counter, DevState* slab_out = nullptr) {
  pdl_enter();
  MG_GATE(gst);
  double g = 0.0, bb = 0.0, a2 = 0.0;
  const long long n = 3 * (L.v_hi() - L.v_lo());
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const long long i = lv_vidx(L, k);
    const double xv = (double)x[i];
    g = fma(xv, (double)kv[i], g);
    bb = fma(xv, (double)t[i], bb);
    a2 = fma(xv, (double)b[i], a2);
  }
  __shared__ double tot[3];
  double v[3] = {g, bb, a2};
  if (grid_reduce<3>(v, partials, counter, tot) && threadIdx.x == 0) {
    if (slab_out) {
      slab_out->sums[0] = tot[0];
      slab_out->sums[1] = tot[1];
      slab_out->sums[2] = tot[2];
      return;
    }
    kc_coeffs(kc, tot[0], tot[1], tot[2]);
  }
}
__global__ void k_kc_finish2(const DevState* st, double* __restrict__ kc, const DevState* gst) {
  pdl_enter();
  MG_GATE(gst);
  kc_coeffs(kc, st->sums[0], st->sums[1], st->sums[2]);
}
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_kc_combine(LvGeo L, T* __restrict__ x, const T* __restrict__ kx, const double* __restrict__ kc,
             const DevState* gst) {
  pdl_enter();
  MG_GATE(gst);
  const double c1 = kc[2], c2 = kc[3];
  const long long n = 3 * (L.v_hi() - L.v_lo());
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const long long i = lv_vidx(L, k);
    x[i] = (T)fma(c1, (double)kx[i], c2 * (double)x[i]);
  }
}

// ---------------------------------------------------------------------------
// Smoother weights (M5): power steps v <- D^-1 A v from a fixed start vector,
// then w_l = theta (v^T D v) / (v^T A v) = theta / lam_l.
// Start vector: DOF k of the level's external numbering (3 n + c) gets
// 2 u - 1, u = (splitmix64(k) >> 11) 2^-53; 0 on fixed DOFs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double mg_hash_unit(unsigned long long k) {
  unsigned long long z = k + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
}

// Node planes [xa, xb] (global x) of a vector stored with local plane 0 at
// global x0 (a slab: x0 = ex0, the ghost planes included; one level: x0 = 0);
// the hash uses global coordinates (nxg = global element count in x), so every
// slab produces the same entries as the single-slab vector.
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_start_vec(LvGeo L, int x0, int xa, int xb, int nxg, const uint8_t* __restrict__ fix, T* __restrict__ v) {
  pdl_enter();
  const long long tot = (long long)(xb - xa + 1) * (L.ny + 1) * (L.nz + 1);
  const LvGeo D{xb - xa, L.ny, L.nz, L.NY, L.nplane, L.ncomp};   // decode range only
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(D, k, ix, iy, iz);
    ix += xa;
    const long long i = L.n(ix - x0, iy, iz);
    const unsigned long long ext = ((unsigned long long)iz * (nxg + 1) + ix) * (L.ny + 1) + iy;
    const uint8_t fm = fix[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) v[i + c * L.ncomp] = (T)(((fm >> c) & 1) ? 0.0 : mg_hash_unit(3 * ext + c));
  }
}

constexpr int kMgScaleOff = 17;   // mg_om layout: [0,16) weights, [16] = 1.0, [17,33) power-vector scales

template <bool kNodeD, typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_rayleigh(LvGeo L, const T* __restrict__ v, const T* __restrict__ t, const T* __restrict__ invd,
              const uint8_t* __restrict__ fix, double theta, double* __restrict__ om_out,
              double* partials, unsigned int* counter, DevState* st = nullptr) {
  pdl_enter();
  const long long tot = L.nodes();
  double vt = 0.0, vdv = 0.0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    const long long i = L.n(ix, iy, iz);
    const uint8_t fm = fix[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if ((fm >> c) & 1) continue;
      const long long o = i + c * L.ncomp;
      const double vv = (double)v[o];
      vt = fma(vv, (double)t[o], vt);
      vdv = fma(vv * vv, 1.0 / (double)(kNodeD ? invd[i] : invd[o]), vdv);
    }
  }
  __shared__ double tot_sh[2];
  double r[2] = {vt, vdv};
  if (grid_reduce<2>(r, partials, counter, tot_sh) && threadIdx.x == 0) {
    if (st) {   // slab partial: (v.t, v.Dv) allreduced, then k_mg_rayleigh_finish
      st->sums[0] = tot_sh[0];
      st->sums[1] = tot_sh[1];
      return;
    }
    om_out[0] = theta * tot_sh[1] / tot_sh[0];
    // 1 / ||v||_D: the vector kept for the next design's warm start is stored
    // normalised (unnormalised, it grows by ~lam per power step and overflows
    // after a few dozen designs in fp32, a few hundred in fp64)
    om_out[kMgScaleOff] = tot_sh[1] > 0.0 ? 1.0 / sqrt(tot_sh[1]) : 1.0;
  }
}

__global__ void k_mg_rayleigh_finish(const DevState* st, double theta, double* __restrict__ om_out) {
  pdl_enter();
  om_out[0] = theta * st->sums[1] / st->sums[0];
  om_out[kMgScaleOff] = st->sums[1] > 0.0 ? 1.0 / sqrt(st->sums[1]) : 1.0;
}

// dst = s * src (s on the device: the power vector's 1/||v||_D)
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_scale_copy(const T* __restrict__ src, T* __restrict__ dst, long long n, const double* __restrict__ sp) {
  pdl_enter();
  const double sc = *sp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = (T)(sc * (double)src[i]);
}

// ---------------------------------------------------------------------------
// Stored-level operator q = mask(A x) (node-centric gather over the <= 8
// elements of each node; each element matrix is read once in total).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_apply_asm(LvGeo L, const double* __restrict__ K, const T* __restrict__ x,
               const uint8_t* __restrict__ fix, T* __restrict__ q, const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  const long long tot = L.nodes(), nel = L.nel();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int dz = 0; dz < 2; ++dz)
      for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy) {
          const int ex = ix - 1 + dx, ey = iy - 1 + dy, ez = iz - 1 + dz;
          if (ex < 0 || ex >= L.nx || ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
          const long long e = ((long long)ex * L.nz + ez) * L.ny + ey;
          const int a = mg_lidx(1 - dx, 1 - dy, 1 - dz);
          double xe[24];
#pragma unroll
          for (int bb = 0; bb < 8; ++bb) {
            const long long n = L.n(ex + corner_dx(bb), ey + corner_dy(bb), ez + corner_dz(bb));
#pragma unroll
            for (int c = 0; c < 3; ++c) xe[3 * bb + c] = (double)x[n + c * L.ncomp];
          }
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const double* row = K + (long long)((3 * a + i) * 24) * nel + e;
            double s = 0.0;
#pragma unroll
            for (int cc = 0; cc < 24; ++cc) s = fma(row[(long long)cc * nel], xe[cc], s);
            acc[i] += s;
          }
        }
    const long long i = L.n(ix, iy, iz);
    const uint8_t fm = fix[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) q[i + c * L.ncomp] = (T)(((fm >> c) & 1) ? 0.0 : acc[c]);
  }
}

// Inverse diagonal of a stored level (0 on fixed DOFs).
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_diag_asm(LvGeo L, const double* __restrict__ K, const uint8_t* __restrict__ fix, T* __restrict__ invd) {
  pdl_enter();
  const long long tot = L.nodes(), nel = L.nel();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int dz = 0; dz < 2; ++dz)
      for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy) {
          const int ex = ix - 1 + dx, ey = iy - 1 + dy, ez = iz - 1 + dz;
          if (ex < 0 || ex >= L.nx || ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
          const long long e = ((long long)ex * L.nz + ez) * L.ny + ey;
          const int a = mg_lidx(1 - dx, 1 - dy, 1 - dz);
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[c] += K[(long long)((3 * a + c) * 25) * nel + e];
        }
    const long long i = L.n(ix, iy, iz);
    const uint8_t fm = fix[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) invd[i + c * L.ncomp] = (T)(((fm >> c) & 1) ? 0.0 : 1.0 / acc[c]);
  }
}

// Inverse diagonal of level 1 straight from the fine moduli (level 1 applied
// matrix-free as P^T K P): diag = sum_e sum_c E_c diag(M_c).
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_diag_l1(Geo g, LvGeo L, const double* __restrict__ E, const uint8_t* __restrict__ fix,
             T* __restrict__ invd) {
  pdl_enter();
  const long long tot = L.nodes();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int dz = 0; dz < 2; ++dz)
      for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy) {
          const int ex = ix - 1 + dx, ey = iy - 1 + dy, ez = iz - 1 + dz;
          if (ex < 0 || ex >= L.nx || ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
          const int a = mg_lidx(1 - dx, 1 - dy, 1 - dz);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int fx = 2 * ex + (c & 1), fy = 2 * ey + ((c >> 1) & 1), fz = 2 * ez + (c >> 2);
            if (fx >= g.nelx || fy >= g.nely || fz >= g.nelz) continue;
            const double Ef = E[elem_idx(g, fx, fy, fz)];
#pragma unroll
            for (int i = 0; i < 3; ++i) acc[i] = fma(Ef, c_mg_diag8[24 * c + 3 * a + i], acc[i]);
          }
        }
    const long long i = L.n(ix, iy, iz);
    const uint8_t fm = fix[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) invd[i + c * L.ncomp] = (T)(((fm >> c) & 1) ? 0.0 : 1.0 / acc[c]);
  }
}

// ---------------------------------------------------------------------------
// Element matrices of level log2(S) straight from the fine moduli:
//   K_e[k] = sum_f E_f tab[f][k],  f = fx + S fy + S^2 fz over the S^3 fine
// elements of e (E = 0 outside the fine domain).  Thread per element; the
// table is staged through shared memory in chunks of kCh entries.
// ---------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(kBlock)
k_mg_asm_fine(Geo g, LvGeo L, const double* __restrict__ E, const double* __restrict__ tab,
              double* __restrict__ K) {
  pdl_enter();
  constexpr int NT = S * S * S, kCh = 32;
  __shared__ double tb[NT][kCh];
  const long long nel = L.nel();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double Ef[NT];
  if (e < nel) {
    const int ey = (int)(e % L.ny);
    const long long t = e / L.ny;
    const int ez = (int)(t % L.nz), ex = (int)(t / L.nz);
#pragma unroll
    for (int f = 0; f < NT; ++f) {
      const int fx = S * ex + f % S, fy = S * ey + (f / S) % S, fz = S * ez + f / (S * S);
      Ef[f] = (fx < g.nelx && fy < g.nely && fz < g.nelz) ? E[elem_idx(g, fx, fy, fz)] : 0.0;
    }
  }
  // symmetric: the 300 upper-triangle entries, each written to (r, s) and (s, r)
  for (int u0 = 0; u0 < 300; u0 += kCh) {
    __syncthreads();
    for (int t = threadIdx.x; t < NT * kCh; t += blockDim.x) {
      const int u = u0 + t % kCh;
      tb[t / kCh][t % kCh] = u < 300 ? tab[(t / kCh) * 576 + c_mg_upair[u]] : 0.0;
    }
    __syncthreads();
    if (e < nel) {
      for (int kk = 0; kk < kCh && u0 + kk < 300; ++kk) {
        double s = 0.0;
#pragma unroll
        for (int f = 0; f < NT; ++f) s = fma(Ef[f], tb[f][kk], s);
        const int rs = c_mg_upair[u0 + kk], r = rs / 24, c = rs % 24;
        K[(long long)rs * nel + e] = s;
        K[(long long)(c * 24 + r) * nel + e] = s;
      }
    }
  }
}

// Level 2 as a GEMM: K2[rs][e] = sum_f E_f(e) tab64[f][rs] (linear in the 64
// fine moduli of a level-2 element); this gathers Eg[e + nel * f] (column-major
// nel x 64) for cuBLAS DGEMM.  Child f = (fx, fy, fz) = (f % 4, (f / 4) % 4, f / 16)
// as in k_mg_asm_fine<4>; children outside the fine grid give 0.
__global__ void __launch_bounds__(kBlock)
k_mg_gather64(Geo g, LvGeo L, const double* __restrict__ E, double* __restrict__ Eg) {
  pdl_enter();
  const long long nel = L.nel(), tot = 64 * nel;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(t / nel);
    const long long e = t - (long long)f * nel;
    const int ey = (int)(e % L.ny);
    const long long r = e / L.ny;
    const int ez = (int)(r % L.nz), ex = (int)(r / L.nz);
    const int fx = 4 * ex + f % 4, fy = 4 * ey + (f / 4) % 4, fz = 4 * ez + f / 16;
    Eg[t] = (fx < g.nelx && fy < g.nely && fz < g.nelz) ? E[elem_idx(g, fx, fy, fz)] : 0.0;
  }
}

// Element matrices of level l+1 from the stored level l (Galerkin per child):
//   KC_e[3R+i][3S+j] = sum_c sum_{A,B} w[c][A][R] KF_child(c)[3A+i][3B+j] w[c][B][S]
// Same product, tiled for memory efficiency: a CTA owns 8 coarse elements
// consecutive in y (fixed ex, ez) and walks the 4 (cx, cz) child pairs; for each
// pair the 16 fine elements (cy = 0, 1 of each coarse element, consecutive in the
// fine y) are staged in shared memory, every entry read once and coalesced.
// Thread (e, s) builds column s = 3S + j of its coarse element:
//   v[(A,i)] = sum_{B} w[c][B][S] KF_c[(A,i),(B,j)],  KC[(R,i), s] += sum_A w[c][A][R] v[(A,i)].
constexpr int kGalTile = 8;
__global__ void __launch_bounds__(kGalTile * 24, 2)
k_mg_asm_galerkin_t(LvGeo F, const double* __restrict__ KF, LvGeo Cg, double* __restrict__ KC) {
  pdl_enter();
  extern __shared__ double sK[];                 // [576][2 * kGalTile]
  constexpr int NF = 2 * kGalTile;
  const int el = threadIdx.x, sc = threadIdx.y;  // coarse element in the tile, output column
  const int tid = sc * kGalTile + el, nth = kGalTile * 24;
  const int ey0 = blockIdx.x * kGalTile, ez = blockIdx.y, ex = blockIdx.z;
  const int ey = ey0 + el;
  const long long nelC = Cg.nel(), nelF = F.nel();
  const int S = sc / 3, j = sc % 3;
  double acc[24];
#pragma unroll
  for (int r = 0; r < 24; ++r) acc[r] = 0.0;
  for (int pr = 0; pr < 4; ++pr) {
    const int cx = pr & 1, cz = pr >> 1;
    const int fx = 2 * ex + cx, fz = 2 * ez + cz;
    const bool plane_ok = fx < F.nx && fz < F.nz;
    __syncthreads();
    if (plane_ok) {
      const long long fbase = ((long long)fx * F.nz + fz) * F.ny + 2 * ey0;
      for (int t = tid; t < 576 * NF; t += nth) {
        const int q = t / NF, f = t - q * NF;
        sK[t] = (2 * ey0 + f < F.ny) ? KF[(long long)q * nelF + fbase + f] : 0.0;
      }
    }
    __syncthreads();
    if (!plane_ok || ey >= Cg.ny) continue;
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      const int c = cx + 2 * cy + 4 * cz;
      const int f = 2 * el + cy;
      double v[24];
#pragma unroll
      for (int r = 0; r < 24; ++r) v[r] = 0.0;
      const int nb = c_mg_nzN[c][S];
      for (int ib = 0; ib < nb; ++ib) {
        const int B = c_mg_nzA[c][S][ib];
        const double wb = c_mg_nzW[c][S][ib];
#pragma unroll
        for (int r = 0; r < 24; ++r) v[r] = fma(wb, sK[(r * 24 + 3 * B + j) * NF + f], v[r]);
      }
      // acc += W_c^T v with w[c][A][R] = prod_d (R_d ? t_d : 1 - t_d), t_d = (c_d + A_d) / 2
      // (SPEC corner order: A_x = ((A + 1) >> 1) & 1, A_y = (A >> 1) & 1, A_z = A >> 2);
      // fully unrolled so v and acc stay in registers
      const int cd[3] = {cx, cy, cz};
#pragma unroll
      for (int A = 0; A < 8; ++A) {
        const int ad[3] = {((A + 1) >> 1) & 1, (A >> 1) & 1, A >> 2};
        double t[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) t[d] = 0.5 * (double)(cd[d] + ad[d]);
#pragma unroll
        for (int R = 0; R < 8; ++R) {
          const int rd[3] = {((R + 1) >> 1) & 1, (R >> 1) & 1, R >> 2};
          const double w = (rd[0] ? t[0] : 1.0 - t[0]) * (rd[1] ? t[1] : 1.0 - t[1]) * (rd[2] ? t[2] : 1.0 - t[2]);
#pragma unroll
          for (int i = 0; i < 3; ++i) acc[3 * R + i] = fma(w, v[3 * A + i], acc[3 * R + i]);
        }
      }
    }
  }
  if (ey >= Cg.ny) return;
  const long long e = ((long long)ex * Cg.nz + ez) * Cg.ny + ey;
#pragma unroll
  for (int r = 0; r < 24; ++r) KC[(long long)(r * 24 + sc) * nelC + e] = acc[r];
}

// ---------------------------------------------------------------------------
// Level 1 matrix-free: y = P^T K(E) P x, element by element in the Walsh
// domain.  With H the unnormalised +-1 transform of the 8 corners (natural
// index k = ax + 2 ay + 4 az, entry (-1)^{popcount(m & k)}) and KE = H^T B H
// (B block-diagonal, wht_block), the Galerkin element matrix of a coarse
// element is K1_e = H^T [ sum_c E_c T_c^T B T_c ] H, where T_c = H P_c H^-1
// is, per axis, [[1, s/2], [0, 1/2]] on (sum, difference) pairs (s = +1 for
// the lower child, -1 for the upper).  ~1650 flops per coarse element instead
// of a fine matvec on P x plus two transfers.  Two phases for determinism:
// phase 1 writes each element's 24 outputs, phase 2 sums them per node.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void fwht8(T v[8]) {
#pragma unroll
  for (int b = 1; b < 8; b <<= 1)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (!(k & b)) {
        const T u = v[k], w = v[k | b];
        v[k] = u + w;
        v[k | b] = u - w;
      }
}

constexpr int kL1Block = 128;
template <typename T> __device__ __forceinline__ const WhtKT<T>& wht1_const();
template <> __device__ __forceinline__ const WhtKT<double>& wht1_const<double>() { return c_wht1; }
template <> __device__ __forceinline__ const WhtKT<float>& wht1_const<float>() { return c_wht1f; }

#ifndef TOPO_L1_MINB
#define TOPO_L1_MINB 4   // fp32: 4 CTAs / SM at 128 registers, no spills (measured 0.08 ms less per MG-PCG iteration than 3)
#endif
// Level-1 element operator: W[c][k] = the corner values (natural corner index
// k = ax + 2 ay + 4 az, overwritten), Ech the 8 child moduli -> Yh[c][k] = the
// element's outputs at its corners (K1_e applied matrix-free, see above).
template <typename T>
__device__ __forceinline__ void l1_elem_core(T W[3][8], const T Ech[8], T Yh[3][8]) {
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) Yh[c][k] = T(0);
#pragma unroll
  for (int c = 0; c < 3; ++c) fwht8(W[c]);
  // T_c = Lambda^-1 T''_c with T''_c = [[1, s/2], [0, 1]] per axis, so
  // T_c^T B T_c = T''_c^T (Lambda^-1 B Lambda^-1) T''_c: one FMA per pair each way
  // and the rescaled block constants c_wht1.
  // fp32: children fully unrolled (static E index, no select chain); fp64 keeps
  // the loop rolled for register pressure.  A child outside the fine domain has
  // E = 0 and contributes exactly 0.
#pragma unroll (sizeof(T) == 4 ? 8 : 1)
  for (int ch = 0; ch < 8; ++ch) {
    T Ec = Ech[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) Ec = ch == k ? Ech[k] : Ec;   // register select (folds when unrolled)
    T P[3][8], Q[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m = 0; m < 8; ++m) P[c][m] = W[c][m];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const T hs = ((ch >> d) & 1) ? T(-0.5) : T(0.5);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int m = 0; m < 8; ++m)
          if (!((m >> d) & 1)) P[c][m] = fma(hs, P[c][m | (1 << d)], P[c][m]);
    }
    wht_block_k<T>(wht1_const<T>(), P, Ec, Q);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const T hs = ((ch >> d) & 1) ? T(-0.5) : T(0.5);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int m = 0; m < 8; ++m)
          if (!((m >> d) & 1)) Q[c][m | (1 << d)] = fma(hs, Q[c][m], Q[c][m | (1 << d)]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m = 0; m < 8; ++m) Yh[c][m] += Q[c][m];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) fwht8(Yh[c]);
}

template <typename T, typename TE = double>
__global__ void __launch_bounds__(kL1Block, (sizeof(T) == 4 ? TOPO_L1_MINB : 3))
k_mg_l1_elem(Geo g, LvGeo L, const TE* __restrict__ E, const T* __restrict__ x,
             T* __restrict__ Y, const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  const long long nel = L.nel(), ehi = L.el_hi();   // (x-slabs: the element planes next to the node range)
  for (long long e = L.el_lo() + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ehi;
       e += (long long)gridDim.x * blockDim.x) {
    const unsigned ee = (unsigned)e, ny = (unsigned)L.ny, nz = (unsigned)L.nz;
    const unsigned t = ee / ny, ey = ee - t * ny, ex = t / nz, ez = t - ex * nz;
    T W[3][8], Yh[3][8], Ech[8];
#pragma unroll
    for (int ch = 0; ch < 8; ++ch)     // child moduli first: independent loads off the compute chain
      Ech[ch] = (T)E[elem_idx(g, 2 * ex + (ch & 1), 2 * ey + ((ch >> 1) & 1), 2 * ez + (ch >> 2))];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long n = L.n(ex + (k & 1), ey + ((k >> 1) & 1), ez + (k >> 2));
#pragma unroll
      for (int c = 0; c < 3; ++c) W[c][k] = x[n + c * L.ncomp];
    }
    l1_elem_core<T>(W, Ech, Yh);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int k = 0; k < 8; ++k) Y[(long long)(3 * k + c) * nel + e] = Yh[c][k];
    }
  }
}


// Face-accumulating variant (TOPO_L1_FACE, default): a thread owns one (ey, ez)
// element column and walks kL1CX node planes of it along x; node plane x's
// 4 corners x 3 components are loaded once and shared by elements x - 1 and x,
// and the thread writes the x-complete FACE sums
//   F[x][j][c][col] = (element x-1's ax = 1 corner j) + (element x's ax = 0 corner j),
// j = ay + 2 az, col = ez ny + ey -- 12 values per node plane and column instead
// of 24 per element (half the bytes of the Y round trip), and the gather sums 4
// faces instead of 8 element corners.  The element before a chunk is recomputed
// (1 in kL1CX).  x-slab ranges: node planes [xa, xlast] only.
constexpr int kL1CX = 16;
#ifndef TOPO_L1F_MINB
#define TOPO_L1F_MINB 3
#endif
// kAsync (TOPO_L1F_ASYNC, default): the NEXT step's 12 node values and 8 child
// moduli travel global -> shared by per-thread cp.async (4 / 8 bytes, the thread's
// own slots, two buffers in turn) while this step's element arithmetic runs, so a
// warp no longer waits out the DRAM latency at the top of every step (ncu r02s:
// 38 % long-scoreboard stalls at 12 warps/SM).  Same values, same arithmetic.
template <int B>
__device__ __forceinline__ void cp_async_own(void* s, const void* gp) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sa), "l"(gp), "n"(B) : "memory");
}
template <typename T, typename TE = double, bool kAsync = false>
__global__ void __launch_bounds__(kL1Block, (sizeof(T) == 4 ? TOPO_L1F_MINB : 3))
k_mg_l1_face(Geo g, LvGeo L, const TE* __restrict__ E, const T* __restrict__ x, T* __restrict__ F,
             const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  __shared__ T sB[kAsync ? 2 : 1][kAsync ? 12 : 1][kAsync ? kL1Block : 1];
  __shared__ TE sE[kAsync ? 2 : 1][kAsync ? 8 : 1][kAsync ? kL1Block : 1];
  const int nx = L.nx, ny = L.ny;
  const long long ncol = (long long)L.ny * L.nz;
  const int plo = L.xa, phi = L.xlast() + 1;              // node planes [plo, phi)
  const int nchunk = (phi - plo + kL1CX - 1) / kL1CX;
  __shared__ T sA[12][kL1Block], sacc[12][kL1Block];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncol * nchunk;
       t += (long long)gridDim.x * blockDim.x) {
    const int chunk = (int)(t / ncol);
    const long long col = t - (long long)chunk * ncol;
    const int ez = (int)(col / ny), ey = (int)(col - (long long)ez * ny);
    const int p0 = plo + chunk * kL1CX, p1 = min(p0 + kL1CX, phi);
    // running pointers (advanced one plane per step) and 32-bit in-plane offsets
    const int NY = L.NY;
    const T* xp = x + L.n(p0 - 1, ey, ez);                   // node plane ex (corner j = 0)
    const int onp = (int)L.nplane;
    const long long ebase = elem_idx(g, 2 * (p0 - 1), 2 * ey, 2 * ez);
    const int eplane2 = (int)(2 * g.eplane), EY = g.EY;
    T* fp = F + (long long)(p0 - 1) * 12 * ncol + col;
    const long long fstep = 12 * ncol;
    // per-thread carries in shared memory (slot [c*4+j][thread]): the previous node
    // plane's corners and the running face sum -- kept out of the registers of the
    // element arithmetic
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        sacc[c * 4 + j][threadIdx.x] = T(0);
        sA[c * 4 + j][threadIdx.x] = p0 - 1 >= 0 ? xp[(j >> 1) * NY + (j & 1) + c * L.ncomp] : T(0);
      }
    const TE* ep = E + ebase;
    // step ex's operands -> buffer b (only where the step itself would load them)
    auto prefetch = [&](int ex, const T* xq, const TE* eq, int b) {
      if (ex >= 0 && ex < nx && ex < p1) {
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          cp_async_own<sizeof(TE)>(&sE[b][ch][threadIdx.x], eq + (ch & 1) * (eplane2 / 2) + (ch >> 2) * EY + ((ch >> 1) & 1));
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            cp_async_own<sizeof(T)>(&sB[b][c * 4 + j][threadIdx.x], xq + onp + (j >> 1) * NY + (j & 1) + c * L.ncomp);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if constexpr (kAsync) prefetch(p0 - 1, xp, ep, 0);
    for (int ex = p0 - 1; ex < p1; ++ex, xp += onp, ep += eplane2, fp += fstep) {
      T Yh[3][8];
      const int b = kAsync ? ((ex - (p0 - 1)) & 1) : 0;
      if constexpr (kAsync) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        prefetch(ex + 1, xp + onp, ep + eplane2, b ^ 1);
      }
      if (ex >= 0 && ex < nx) {
        T W[3][8], Ech[8];
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          Ech[ch] = kAsync ? (T)sE[b][ch][threadIdx.x]
                           : (T)ep[(ch & 1) * (eplane2 / 2) + (ch >> 2) * EY + ((ch >> 1) & 1)];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const T bn = kAsync ? sB[b][c * 4 + j][threadIdx.x] : xp[onp + (j >> 1) * NY + (j & 1) + c * L.ncomp];
            W[c][2 * j] = sA[c * 4 + j][threadIdx.x];
            W[c][2 * j + 1] = bn;
            sA[c * 4 + j][threadIdx.x] = bn;
          }
        l1_elem_core<T>(W, Ech, Yh);
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int k = 0; k < 8; ++k) Yh[c][k] = T(0);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (ex >= p0) fp[(j * 3 + c) * ncol] = sacc[c * 4 + j][threadIdx.x] + Yh[c][2 * j];
          sacc[c * 4 + j][threadIdx.x] = Yh[c][2 * j + 1];
        }
    }
  }
}

// sum of the level-1 element outputs at node (ix, iy, iz): kFace -> the 4 face sums
// of k_mg_l1_face, else the 8 element corners of k_mg_l1_elem (fixed order)
template <bool kFace, typename T>
__device__ __forceinline__ void l1_node_sum(const LvGeo& L, const T* __restrict__ Y, int ix, int iy, int iz, T a[3]) {
  a[0] = a[1] = a[2] = T(0);
  if (kFace) {
    const long long ncol = (long long)L.ny * L.nz;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ey = iy - (j & 1), ez = iz - (j >> 1);
      if (ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
      const long long col = (long long)ez * L.ny + ey;
#pragma unroll
      for (int c = 0; c < 3; ++c) a[c] += Y[((long long)(ix * 4 + j) * 3 + c) * ncol + col];
    }
    return;
  }
  const long long nel = L.nel();
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const int dx = d & 1, dy = (d >> 1) & 1, dz = d >> 2;
    const int ex = ix - 1 + dx, ey = iy - 1 + dy, ez = iz - 1 + dz;
    if (ex < 0 || ex >= L.nx || ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
    const long long e = ((long long)ex * L.nz + ez) * L.ny + ey;
    const int kc = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
#pragma unroll
    for (int c = 0; c < 3; ++c) a[c] += Y[(long long)(3 * kc + c) * nel + e];
  }
}

// fp32 copy of the moduli for the fp32 level-1 operator (k_mg_l1_elem<float, float>
// reads half the bytes; (float)E is what it used anyway, so results are unchanged)
__global__ void __launch_bounds__(kBlock)
k_mg_e32(long long n, const double* __restrict__ E, float* __restrict__ E32) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    E32[i] = (float)E[i];
}

// phase 2: q_i = mask( sum over the <= 8 elements of i of Y[corner of i] )
// (kScale: q_i = D^-1 mask(sum), the next power step's vector)
// level-1 damped-Jacobi sweep fused into the gather: x += w D^-1 (b - mask(A x)),
// the same arithmetic as k_mg_l1_gather<false> followed by k_mg_jacobi<1>
// (the sum is rounded to T as it would be stored), without the t round trip
template <typename T, bool kFace = true>
__global__ void __launch_bounds__(kBlock)
k_mg_l1_gather_jac(LvGeo L, const T* __restrict__ Y, const uint8_t* __restrict__ fix, T* __restrict__ x,
                   const T* __restrict__ b, const T* __restrict__ invd, const double* __restrict__ omp,
                   const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  const double omega = *omp;
  const long long tot = L.nodes(), nel = L.nel();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    T a[3];
    l1_node_sum<kFace, T>(L, Y, ix, iy, iz, a);
    const long long i = L.n(ix, iy, iz);
    const uint8_t fm = fix[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long o = i + c * L.ncomp;
      const double q = ((fm >> c) & 1) ? 0.0 : (double)a[c];
      x[o] = ((fm >> c) & 1) ? T(0) : (T)fma(omega * (double)invd[o], (double)b[o] - q, (double)x[o]);
    }
  }
}

template <bool kScale, typename T, bool kFace = true>
__global__ void __launch_bounds__(kBlock)
k_mg_l1_gather(LvGeo L, const T* __restrict__ Y, const uint8_t* __restrict__ fix, T* __restrict__ q,
               const DevState* st, const T* __restrict__ invd) {
  pdl_enter();
  MG_GATE(st);
  const long long tot = L.nodes();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    T a[3];
    l1_node_sum<kFace, T>(L, Y, ix, iy, iz, a);
    T a0 = a[0], a1 = a[1], a2 = a[2];
    const long long i = L.n(ix, iy, iz);
    const uint8_t fm = fix[i];
    if (kScale) {   // invd is 0 on fixed DOFs
      a0 *= invd[i];
      a1 *= invd[i + L.ncomp];
      a2 *= invd[i + 2 * L.ncomp];
    }
    q[i] = (fm & 1) ? T(0) : a0;
    q[i + L.ncomp] = (fm & 2) ? T(0) : a1;
    q[i + 2 * L.ncomp] = (fm & 4) ? T(0) : a2;
  }
}

// ---------------------------------------------------------------------------
// Stored levels are applied through an assembled 27-point block stencil, kept
// symmetric: with b = (dx+1) + 3(dy+1) + 9(dz+1), node i stores its self block
// (b = 13, slot 0) and the 13 forward blocks b = 14..26 (slots 1..13) as
// S[(slot*9 + ci*3 + cj) * ncomp + i]; the backward block A(i, i - d) is the
// transpose of the forward block stored at node i - d.  126 values per node
// instead of 576 per element, no element gathers.  Out-of-domain neighbours
// have zero blocks; pads of x are 0.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_stencil(LvGeo L, const double* __restrict__ K, T* __restrict__ S) {
  pdl_enter();
  const long long tot = L.nodes(), nel = L.nel();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    const long long i = L.n(ix, iy, iz);
    for (int b = 13; b < 27; ++b) {        // self + forward offsets
      const int bx = b % 3 - 1, by = (b / 3) % 3 - 1, bz = b / 9 - 1;
      double blk[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int dz = 0; dz < 2; ++dz)
        for (int dx = 0; dx < 2; ++dx)
          for (int dy = 0; dy < 2; ++dy) {
            const int ex = ix - 1 + dx, ey = iy - 1 + dy, ez = iz - 1 + dz;
            if (ex < 0 || ex >= L.nx || ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
            const int ax = 1 - dx, ay = 1 - dy, az = 1 - dz;          // corner of node i in e
            const int cx = ax + bx, cy = ay + by, cz = az + bz;        // corner of node i + b
            if (cx < 0 || cx > 1 || cy < 0 || cy > 1 || cz < 0 || cz > 1) continue;
            const long long e = ((long long)ex * L.nz + ez) * L.ny + ey;
            const int a = mg_lidx(ax, ay, az), c = mg_lidx(cx, cy, cz);
#pragma unroll
            for (int ci = 0; ci < 3; ++ci)
#pragma unroll
              for (int cj = 0; cj < 3; ++cj) blk[ci * 3 + cj] += K[(long long)((3 * a + ci) * 24 + 3 * c + cj) * nel + e];
          }
#pragma unroll
      for (int t = 0; t < 9; ++t) S[(long long)((b - 13) * 9 + t) * L.ncomp + i] = (T)blk[t];
    }
  }
}

// q = mask(A x) through the stencil; thread per node, 27 neighbour 3-vectors.
// (kU: unroll of the 13 neighbour pairs; fully unrolled (13) the loads of all
// 27 blocks are in flight together: 79 vs 91 us per level-2 apply at config 4,
// the kernel is long-scoreboard bound on its L2/HBM gathers)
#ifndef TOPO_ST_MINB
#define TOPO_ST_MINB 3   // 80 registers, 3 CTAs/SM: 8.82 vs 8.92 ms per MG-PCG iteration at 125 registers, 2 CTAs/SM (same box)
#endif
template <typename T, int kU = 13>
__global__ void __launch_bounds__(kBlock, TOPO_ST_MINB)
k_mg_apply_st(LvGeo L, const T* __restrict__ S, const T* __restrict__ x,
              const uint8_t* __restrict__ fix, T* __restrict__ q, const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  const long long tot = L.nodes();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    const long long i = L.n(ix, iy, iz);
    T a0, a1, a2;
    {   // self block
      const T x0 = x[i], x1 = x[i + L.ncomp], x2 = x[i + 2 * L.ncomp];
      const T* sb = S + i;
      a0 = fma(sb[0], x0, fma(sb[L.ncomp], x1, sb[2 * L.ncomp] * x2));
      a1 = fma(sb[3 * L.ncomp], x0, fma(sb[4 * L.ncomp], x1, sb[5 * L.ncomp] * x2));
      a2 = fma(sb[6 * L.ncomp], x0, fma(sb[7 * L.ncomp], x1, sb[8 * L.ncomp] * x2));
    }
#pragma unroll (kU)
    for (int b = 14; b < 27; ++b) {
      // b = (dx+1) + 3 (dy+1) + 9 (dz+1); layout: x -> nplane, z -> NY, y -> 1
      const long long d = (long long)(b % 3 - 1) * L.nplane + (long long)((b / 3) % 3 - 1) +
                          (long long)(b / 9 - 1) * L.NY;
      const long long so = (long long)((b - 13) * 9) * L.ncomp;
      {   // forward: A(i, i+d) x_{i+d}
        const long long j = i + d;
        const T x0 = x[j], x1 = x[j + L.ncomp], x2 = x[j + 2 * L.ncomp];
        const T* sb = S + so + i;
        a0 = fma(sb[0], x0, fma(sb[L.ncomp], x1, fma(sb[2 * L.ncomp], x2, a0)));
        a1 = fma(sb[3 * L.ncomp], x0, fma(sb[4 * L.ncomp], x1, fma(sb[5 * L.ncomp], x2, a1)));
        a2 = fma(sb[6 * L.ncomp], x0, fma(sb[7 * L.ncomp], x1, fma(sb[8 * L.ncomp], x2, a2)));
      }
      {   // backward: A(i, i-d) = A(i-d, i)^T, stored at node i-d
        const long long j = i - d;
        const T x0 = x[j], x1 = x[j + L.ncomp], x2 = x[j + 2 * L.ncomp];
        const T* sb = S + so + j;
        a0 = fma(sb[0], x0, fma(sb[3 * L.ncomp], x1, fma(sb[6 * L.ncomp], x2, a0)));
        a1 = fma(sb[L.ncomp], x0, fma(sb[4 * L.ncomp], x1, fma(sb[7 * L.ncomp], x2, a1)));
        a2 = fma(sb[2 * L.ncomp], x0, fma(sb[5 * L.ncomp], x1, fma(sb[8 * L.ncomp], x2, a2)));
      }
    }
    const uint8_t fm = fix[i];
    q[i] = (fm & 1) ? T(0) : a0;
    q[i + L.ncomp] = (fm & 2) ? T(0) : a1;
    q[i + 2 * L.ncomp] = (fm & 4) ? T(0) : a2;
  }
}

// Warp-split stencil sweep: a 256-thread block covers 32 consecutive nodes;
// warp w takes the block tasks w, w+8, w+16, w+24 (< 27) of all 32 nodes, so
// every stencil / vector load of a warp is 32 consecutive nodes (coalesced, SoA),
// and the dependency chain per thread is <= 4 tasks; the 8 warps' partial sums
// meet in shared memory and warp 0 finishes the node (fixed order).
//   kFused = false: dst = mask(A src)
//   kFused = true : dst = mask(src + w D^-1 (b - A src))   (dst != src)
//   kFromB (with kFused = false): src is the first sweep from 0, x = w D^-1 b, formed
//     on the fly from b and D^-1 (0 on fixed DOFs); xout = x, dst = mask(A x) --
//     one launch instead of a Jacobi kernel plus the stencil apply
template <bool kFused, typename T, bool kFromB = false>
__global__ void __launch_bounds__(256, 4)
k_mg_sweep_st8(LvGeo L, const T* __restrict__ S, const T* __restrict__ src, const T* __restrict__ b,
               const T* __restrict__ invd, const uint8_t* __restrict__ fix, const double* __restrict__ omp,
               T* __restrict__ dst, const DevState* st, T* __restrict__ xout = nullptr) {
  pdl_enter();
  MG_GATE(st);
  __shared__ double part[8][3][32];
  const long long tot = L.nodes();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long base = (long long)blockIdx.x * 32; base < tot; base += (long long)gridDim.x * 32) {
    const long long k = base + lane;
    const bool ok = k < tot;
    long long i = 0;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0;
    if (ok) {
      int ix, iy, iz;
      lv_decode(L, k, ix, iy, iz);
      i = L.n(ix, iy, iz);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = w + 8 * q;
        if (t >= 27) break;
        const int bb = t == 0 ? 13 : (t <= 13 ? 13 + t : t);
        const long long d = (long long)(bb % 3 - 1) * L.nplane + (long long)((bb / 3) % 3 - 1) +
                            (long long)(bb / 9 - 1) * L.NY;
        const bool back = t >= 14;
        const long long j = back ? i - d : i + d;
        const T* sb = S + (long long)((bb - 13) * 9) * L.ncomp + (back ? j : i);
        double x0, x1, x2;
        if (kFromB) {   // x = w D^-1 b rounded to T, as the Jacobi kernel would store it
          const double om = *omp;
          x0 = (double)(T)(om * (double)invd[j] * (double)b[j]);
          x1 = (double)(T)(om * (double)invd[j + L.ncomp] * (double)b[j + L.ncomp]);
          x2 = (double)(T)(om * (double)invd[j + 2 * L.ncomp] * (double)b[j + 2 * L.ncomp]);
        } else {
          x0 = (double)src[j];
          x1 = (double)src[j + L.ncomp];
          x2 = (double)src[j + 2 * L.ncomp];
        }
        double m[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) m[e] = (double)sb[(long long)e * L.ncomp];
        if (back) {   // transpose
          d0 = fma(m[0], x0, fma(m[3], x1, fma(m[6], x2, d0)));
          d1 = fma(m[1], x0, fma(m[4], x1, fma(m[7], x2, d1)));
          d2 = fma(m[2], x0, fma(m[5], x1, fma(m[8], x2, d2)));
        } else {
          d0 = fma(m[0], x0, fma(m[1], x1, fma(m[2], x2, d0)));
          d1 = fma(m[3], x0, fma(m[4], x1, fma(m[5], x2, d1)));
          d2 = fma(m[6], x0, fma(m[7], x1, fma(m[8], x2, d2)));
        }
      }
    }
    part[w][0][lane] = d0;
    part[w][1][lane] = d1;
    part[w][2][lane] = d2;
    __syncthreads();
    if (w == 0 && ok) {
      double av[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double a = part[0][c][lane];
#pragma unroll
        for (int ww = 1; ww < 8; ++ww) a += part[ww][c][lane];
        av[c] = a;
      }
      const uint8_t fm = fix[i];
      const double omega = kFused ? *omp : 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const long long o = i + c * L.ncomp;
        double v = av[c];
        if (kFused) v = fma(omega * (double)invd[o], (double)b[o] - v, (double)src[o]);
        dst[o] = ((fm >> c) & 1) ? T(0) : (T)v;
        if (kFromB) xout[o] = ((fm >> c) & 1) ? T(0) : (T)(*omp * (double)invd[o] * (double)b[o]);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Coarsest level (M6): dense matrix over free DOFs, Gauss-Jordan inverse,
// dense solve.
// ---------------------------------------------------------------------------
// Thread per (row DOF, neighbour node): A[row][3 neighbour columns] = the sum
// over the elements that hold both nodes, in k_mg_dense_fill's element order
// (dz, dx, dy) -- bitwise its result -- but 81 threads per node instead of one
// (the thread-per-node form ran the whole 225-node coarsest level of config 4
// in one CTA: 330 us of serial, strided read-modify-writes).  A is zeroed
// beforehand; every written entry has exactly one owner.
__global__ void __launch_bounds__(kBlock)
k_mg_dense_fill27(LvGeo L, const double* __restrict__ K, const int* __restrict__ dmap, int ld,
                  double* __restrict__ A) {
  pdl_enter();
  const long long tot = L.nodes() * 81, nel = L.nel();
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long k = t / 81;
    const int rem = (int)(t - k * 81), ci = rem / 27, o = rem - ci * 27;
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    const int row = dmap[L.n(ix, iy, iz) + ci * L.ncomp];
    const int jx = ix + o % 3 - 1, jy = iy + (o / 3) % 3 - 1, jz = iz + o / 9 - 1;
    if (row < 0 || jx < 0 || jx > L.nx || jy < 0 || jy > L.ny || jz < 0 || jz > L.nz) continue;
    const long long nb = L.n(jx, jy, jz);
    double s[3] = {0.0, 0.0, 0.0};
    for (int dz = 0; dz < 2; ++dz)
      for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy) {
          const int ex = ix - 1 + dx, ey = iy - 1 + dy, ez = iz - 1 + dz;
          if (ex < 0 || ex >= L.nx || ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
          const int cx = jx - ex, cy = jy - ey, cz = jz - ez;
          if (cx < 0 || cx > 1 || cy < 0 || cy > 1 || cz < 0 || cz > 1) continue;
          const long long e = ((long long)ex * L.nz + ez) * L.ny + ey;
          const int a = mg_lidx(1 - dx, 1 - dy, 1 - dz), bb = mg_lidx(cx, cy, cz);
#pragma unroll
          for (int cj = 0; cj < 3; ++cj) s[cj] += K[(long long)((3 * a + ci) * 24 + 3 * bb + cj) * nel + e];
        }
#pragma unroll
    for (int cj = 0; cj < 3; ++cj) {
      const int col = dmap[nb + cj * L.ncomp];
      if (col >= 0) A[(long long)row * ld + col] = s[cj];
    }
  }
}

// dmap[level idx of DOF] = dense index or -1 (fixed / pad).  Thread per node:
// it owns (zeroes and fills) its rows; no atomics.
__global__ void __launch_bounds__(kBlock)
k_mg_dense_fill(LvGeo L, const double* __restrict__ K, const int* __restrict__ dmap, int ld,
                double* __restrict__ A) {
  pdl_enter();
  const long long tot = L.nodes(), nel = L.nel();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    lv_decode(L, k, ix, iy, iz);
    const long long i = L.n(ix, iy, iz);
    int rows[3];   // (A is zeroed beforehand; each row is owned by one thread)
#pragma unroll
    for (int c = 0; c < 3; ++c) rows[c] = dmap[i + c * L.ncomp];
    for (int dz = 0; dz < 2; ++dz)
      for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy) {
          const int ex = ix - 1 + dx, ey = iy - 1 + dy, ez = iz - 1 + dz;
          if (ex < 0 || ex >= L.nx || ey < 0 || ey >= L.ny || ez < 0 || ez >= L.nz) continue;
          const long long e = ((long long)ex * L.nz + ez) * L.ny + ey;
          const int a = mg_lidx(1 - dx, 1 - dy, 1 - dz);
          for (int bb = 0; bb < 8; ++bb) {
            const long long nb = L.n(ex + corner_dx(bb), ey + corner_dy(bb), ez + corner_dz(bb));
            for (int cj = 0; cj < 3; ++cj) {
              const int col = dmap[nb + cj * L.ncomp];
              if (col < 0) continue;
#pragma unroll
              for (int ci = 0; ci < 3; ++ci)
                if (rows[ci] >= 0)
                  A[(long long)rows[ci] * ld + col] += K[(long long)((3 * a + ci) * 24 + 3 * bb + cj) * nel + e];
            }
          }
        }
  }
}

// ---------------------------------------------------------------------------
// Coarsest dense inverse (column-major, n_pad = multiple of kGjB, padding =
// identity) by a blocked symmetric sweep (below); SPD needs no pivoting (the
// pivot blocks are Schur-complement blocks).
// ---------------------------------------------------------------------------
constexpr int kGjB = 64;

constexpr int kGjInvNJ = 4;    // pivot-block inverse: columns per thread, 1024 threads (16 was slower)
// ---------------------------------------------------------------------------
// Symmetric blocked sweep (the coarsest inverse, M6): only the lower triangle
// of S (column-major, S(i, j) at S[j ld + i], i >= j) is kept.  Sweeping the
// pivot block K (P = S_KK^-1, C = S_:,K with rows K zero):
//   S_ij -= C_i P C_j^T (i, j not in K; one SYRKX on the lower triangle),
//   S_iK = C_i P, S_KK = -P.
// After all blocks S = -A^-1; the last kernel writes the full symmetric A^-1.
// (Half the flops of the Gauss-Jordan rank updates.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double sym_lo(const double* S, int ld, int i, int j) {
  return i >= j ? S[(long long)j * ld + i] : S[(long long)i * ld + j];
}

// P = S_KK^-1 from the lower triangle: Gauss-Jordan in one CTA of b*b/kGjInvNJ threads;
// thread (i, j0) keeps s_{i, j0 + JS m} in registers, the pivot column and row go
// through shared memory (two barriers per pivot)
__global__ void __launch_bounds__(kGjB * kGjB / kGjInvNJ)
k_sw_block_inv(const double* __restrict__ S, int ld, int k0, double* __restrict__ P) {
  pdl_enter();
  constexpr int NJ = kGjInvNJ, JS = kGjB / NJ;
  __shared__ double col[kGjB], row[kGjB], pinv;
  const int i = threadIdx.x % kGjB, j0 = threadIdx.x / kGjB;
  double a[NJ];
#pragma unroll
  for (int m = 0; m < NJ; ++m) a[m] = sym_lo(S, ld, k0 + i, k0 + j0 + JS * m);
  for (int k = 0; k < kGjB; ++k) {
#pragma unroll
    for (int m = 0; m < NJ; ++m) {
      if (j0 + JS * m == k) col[i] = a[m];
      if (i == k) row[j0 + JS * m] = a[m];
      if (i == k && j0 + JS * m == k) pinv = 1.0 / a[m];   // one fp64 division per pivot, not one per thread
    }
    __syncthreads();
    const double ip = pinv;
    const double cik = col[i];
#pragma unroll
    for (int m = 0; m < NJ; ++m) {
      const int j = j0 + JS * m;
      double v;
      if (i == k && j == k) v = ip;
      else if (i == k) v = row[j] * ip;
      else if (j == k) v = -cik * ip;
      else v = a[m] - cik * row[j] * ip;
      a[m] = v;
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < NJ; ++m) P[(j0 + JS * m) * kGjB + i] = a[m];
}

// C = S_:,K (rows K zero), read from the lower triangle (n_pad x b, column-major)
__global__ void __launch_bounds__(kBlock)
k_sw_take_col(const double* __restrict__ S, int ld, int k0, double* __restrict__ C) {
  pdl_enter();
  const long long tot = (long long)ld * kGjB;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % ld), j = (int)(t / ld);
    C[t] = (i >= k0 && i < k0 + kGjB) ? 0.0 : sym_lo(S, ld, i, k0 + j);
  }
}

// S_iK = (C P)_i for i not in K, S_KK = -P (lower triangle)
__global__ void __launch_bounds__(kBlock)
k_sw_put_panel(double* __restrict__ S, int ld, int k0, const double* __restrict__ CP, const double* __restrict__ P) {
  pdl_enter();
  const long long tot = (long long)ld * kGjB;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % ld), jj = (int)(t / ld), k = k0 + jj;
    if (i >= k0 && i < k0 + kGjB) {
      if (i >= k) S[(long long)k * ld + i] = -P[jj * kGjB + (i - k0)];
    } else if (i > k) {
      S[(long long)k * ld + i] = CP[t];
    } else {
      S[(long long)i * ld + k] = CP[t];
    }
  }
}

// A^-1 = -S, full symmetric (the coarse solve reads whole rows)
__global__ void __launch_bounds__(kBlock)
k_sw_finish(double* __restrict__ S, int ld) {
  pdl_enter();
  const long long tot = (long long)ld * ld;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % ld), j = (int)(t / ld);
    if (i > j) {
      const double v = -S[t];
      S[t] = v;
      S[(long long)i * ld + j] = v;
    } else if (i == j) {
      S[t] = -S[t];
    }
  }
}

__global__ void k_gj_pad(double* __restrict__ A, int n, int ld) {
  pdl_enter();
  for (int t = threadIdx.x + blockIdx.x * blockDim.x; t < ld - n; t += gridDim.x * blockDim.x)
    A[(long long)(n + t) * ld + n + t] = 1.0;
}

// One Gauss-Jordan pivot step (in place on SPD, no pivoting), ping-pong:
//   out_kk = 1/p, out_kj = a_kj/p, out_ik = -a_ik/p, out_ij = a_ij - a_ik a_kj / p.
// After steps k = 0..n-1 the buffer holds A^-1.
__global__ void __launch_bounds__(kBlock)
k_mg_gj_step(const double* __restrict__ a, double* __restrict__ o, int n, int k) {
  pdl_enter();
  const long long tot = (long long)n * n;
  const double p = a[(long long)k * n + k], ip = 1.0 / p;
  for (long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x; id < tot;
       id += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(id / n), j = (int)(id - (long long)i * n);
    double v;
    if (i == k && j == k) v = ip;
    else if (i == k) v = a[id] * ip;
    else if (j == k) v = -a[id] * ip;
    else v = a[id] - a[(long long)i * n + k] * a[(long long)k * n + j] * ip;
    o[id] = v;
  }
}

// x[imap[r]] = sum_j Ainv[r][j] b[imap[j]]  (warp per row, fixed lane order)
template <typename T>
__global__ void __launch_bounds__(kBlock)
k_mg_coarse_solve(const double* __restrict__ Ainv, int n, int ld, const long long* __restrict__ imap,
                  const T* __restrict__ b, T* __restrict__ x, const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < n; r += nwarp) {
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s = fma(Ainv[(long long)r * ld + j], (double)b[imap[j]], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) x[imap[r]] = (T)s;
  }
}

// fp32 hierarchy: the coarsest inverse rounded to fp32 (half the bytes: 60 MB at
// config 4, L2-resident across the K-cycle's repeated coarsest solves); b is
// gathered once per block into shared memory; fp64 accumulation.
__global__ void k_mg_inv_to32(const double* __restrict__ A, float* __restrict__ A32, long long n) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    A32[i] = (float)A[i];
}
__global__ void __launch_bounds__(kBlock)
k_mg_coarse_solve32(const float* __restrict__ Ainv, int n, int ld, const long long* __restrict__ imap,
                    const float* __restrict__ b, float* __restrict__ x, const DevState* st) {
  pdl_enter();
  MG_GATE(st);
  extern __shared__ float bsh[];
  for (int j = threadIdx.x; j < n; j += blockDim.x) bsh[j] = b[imap[j]];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < n; r += nwarp) {
    const float* row = Ainv + (long long)r * ld;
    double s = 0.0;
    for (int j = lane * 4; j < n; j += 128) {   // ld is a multiple of 64: 16-byte row chunks
      const float4 a = *reinterpret_cast<const float4*>(row + j);
      s = fma((double)a.x, (double)bsh[j], s);
      if (j + 1 < n) s = fma((double)a.y, (double)bsh[j + 1], s);
      if (j + 2 < n) s = fma((double)a.z, (double)bsh[j + 2], s);
      if (j + 3 < n) s = fma((double)a.w, (double)bsh[j + 3], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) x[imap[r]] = (float)s;
  }
}

// ---------------------------------------------------------------------------
// Dense fp64 "NT" product with an inner dimension of 64 (hand-written; replaces
// the cuBLAS DGEMM / DSYRKX calls of round 1):
//   Cm[i + j ldc] = beta Cm[..] + alpha sum_{t < 64} A[i + t lda] B[j + t ldb]
// for i < M, j < N (lower = 1: only i >= j).  Column-major like BLAS.  Uses:
//   level-2 Galerkin   K2 = Eg tab64^T            (M = nel_2, N = 576)
//   symmetric sweep    CP = C P  (P symmetric)    (M = n_pad, N = 64)
//                      S -= C (CP)^T, lower       (M = N = n_pad)
// A 64 x 64 output tile per 256-thread block, 4 x 4 outputs per thread, the
// 64-deep operands staged in shared memory in two halves.
// ---------------------------------------------------------------------------
constexpr int kNtTile = 64;
__global__ void __launch_bounds__(256)
k_dgemm_nt64(const double* __restrict__ A, long long lda, const double* __restrict__ B, long long ldb,
             double* __restrict__ Cm, long long ldc, int M, int N, double alpha, double beta, int lower) {
  pdl_enter();
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (lower && bj > bi) return;
  __shared__ double As[32][kNtTile + 1], Bs[32][kNtTile + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = bi * kNtTile, j0 = bj * kNtTile;
  double acc[4][4] = {};
  for (int h = 0; h < 2; ++h) {
    for (int q = tid; q < 32 * kNtTile; q += 256) {   // q = t * 64 + r: r fastest (coalesced)
      const int r = q & (kNtTile - 1), t = q >> 6;
      const int ia = i0 + r, jb = j0 + r;
      As[t][r] = ia < M ? A[ia + (long long)(h * 32 + t) * lda] : 0.0;
      Bs[t][r] = jb < N ? B[jb + (long long)(h * 32 + t) * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int t = 0; t < 32; ++t) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[t][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[t][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + ty * 4 + a, j = j0 + tx * 4 + b;
      if (i >= M || j >= N || (lower && i < j)) continue;
      double* c = Cm + i + (long long)j * ldc;
      *c = beta == 0.0 ? alpha * acc[a][b] : fma(alpha, acc[a][b], beta * *c);
    }
}

// Same product on the fp64 tensor cores (DMMA, mma.sync m8n8k4 .f64) for the
// large level-2 Galerkin product (M = nel_2 = 524 288 at config 4, N = 576):
// block tile 128 (M) x 64 (N), 8 warps of 32 x 32 (4 x 4 m8n8 tiles, 32
// accumulators per thread), the whole 64-deep operands in shared memory.
// N must be a multiple of 64 (576 is); beta = 0, no triangle.
constexpr int kTcM = 128, kTcN = 64, kTcK = 64, kTcPadA = kTcM + 1, kTcPadB = kTcN + 1;
constexpr int kTcSmem = (kTcK * kTcPadA + kTcK * kTcPadB) * 8;
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(256)
k_dgemm_nt64_tc(const double* __restrict__ A, long long lda, const double* __restrict__ B, long long ldb,
                double* __restrict__ Cm, long long ldc, int M, int N, double alpha) {
  pdl_enter();
  extern __shared__ double tsm[];
  double* As = tsm;                       // [t][i], pitch kTcPadA
  double* Bs = tsm + kTcK * kTcPadA;      // [t][j], pitch kTcPadB
  const int i0 = blockIdx.y * kTcM, j0 = blockIdx.x * kTcN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < kTcK * kTcM; q += 256) {
    const int r = q & (kTcM - 1), t = q / kTcM;
    As[t * kTcPadA + r] = (i0 + r) < M ? A[(i0 + r) + (long long)t * lda] : 0.0;
  }
  for (int q = tid; q < kTcK * kTcN; q += 256) {
    const int r = q & (kTcN - 1), t = q / kTcN;
    Bs[t * kTcPadB + r] = (j0 + r) < N ? B[(j0 + r) + (long long)t * ldb] : 0.0;
  }
  __syncthreads();
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;   // 4 x 2 warps
  const int g = lane >> 2, tg = lane & 3;
  double acc[4][4][2] = {};
  for (int k0 = 0; k0 < kTcK; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = As[(k0 + tg) * kTcPadA + wm + mi * 8 + g];   // A(row g, col tg)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(k0 + tg) * kTcPadB + wn + ni * 8 + g];   // B(row tg, col g)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni], a[mi], b[ni]);
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + wm + mi * 8 + g, j = j0 + wn + ni * 8 + tg * 2 + e;   // C(row g, col 2 tg + e)
        if (i < M && j < N) Cm[i + (long long)j * ldc] = alpha * acc[mi][ni][e];
      }
}

// Persistent, pipelined form of k_dgemm_nt64_tc (the level-2 Galerkin product):
// one CTA per SM walks its M tiles; a tile's 128 x 64 A block is loaded ONCE and
// kept for all N / 64 output blocks (the one-shot kernel re-read it per block);
// the next stage's B block (64 x 64, L2-resident) and, at a tile boundary, the
// next A block are in flight (cp.async, 8-byte, zero-filled past M) while the
// current stage runs on the DMMA pipe.  Stage s = (tile s / nb, N block s % nb).
// Row pitches 132 / 68 doubles: the m8n8k4 operand reads (lane = 4 g + tg,
// address (k0 + tg) pitch + g) hit distinct banks.  Same k order as the one-shot
// kernel (4-deep DMMA steps, k ascending): bitwise the same C.
constexpr int kT2PA = 132, kT2PB = 68;
constexpr int kT2Smem = (2 * kTcK * kT2PA + 2 * kTcK * kT2PB) * 8;   // 204 800 B: 1 CTA/SM
__device__ __forceinline__ void cp_async8(double* s, const double* g, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(g), "r"(pred ? 8 : 0) : "memory");
}
__global__ void __launch_bounds__(256, 1)
k_dgemm_nt64_tc2(const double* __restrict__ A, long long lda, const double* __restrict__ B, long long ldb,
                 double* __restrict__ Cm, long long ldc, int M, int N, double alpha) {
  pdl_enter();
  extern __shared__ double tsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = N / kTcN;
  const long long ntile = (M + kTcM - 1) / kTcM;
  const long long my_tiles = ntile > blockIdx.x ? (ntile - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long S = my_tiles * nb;
  auto bufA = [&](long long k) { return tsm + (k & 1) * (kTcK * kT2PA); };
  auto bufB = [&](long long s) { return tsm + 2 * kTcK * kT2PA + (s & 1) * (kTcK * kT2PB); };
  auto issue = [&](long long s) {   // stage s's B block, and its A block if s starts a tile
    const long long k = s / nb;
    const int jb = (int)(s - k * nb);
    if (jb == 0) {
      const long long i0 = (blockIdx.x + k * gridDim.x) * kTcM;
      double* As = bufA(k);
      for (int q = tid; q < kTcK * kTcM; q += 256) {
        const int r = q & (kTcM - 1), t = q / kTcM;
        const bool ok = i0 + r < M;
        cp_async8(As + t * kT2PA + r, ok ? A + (i0 + r) + (long long)t * lda : A, ok);
      }
    }
    double* Bs = bufB(s);
    for (int q = tid; q < kTcK * kTcN; q += 256) {
      const int r = q & (kTcN - 1), t = q / kTcN;
      cp_async8(Bs + t * kT2PB + r, B + (jb * kTcN + r) + (long long)t * ldb, true);
    }
  };
  if (S > 0) issue(0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;   // 4 x 2 warps
  const int g = lane >> 2, tg = lane & 3;
  for (long long s = 0; s < S; ++s) {
    if (s + 1 < S) issue(s + 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const long long k = s / nb;
    const int jb = (int)(s - k * nb);
    const double* As = bufA(k);
    const double* Bs = bufB(s);
    double acc[4][4][2] = {};
#pragma unroll 4
    for (int k0 = 0; k0 < kTcK; k0 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[(k0 + tg) * kT2PA + wm + mi * 8 + g];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(k0 + tg) * kT2PB + wn + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni], a[mi], b[ni]);
    }
    const long long i0 = (blockIdx.x + k * gridDim.x) * kTcM;
    const int j0 = jb * kTcN;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const long long i = i0 + wm + mi * 8 + g;
          const int j = j0 + wn + ni * 8 + tg * 2 + e;
          if (i < M) Cm[i + (long long)j * ldc] = alpha * acc[mi][ni][e];
        }
    __syncthreads();   // stage s's buffers are refilled by issue(s + 2)
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace topo
