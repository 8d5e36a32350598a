// sm_100a kernels of the SIMP hot path.
// fp64 throughout; no tensor cores (tcgen05 has no f64 kind).
#pragma once
#include "common.cuh"
#include "matvec_wht.cuh"

namespace topo {

constexpr int kMaxStencil = 1331;      // (2R+1)^3 for R <= 5 (rmin <= 6)
__constant__ double c_KE[576];          // element stiffness, row-major 24x24
__constant__ int4 c_st_off[kMaxStencil];  // filter stencil offsets (dx, dy, dz, -)
__constant__ double c_st_w[kMaxStencil];  // rmin - |d|

struct Material { double E0, Emin, penal, kd; };

// local index of the element corner (a,b,c) in SPEC S:45 order
__host__ __device__ constexpr int lidx(int a, int b, int c) {
  return 4 * c + (b ? (a ? 2 : 3) : (a ? 1 : 0));
}

__device__ __forceinline__ bool decode_node(const Geo& g, long long i, int& ix, int& iy, int& iz) {
  const long long pl = i / g.nplane;
  const int rem = (int)(i - pl * g.nplane);
  const int zs = rem / g.NY, ys = rem - zs * g.NY;
  ix = (int)pl - 1 + g.ex0;
  iy = ys - 1;
  iz = zs - 1;
  return (ys >= 1) & (ys <= g.nely + 1) & (zs >= 1) & (zs <= g.nelz + 1);
}
__device__ __forceinline__ bool decode_elem(const Geo& g, long long i, int& ex, int& ey, int& ez) {
  const long long pl = i / g.eplane;
  const int rem = (int)(i - pl * g.eplane);
  const int zs = rem / g.EY, ys = rem - zs * g.EY;
  ex = (int)pl - g.H + g.ex0;
  ey = ys - 1;
  ez = zs - 1;
  return (ys >= 1) & (ys <= g.nely) & (zs >= 1) & (zs <= g.nelz);
}

// ===========================================================================
// A1  SIMP modulus  E_e = Emin + xPhys_e^p (E0 - Emin)          (§2.3)
//     over every in-domain element of the local array (owned + halos).
// ===========================================================================
// x^p for the SIMP power: small integer exponents (p = 3, the configs' and the
// paper's "commonly 3", and p - 1 = 2) by multiplication -- the general pow is
// ~50 fp64 instructions and dominated k_sens / k_efield
__device__ __forceinline__ double simp_pow(double x, double p) {
  if (p == 3.0) return x * x * x;
  if (p == 2.0) return x * x;
  if (p == 1.0) return x;
  return pow(x, p);
}

__global__ void k_efield(Geo g, Material m, const double* __restrict__ xphys,
                         double* __restrict__ E) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.nelloc;
       i += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    if (!decode_elem(g, i, ex, ey, ez) || ex < 0 || ex >= g.nelx) continue;
    E[i] = m.Emin + simp_pow(xphys[i], m.penal) * (m.E0 - m.Emin);
  }
}

// Jacobi inverse diagonal per node: 1/(kd * sum_{e ni n} E_e).
// diag(K) is one scalar per node because every KE_ii = (lambda+4mu)/9.
__global__ void k_invdiag(Geo g, Material m, const double* __restrict__ E,
                          const uint8_t* __restrict__ fixm, double* __restrict__ invd) {
  pdl_enter();
  const long long b = g.nplane, e = (long long)(g.nown + 1) * g.nplane;
  for (long long i = b + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e;
       i += (long long)gridDim.x * blockDim.x) {
    int ix, iy, iz;
    if (!decode_node(g, i, ix, iy, iz)) continue;
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 8; ++d)
      s += E[elem_idx(g, ix - 1 + (d & 1), iy - 1 + ((d >> 1) & 1), iz - 1 + (d >> 2))];
    // one scalar per node (r is exactly 0 on fixed DOFs, so no mask is needed)
    invd[i] = 1.0 / (m.kd * s);
  }
}

// ===========================================================================
// A3/A4  PCG vector kernels over the owned node planes (pads are zero and
// stay zero).  SoA: component stride ncomp.
// ===========================================================================
// kMG: beta and rz (= r.z) come from the V-cycle's last sweep (k_mg_jacobi<2>),
// so only the iteration count, the pending-u bookkeeping and the stopping test
// are updated here.
template <bool kMG = false>
__device__ __forceinline__ void cg_finish_update(DevState* st, double rz_new, double rr, int even) {
  if (even) {                 // u update deferred: the next (odd) update applies both steps
    st->alpha_prev = st->alpha;
    st->pending = 1;
  } else {
    st->pending = 0;
  }
  if (!kMG) {
    st->beta = rz_new / st->rz;
    st->rz = rz_new;
  }
  st->rr = rr;
  st->it += 1;
  st->fresh = 0;
  if ((!isfinite(rr) || !isfinite(rz_new)) && !st->solo) {
    st->status = 3;
    st->done = 1;
  } else if (!st->solo && rr <= st->tol2 * st->bb) {
    st->done = 1;
  } else if (st->it >= st->max_it) {
    st->status = 2;
    st->done = 1;
  }
}

// PCG vector update, u updated every other iteration:
//   even slot (kU = false): r -= alpha q                            (u pending)
//   odd slot  (kU = true) : u += alpha_prev p_prev + alpha p ; r -= alpha q
// r is 0 on fixed DOFs (q comes unmasked from the matvec); partial
// (r M^{-1} r, r r).  double2 over pairs of nodes of the owned planes (pads
// are zero and stay zero).  Saves one read+write of u every second iteration.
// TK: type of r and q (double; float for the fp32 Krylov vectors of the
// multigrid PCG, SURVEY f3 -- the true residual is always fp64, so the fp32
// recursion only decides when to check it)
template <typename TK> struct Vec2T { using t = double2; };
template <> struct Vec2T<float> { using t = float2; };
template <bool kU, bool kMG, typename TK = double>
__global__ void __launch_bounds__(kBlock, 2)
k_update(Geo g, DevState* st, double* __restrict__ u, TK* __restrict__ r,
         const double* __restrict__ pprev, const double* __restrict__ p, const TK* __restrict__ q,
         const double* __restrict__ invd, const uint8_t* __restrict__ fixm, double* partials,
         unsigned int* counter, int finish) {
  pdl_enter();
  using V2 = typename Vec2T<TK>::t;
  if (st->done) return;
  const double alpha = st->alpha, alpha_prev = kU ? st->alpha_prev : 0.0;
  const long long b0 = g.nplane, npair = (long long)g.nown * g.nplane / 2;
  const long long nc = g.ncomp;
  double rz = 0.0, rr = 0.0;
  constexpr int UN = kU ? 1 : 2;            // pairs per thread per trip: all loads issued first
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; j0 < npair; j0 += UN * stride) {
    V2 rv[UN][3], qq[UN][3];
    double2 uu[UN][3], p0[UN][3], pp[UN][3], iv[UN];
    uchar2 fm[UN];
    bool ok[UN];
#pragma unroll
    for (int w = 0; w < UN; ++w) {
      const long long j = j0 + w * stride;
      ok[w] = j < npair;
      const long long i = b0 + 2 * (ok[w] ? j : j0);
      if (!kMG) iv[w] = *reinterpret_cast<const double2*>(invd + i);
      fm[w] = *reinterpret_cast<const uchar2*>(fixm + i);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const long long k = i + c * nc;
        rv[w][c] = *reinterpret_cast<const V2*>(r + k);
        qq[w][c] = *reinterpret_cast<const V2*>(q + k);
        if (kU) {
          uu[w][c] = *reinterpret_cast<const double2*>(u + k);
          p0[w][c] = *reinterpret_cast<const double2*>(pprev + k);
          pp[w][c] = *reinterpret_cast<const double2*>(p + k);
        }
      }
    }
#pragma unroll
    for (int w = 0; w < UN; ++w) {
      if (!ok[w]) continue;
      const long long i = b0 + 2 * (j0 + w * stride);
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const long long k = i + c * nc;
        if (kU) {
          double2 un;
          un.x = fma(alpha, pp[w][c].x, fma(alpha_prev, p0[w][c].x, uu[w][c].x));
          un.y = fma(alpha, pp[w][c].y, fma(alpha_prev, p0[w][c].y, uu[w][c].y));
          *reinterpret_cast<double2*>(u + k) = un;
        }
        V2 rn;
        rn.x = (TK)((fm[w].x >> c) & 1 ? 0.0 : fma(-alpha, (double)qq[w][c].x, (double)rv[w][c].x));
        rn.y = (TK)((fm[w].y >> c) & 1 ? 0.0 : fma(-alpha, (double)qq[w][c].y, (double)rv[w][c].y));
        *reinterpret_cast<V2*>(r + k) = rn;
        s0 = fma((double)rn.x, (double)rn.x, s0);
        s1 = fma((double)rn.y, (double)rn.y, s1);
      }
      if (!kMG) rz = fma(s0, iv[w].x, fma(s1, iv[w].y, rz));
      rr += s0 + s1;
    }
  }
  __shared__ double tot[2];
  double v[2] = {rz, rr};
  if (grid_reduce<2>(v, partials, counter, tot) && threadIdx.x == 0) {
    if (finish) cg_finish_update<kMG>(st, tot[0], tot[1], kU ? 0 : 1);
    else { st->sums[0] = tot[0]; st->sums[1] = tot[1]; }
  }
}

// out = 1/v (0 where v = 0: padding elements): the filter's 1/Hs
__global__ void k_recip(long long n, const double* __restrict__ v, double* __restrict__ out) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = v[i] != 0.0 ? 1.0 / v[i] : 0.0;
}

// dst = (double) src over a whole buffer (the fp32 Krylov residual back into r after a solve)
__global__ void k_f2d(long long n, const float* __restrict__ src, double* __restrict__ dst) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = (double)src[i];
}

// u += alpha_prev p (the deferred half-step) when the solve stops after an even slot
__global__ void k_flush_u(Geo g, double alpha_prev, double* __restrict__ u, const double* __restrict__ p) {
  pdl_enter();
  const long long b0 = g.nplane, n = (long long)g.nown * g.nplane;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < 3 * n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long c = k / n, i = b0 + (k - c * n) + c * g.ncomp;
    u[i] = fma(alpha_prev, p[i], u[i]);
  }
}
__global__ void k_clear_pending(DevState* st) {
  pdl_enter(); st->pending = 0; }

// Multi-slab finish kernels (after the allreduce of st->sums).
__global__ void k_finish_alpha(DevState* st) {
  pdl_enter();
  if (st->done) return;
  const double pq = st->sums[0];
  st->pq = pq;
  if (!(pq > 0.0) || !isfinite(pq)) {
    if (st->solo) st->alpha = 0.0;
    else { st->status = 3; st->done = 1; }
  } else st->alpha = st->rz / pq;
}
template <bool kMG = false>
__global__ void k_finish_update(DevState* st, int even) {
  pdl_enter();
  if (st->done) return;
  cg_finish_update<kMG>(st, st->sums[0], st->sums[1], even);
}
// multigrid PCG: rho = r.V(r) of the V-cycle's last sweep (allreduced) -> beta, rz
// flex (K-cycle, reading M9): Polak-Ribiere beta = -alpha (q.z)/rz, q.z in sums[1]
__global__ void k_finish_rho(DevState* st, int flex) {
  pdl_enter();
  if (st->done) return;
  const double rho = st->sums[0];
  if ((!(rho > 0.0) || !isfinite(rho)) && st->solo) {
    st->beta = 0.0;
  } else if (!(rho > 0.0) || !isfinite(rho)) {
    st->status = 3;
    st->done = 1;
  } else {
    st->beta = st->fresh ? 0.0 : flex ? -st->alpha * st->sums[1] / st->rz : rho / st->rz;
    st->rz = rho;
  }
}

// r = f - q, 0 on fixed DOFs (q arrives unmasked from the matvec); partial
// (r M^{-1} r, r r).  Used at PCG start and for the true-residual check.
template <typename TK = double>
__global__ void __launch_bounds__(kBlock)
k_residual(Geo g, DevState* st, const double* __restrict__ f, const double* __restrict__ q,
           const double* __restrict__ invd, const uint8_t* __restrict__ fixm, TK* __restrict__ r,
           int write_r, double* partials, unsigned int* counter) {
  pdl_enter();
  const long long b0 = g.nplane, n = (long long)g.nown * g.nplane;
  double rz = 0.0, rr = 0.0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long i = b0 + k;
    const uint8_t fm = fixm[i];
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double rv = (fm >> c) & 1 ? 0.0 : f[i + c * g.ncomp] - q[i + c * g.ncomp];
      if (write_r) {
        r[i + c * g.ncomp] = (TK)rv;
        rv = (double)(TK)rv;   // the sums of the vector the recursion continues from
      }
      s = fma(rv, rv, s);
    }
    rz = fma(s, invd[i], rz);
    rr += s;
  }
  __shared__ double tot[2];
  double v[2] = {rz, rr};
  if (grid_reduce<2>(v, partials, counter, tot) && threadIdx.x == 0) {
    st->sums[0] = tot[0];
    st->sums[1] = tot[1];
  }
}

// generic dot over owned node planes: sums[slot] = a . b
__global__ void __launch_bounds__(kBlock)
k_dot(Geo g, DevState* st, const double* __restrict__ a, const double* __restrict__ b,
      int slot, double* partials, unsigned int* counter) {
  pdl_enter();
  const long long b0 = g.nplane, n = (long long)g.nown * g.nplane;
  double s = 0.0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < 3 * n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long c = k / n, i = b0 + (k - c * n) + c * g.ncomp;
    s = fma(a[i], b[i], s);
  }
  __shared__ double tot[1];
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter, tot) && threadIdx.x == 0) st->sums[slot] = tot[0];
}

// ===========================================================================
// A5  ce = u_e^T KE u_e ; dc = -p xPhys^(p-1)(E0-Emin) ce (0 on passive);
//     partial c = sum E ce.                                     (§2.3)
// ===========================================================================
__global__ void __launch_bounds__(kBlock)
k_sens(Geo g, DevState* st, Material m, const double* __restrict__ u,
       const double* __restrict__ E, const double* __restrict__ xphys,
       const uint8_t* __restrict__ passive, double* __restrict__ ce, double* __restrict__ dc,
       double* partials, unsigned int* counter) {
  pdl_enter();
  // ce = u_e^T KE u_e = P^T B P with P = H u_e (KE = H^T B H, B block-diagonal in
  // the Walsh basis, matvec_wht.cuh): ~140 fp64 ops instead of the 576-FMA
  // dense quadratic form (SURVEY App. A "The same factorisation gives ce")
  const long long b0 = (long long)g.H * g.eplane, e0 = (long long)(g.H + g.nex) * g.eplane;
  double csum = 0.0;
  for (long long i = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e0;
       i += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    if (!decode_elem(g, i, ex, ey, ez)) continue;
    double P[3][8], Q[3][8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {     // natural corner index k = ax + 2 ay + 4 az
      const long long n = node_idx(g, ex + (k & 1), ey + ((k >> 1) & 1), ez + (k >> 2));
#pragma unroll
      for (int c = 0; c < 3; ++c) P[c][k] = u[n + c * g.ncomp];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int bb = 1; bb < 8; bb <<= 1)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (!(k & bb)) {
            const double x0 = P[c][k], x1 = P[c][k | bb];
            P[c][k] = x0 + x1;
            P[c][k | bb] = x0 - x1;
          }
    wht_block(P, 1.0, Q);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) s = fma(P[c][k], Q[c][k], s);
    ce[i] = s;
    const double xp = xphys[i];
    dc[i] = passive[i] ? 0.0 : -m.penal * simp_pow(xp, m.penal - 1.0) * (m.E0 - m.Emin) * s;
    csum = fma(E[i], s, csum);
  }
  __shared__ double tot[1];
  double v[1] = {csum};
  if (grid_reduce<1>(v, partials, counter, tot) && threadIdx.x == 0) st->sums[0] = tot[0];
}

// A5 x-marching: a thread owns one (ey, ez) element column and walks kSensCX
// elements along x; the 4 corners x 3 components of each node plane are loaded
// once and shared by the two elements left and right of it (12 instead of 24
// loads per element; the next plane's loads are issued before the current
// element's arithmetic).  Same per-element arithmetic as k_sens.
constexpr int kSensCX = 16;
__global__ void __launch_bounds__(kBlock, 2)
k_sens_x(Geo g, DevState* st, Material m, const double* __restrict__ u,
         const double* __restrict__ E, const double* __restrict__ xphys,
         const uint8_t* __restrict__ passive, double* __restrict__ ce, double* __restrict__ dc,
         double* partials, unsigned int* counter) {
  pdl_enter();
  const long long ncol = (long long)g.nely * g.nelz;
  const int nchunk = (g.nex + kSensCX - 1) / kSensCX;
  double csum = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncol * nchunk;
       t += (long long)gridDim.x * blockDim.x) {
    const int chunk = (int)(t / ncol);
    const long long col = t - (long long)chunk * ncol;
    const int ez = (int)(col / g.nely), ey = (int)(col - (long long)ez * g.nely);
    const int xa = g.ex0 + chunk * kSensCX, xb = min(xa + kSensCX, g.ex0 + g.nex);
    // corners of a node plane, j = ay + 2 az
    const long long n0 = node_idx(g, xa, ey, ez);
    long long o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = (long long)(j >> 1) * g.NY + (j & 1);
    double A[3][4], B[3][4];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 4; ++j) A[c][j] = u[n0 + o[j] + c * g.ncomp];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < 4; ++j) B[c][j] = u[n0 + g.nplane + o[j] + c * g.ncomp];
    long long e = elem_idx(g, xa, ey, ez);
    double Ee = E[e], xp = xphys[e];   // this element's scalars; the next element's are loaded one step ahead
    uint8_t pv = passive[e];
    for (int ex = xa; ex < xb; ++ex, e += g.eplane) {
      double P[3][8], Q[3][8];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) {   // natural corner index k = ax + 2 ay + 4 az = ax + 2 j
          P[c][2 * j] = A[c][j];
          P[c][2 * j + 1] = B[c][j];
          A[c][j] = B[c][j];
        }
      if (ex + 1 < xb) {                // next plane's corners, in flight during the arithmetic
        const long long nn = n0 + (long long)(ex + 2 - xa) * g.nplane;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int j = 0; j < 4; ++j) B[c][j] = u[nn + o[j] + c * g.ncomp];
      }
      const double Ec = Ee, xc = xp;
      const uint8_t pc = pv;
      if (ex + 1 < xb) {
        Ee = E[e + g.eplane];
        xp = xphys[e + g.eplane];
        pv = passive[e + g.eplane];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int bb = 1; bb < 8; bb <<= 1)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (!(k & bb)) {
              const double x0 = P[c][k], x1 = P[c][k | bb];
              P[c][k] = x0 + x1;
              P[c][k | bb] = x0 - x1;
            }
      wht_block(P, 1.0, Q);
      double sv = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 8; ++k) sv = fma(P[c][k], Q[c][k], sv);
      ce[e] = sv;
      dc[e] = pc ? 0.0 : -m.penal * simp_pow(xc, m.penal - 1.0) * (m.E0 - m.Emin) * sv;
      csum = fma(Ec, sv, csum);
    }
  }
  __shared__ double tot[1];
  double v[1] = {csum};
  if (grid_reduce<1>(v, partials, counter, tot) && threadIdx.x == 0) st->sums[0] = tot[0];
}

// ===========================================================================
// A6  rmin cone filter (§2.4), truncated at the domain boundary.
// out_i = post_i * sum_j H_ij val_j over in-domain j of the stencil.
// ===========================================================================
enum FiltMode { F_HS = 0, F_X0 = 1, F_DIV = 2, F_XDC = 3, F_PLAIN = 4 };
//  F_HS   : out = sum H                                  (row sums Hs)
//  F_X0   : out = (sum H a)/Hs, passive -> 0 void, 1 solid (density filter of x; R27)
//  F_DIV  : out = sum H (a/b)                             (H(dc/Hs), H(dv/Hs))
//  F_XDC  : out = (sum H a b)/(Hs max(1e-3, a_i))         (sensitivity filter, a=x, b=dc)
//  F_PLAIN: out = (sum H a)/Hs                            (plain)
template <int MODE>
__global__ void __launch_bounds__(kBlock)
k_filter(Geo g, int nst, const double* __restrict__ a, const double* __restrict__ b,
         const double* __restrict__ hs, const uint8_t* __restrict__ passive,
         double* __restrict__ out, int all_local) {
  pdl_enter();
  // all_local: evaluate on every in-domain local element (Hs incl. halos), else owned only
  const long long b0 = all_local ? 0 : (long long)g.H * g.eplane;
  const long long e0 = all_local ? g.nelloc : (long long)(g.H + g.nex) * g.eplane;
  for (long long i = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e0;
       i += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    if (!decode_elem(g, i, ex, ey, ez) || ex < 0 || ex >= g.nelx) continue;
    double s = 0.0;
    for (int k = 0; k < nst; ++k) {
      const int4 o = c_st_off[k];
      const int jx = ex + o.x, jy = ey + o.y, jz = ez + o.z;
      if (jx < 0 || jx >= g.nelx || jy < 0 || jy >= g.nely || jz < 0 || jz >= g.nelz) continue;
      const long long j = i + (long long)o.x * g.eplane + (long long)o.z * g.EY + o.y;
      double v;
      if (MODE == F_HS) v = 1.0;
      else if (MODE == F_DIV) v = a[j] / b[j];
      else if (MODE == F_XDC) v = a[j] * b[j];
      else v = a[j];
      s = fma(c_st_w[k], v, s);
    }
    double r;
    if (MODE == F_HS || MODE == F_DIV) r = s;
    else if (MODE == F_XDC) r = s / (hs[i] * fmax(1e-3, a[i]));
    else r = s / hs[i];
    if (MODE == F_X0 && passive[i]) r = passive[i] == kSolid ? 1.0 : 0.0;   // R14, R27
    out[i] = r;
  }
}

// Filter, fast path: the per-element operand v_j (a_j, a_j/b_j or a_j b_j) is
// written once into a zero-padded copy (R pad elements in y and z; x halos are
// the element array's own H >= R planes, 0 outside the domain), so the stencil
// sum is a branch-free gather at constant offsets (c_st_poff) and the
// truncation at the domain boundary comes from the zero padding.
__constant__ int c_st_poff[kMaxStencil];

struct FiltPad { int FY, FZ, R; long long fplane; };   // padded layout: (exl*FZ + ez+R)*FY + ey+R

template <int MODE>
__global__ void __launch_bounds__(kBlock)
k_filt_prep(Geo g, FiltPad fp, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ vpad) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.nelloc;
       i += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    if (!decode_elem(g, i, ex, ey, ez) || ex < 0 || ex >= g.nelx) continue;
    const long long exl = ex - g.ex0 + g.H;
    double v;
    if (MODE == F_DIV) v = a[i] / b[i];
    else if (MODE == F_XDC) v = a[i] * b[i];
    else v = a[i];
    vpad[exl * fp.fplane + (long long)(ez + fp.R) * fp.FY + ey + fp.R] = v;
  }
}

template <int MODE>
__global__ void __launch_bounds__(kBlock)
k_filt_apply(Geo g, FiltPad fp, int nst, const double* __restrict__ vpad, const double* __restrict__ a,
             const double* __restrict__ hs, const uint8_t* __restrict__ passive, double* __restrict__ out) {
  pdl_enter();
  const long long b0 = (long long)g.H * g.eplane, e0 = (long long)(g.H + g.nex) * g.eplane;
  for (long long i = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e0;
       i += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    if (!decode_elem(g, i, ex, ey, ez)) continue;
    const long long ip = (long long)(ex - g.ex0 + g.H) * fp.fplane + (long long)(ez + fp.R) * fp.FY + ey + fp.R;
    double s = 0.0;
    for (int k = 0; k < nst; ++k) s = fma(c_st_w[k], vpad[ip + c_st_poff[k]], s);
    double r;
    if (MODE == F_DIV) r = s;
    else if (MODE == F_XDC) r = s / (hs[i] * fmax(1e-3, a[i]));
    else r = s / hs[i];
    if (MODE == F_X0 && passive[i]) r = passive[i] == kSolid ? 1.0 : 0.0;   // R14, R27
    out[i] = r;
  }
}

// ===========================================================================
// A7  OC bisection (§2.3).  xnew(lambda) = max(0, x-m, min(1, x+m,
// x sqrt(max(0, -dc~/(dv~ lambda))))); mode 0 volume V = sum_j dv~_j xnew_j
// (= sum_{i in D} xPhys_i, H symmetric; R26), modes 1/2 V = sum_{j in D}
// xnew_j.
//  * k_oc_prep stores A = x sqrt(max(0, -dc~/dv~)) once (0 on passive elements
//    and pads), so a candidate is A / sqrt(lambda) and a pass needs no division,
//    square root, index decode or passive mask (x = A = 0 there gives xnew = 0).
//  * One pass evaluates the 7 midpoints of the next 3 bisection levels (heap
//    order) and the last block walks the tree exactly as the sequential loop
//    would (same lmid arithmetic, same strict V > target test, stop on the
//    bracket tolerance), so ~80 passes become ~27.
// ===========================================================================
constexpr int kOcCand = 7;

__device__ __forceinline__ double oc_xnew(double x, double A, double s, double move) {
  return fmax(0.0, fmax(x - move, fmin(1.0, fmin(x + move, A * s))));
}

// heap-ordered midpoints lam[1..7] of 3 bisection levels below the bracket [l1, l2]
__device__ __forceinline__ void oc_tree(double l1, double l2, double lam[kOcCand + 1]) {
  double a[kOcCand + 1], b[kOcCand + 1];
  a[1] = l1;
  b[1] = l2;
#pragma unroll
  for (int k = 1; k <= kOcCand; ++k) {
    lam[k] = 0.5 * (b[k] + a[k]);
    if (2 * k <= kOcCand) {
      a[2 * k] = a[k];          // V <= target: l2 = lmid
      b[2 * k] = lam[k];
      a[2 * k + 1] = lam[k];    // V > target: l1 = lmid
      b[2 * k + 1] = b[k];
    }
  }
}

__device__ __forceinline__ void oc_walk(DevState* st, const double* V) {
  double lam[kOcCand + 1];
  oc_tree(st->l1, st->l2, lam);
  int k = 1;
  for (int lvl = 0; lvl < 3 && st->oc_active; ++lvl) {
    st->lmid = lam[k];
    st->vol = V[k - 1];
    if (V[k - 1] > st->target) {
      st->l1 = lam[k];
      k = 2 * k + 1;
    } else {
      st->l2 = lam[k];
      k = 2 * k;
    }
    st->oc_pass += 1;
    st->oc_active = ((st->l2 - st->l1) / (st->l1 + st->l2) > st->oc_tol) ? 1 : 0;
  }
}

__global__ void __launch_bounds__(kBlock)
k_oc_prep(Geo g, const double* __restrict__ x, const double* __restrict__ dcf, const double* __restrict__ dvf,
          const uint8_t* __restrict__ passive, double* __restrict__ A) {
  pdl_enter();
  const long long b0 = (long long)g.H * g.eplane, e0 = (long long)(g.H + g.nex) * g.eplane;
  for (long long i = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e0;
       i += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    const bool in = decode_elem(g, i, ex, ey, ez);
    const uint8_t pv = in ? passive[i] : 0;
    // passive solid (R27): A = +inf makes every candidate clamp(A s, lo, hi) = 1
    // (s = 1/sqrt(lambda) > 0, hi = min(1, 1 + m) = 1), in the full, frozen and
    // compacted passes alike; void / pads: x = A = 0 gives xnew = 0
    A[i] = !in ? 0.0 : pv == kSolid ? (double)INFINITY : pv ? 0.0 : x[i] * sqrt(fmax(0.0, -dcf[i] / dvf[i]));
  }
}

template <int MODE0>
__global__ void __launch_bounds__(kBlock)
k_oc_pass(Geo g, DevState* st, double move, const double* __restrict__ x, const double* __restrict__ A,
          const double* __restrict__ dvf, double* partials, unsigned int* counter, int finish) {
  pdl_enter();
  if (!st->oc_active) return;
  double lam[kOcCand + 1], sc[kOcCand], vol[kOcCand];
  oc_tree(st->l1, st->l2, lam);
#pragma unroll
  for (int k = 0; k < kOcCand; ++k) {
    sc[k] = 1.0 / sqrt(lam[k + 1]);
    vol[k] = 0.0;
  }
  // element pairs (double2: b0 and the plane size are even, so pairs are
  // 16-byte aligned); 2 pairs per trip with all 6 vector loads issued before
  // any use (the pass is latency-bound otherwise).  An out-of-range pair reads
  // pair 0 and is weighted by 0.
  const unsigned b0 = (unsigned)(g.H * g.eplane), e0 = (unsigned)((g.H + g.nex) * g.eplane);
  const unsigned np = (e0 - b0) / 2;        // (e0 - b0) = nex * eplane is even
  const unsigned stride = gridDim.x * blockDim.x;
  const double2* x2 = reinterpret_cast<const double2*>(x + b0);
  const double2* a2 = reinterpret_cast<const double2*>(A + b0);
  const double2* d2 = reinterpret_cast<const double2*>(dvf + b0);
  for (unsigned p0 = blockIdx.x * blockDim.x + threadIdx.x; p0 < np; p0 += 2 * stride) {
    double2 xv[2], av[2], dv[2];
    double wv[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const unsigned pj = p0 + j * stride;
      const bool ok = pj < np;
      const unsigned q = ok ? pj : 0u;
      xv[j] = __ldg(x2 + q);
      av[j] = __ldg(a2 + q);
      dv[j] = MODE0 ? __ldg(d2 + q) : make_double2(1.0, 1.0);
      wv[j] = ok ? 1.0 : 0.0;
    }
    // L2 prefetch of the next trip's pairs (ptxas sinks the second pair's loads
    // behind the first pair's compute; the prefetches keep DRAM busy meanwhile)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const unsigned pn = p0 + (2 + j) * stride;
      if (pn < np) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x2 + pn));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a2 + pn));
        if (MODE0) asm volatile("prefetch.global.L2 [%0];" ::"l"(d2 + pn));
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      // lambda-independent clamp bounds: xnew = min(hi, max(lo, A s)) (= oc_xnew exactly)
      const double lo0 = fmax(0.0, xv[j].x - move), hi0 = fmin(1.0, xv[j].x + move);
      const double lo1 = fmax(0.0, xv[j].y - move), hi1 = fmin(1.0, xv[j].y + move);
      const double w0 = wv[j] * dv[j].x, w1 = wv[j] * dv[j].y;
#pragma unroll
      for (int k = 0; k < kOcCand; ++k) {
        vol[k] = fma(w0, fmin(hi0, fmax(lo0, av[j].x * sc[k])), vol[k]);
        vol[k] = fma(w1, fmin(hi1, fmax(lo1, av[j].y * sc[k])), vol[k]);
      }
    }
  }
  __shared__ double tot[kOcCand];
  if (grid_reduce<kOcCand>(vol, partials, counter, tot) && threadIdx.x == 0) {
    if (finish) oc_walk(st, tot);
    else
      for (int k = 0; k < kOcCand; ++k) st->sums[k] = tot[k];
  }
}
// ---------------------------------------------------------------------------
// OC frozen set: once the bracket [l1, l2] (l1 > 0) is narrow, s = 1/sqrt(lambda)
// stays in [1/sqrt(l2), 1/sqrt(l1)] for every lambda the bisection can still
// evaluate, and an element's xnew = clamp(A s, lo, hi) is either
//   fixed at lo (A s_hi <= lo) or at hi (A s_lo >= hi): a constant, or
//   unclamped (lo <= A s_lo, A s_hi <= hi): linear in s, dv~ A s,
//   or crossing a bound inside the bracket (active).
// F = sum of the constants and G = sum dv~ A over the linear class are formed
// once; the active elements are compacted (in element order) and later passes
// evaluate V(s) = F + s G + sum_active -- the same terms as the full sum up to
// the order of the additions.  Applied twice (two nested brackets) with
// ping-pong arrays.  Block b owns the contiguous chunk [b chunk, (b+1) chunk),
// so the compaction order is deterministic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int oc_class(double x, double A, double move, double slo, double shi) {
  const double lo = fmax(0.0, x - move), hi = fmin(1.0, x + move);
  if (A * shi <= lo) return 0;                   // fixed at lo
  if (A * slo >= hi) return 1;                   // fixed at hi
  if (lo <= A * slo && A * shi <= hi) return 2;  // unclamped: linear in s
  return 3;                                      // crossing: active
}

template <int MODE0>
__global__ void __launch_bounds__(kBlock)
k_oc_freeze(long long n0, const long long* __restrict__ nptr, const double* __restrict__ x, const double* __restrict__ A,
            const double* __restrict__ dvf, DevState* st, double move, unsigned chunk,
            unsigned* __restrict__ counts, double* partials, unsigned int* counter) {
  pdl_enter();
  const double slo = 1.0 / sqrt(st->l2), shi = 1.0 / sqrt(st->l1);
  const long long n = nptr ? *nptr : n0;   // stage 2 reads the stage-1 active count on the device
  const long long c0 = (long long)blockIdx.x * chunk, c1 = min(n, c0 + (long long)chunk);
  double fz = 0.0, lin = 0.0;
  unsigned na = 0;
  for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const double xv = x[i], av = A[i], dv = MODE0 ? dvf[i] : 1.0;
    const int c = oc_class(xv, av, move, slo, shi);
    if (c == 3) ++na;
    else if (c == 2) lin = fma(dv, av, lin);
    else fz = fma(dv, c == 0 ? fmax(0.0, xv - move) : fmin(1.0, xv + move), fz);
  }
  __shared__ unsigned cnt_sh;
  if (threadIdx.x == 0) cnt_sh = 0;
  __syncthreads();
  atomicAdd(&cnt_sh, na);   // integer: order-independent
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = cnt_sh;
  __shared__ double tot[2];
  double v[2] = {fz, lin};
  if (grid_reduce<2>(v, partials, counter, tot) && threadIdx.x == 0) {
    st->oc_frozen += tot[0];
    st->oc_lin += tot[1];
  }
}

// exclusive scan of the per-block active counts (one thread; nb <= a few thousand)
__global__ void k_oc_scan(const unsigned* __restrict__ counts, int nb, unsigned* __restrict__ offs, DevState* st) {
  pdl_enter();
  if (threadIdx.x != 0) return;
  unsigned long long run = 0;
  for (int b = 0; b < nb; ++b) {
    offs[b] = (unsigned)run;
    run += counts[b];
  }
  st->oc_nact = (long long)run;
}

// compaction in element order: tiles of blockDim elements, block-wide scan of the flags
template <int MODE0>
__global__ void __launch_bounds__(kBlock)
k_oc_compact(long long n0, const long long* __restrict__ nptr, const double* __restrict__ x, const double* __restrict__ A,
             const double* __restrict__ dvf, const DevState* st, double move, unsigned chunk,
             const unsigned* __restrict__ offs, double* __restrict__ cx, double* __restrict__ cA,
             double* __restrict__ cdv) {
  pdl_enter();
  const double slo = 1.0 / sqrt(st->l2), shi = 1.0 / sqrt(st->l1);
  const long long n = nptr ? *nptr : n0;   // stage 2 reads the stage-1 active count on the device
  const long long c0 = (long long)blockIdx.x * chunk, c1 = min(n, c0 + (long long)chunk);
  __shared__ unsigned wsum[kBlock / 32];
  unsigned base = offs[blockIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long t0 = c0; t0 < c1; t0 += blockDim.x) {
    const long long i = t0 + threadIdx.x;
    double xv = 0.0, av = 0.0, dv = 0.0;
    bool act = false;
    if (i < c1) {
      xv = x[i];
      av = A[i];
      dv = MODE0 ? dvf[i] : 1.0;
      act = oc_class(xv, av, move, slo, shi) == 3;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    unsigned before = 0, total = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      if (k < w) before += wsum[k];
      total += wsum[k];
    }
    if (act) {
      const unsigned o = base + before + __popc(bal & ((1u << lane) - 1u));
      cx[o] = xv;
      cA[o] = av;
      cdv[o] = dv;
    }
    base += total;
    __syncthreads();
  }
}

// a bisection pass over the compacted active elements: V(s) = F + s G + sum_active
__global__ void __launch_bounds__(kBlock)
k_oc_pass_c(DevState* st, double move, const double* __restrict__ cx, const double* __restrict__ cA,
            const double* __restrict__ cdv, double* partials, unsigned int* counter, int finish) {
  pdl_enter();
  if (!st->oc_active) return;
  double lam[kOcCand + 1], sc[kOcCand], vol[kOcCand];
  oc_tree(st->l1, st->l2, lam);
#pragma unroll
  for (int k = 0; k < kOcCand; ++k) {
    sc[k] = 1.0 / sqrt(lam[k + 1]);
    vol[k] = 0.0;
  }
  const long long n = st->oc_nact;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double xv = cx[i], av = cA[i], dv = cdv[i];
    const double lo = fmax(0.0, xv - move), hi = fmin(1.0, xv + move);
#pragma unroll
    for (int k = 0; k < kOcCand; ++k) vol[k] = fma(dv, fmin(hi, fmax(lo, av * sc[k])), vol[k]);
  }
  __shared__ double tot[kOcCand];
  if (grid_reduce<kOcCand>(vol, partials, counter, tot) && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kOcCand; ++k) tot[k] += fma(sc[k], st->oc_lin, st->oc_frozen);
    if (finish) oc_walk(st, tot);
    else
      for (int k = 0; k < kOcCand; ++k) st->sums[k] = tot[k];
  }
}

// ---------------------------------------------------------------------------
// OC phase 1 in two passes.  While l1 = 0 the bisection evaluates exactly
// lmid_k = lmax 2^-k (k = 1, 2, ...) and moves l2 down until the first k* with
// V(lmid_k*) > target (V is monotone in lambda).  Two 7-candidate passes find
// k* (pass A: k = 8, 16, ..., 56; pass B: the 7 k's below the first hit) and the
// state jumps to where the sequential loop would be after k* steps: l1 =
// lmid_k*, l2 = lmid_(k*-1), lmid = lmid_k*, k* bisection steps counted.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int oc_gk(const DevState* st, int stage, int j) {
  return stage == 0 ? 8 * (j + 1) : st->oc_glo + 1 + j;
}

__device__ __forceinline__ void oc_gwalk(DevState* st, int stage, const double* V) {
  int hit = -1;
  for (int j = 0; j < kOcCand; ++j)
    if (V[j] > st->target) { hit = j; break; }
  if (stage == 0) {
    st->oc_glo = hit < 0 ? 8 * kOcCand : 8 * hit;
    st->oc_ghi = hit < 0 ? 0 : 8 * (hit + 1);
    st->oc_gvhi = hit < 0 ? 0.0 : V[hit];
    return;
  }
  int ks;
  double vs;
  if (hit >= 0) {
    ks = st->oc_glo + 1 + hit;
    vs = V[hit];
  } else if (st->oc_ghi > 0) {
    ks = st->oc_ghi;
    vs = st->oc_gvhi;
  } else {   // no crossing within k <= 63: take the 63 steps that moved l2 only
    const int k = st->oc_glo + kOcCand;
    st->l2 = ldexp(st->l2, -k);
    st->lmid = st->l2;
    st->vol = V[kOcCand - 1];
    st->oc_pass += k;
    return;
  }
  const double lmax = st->l2;
  st->l1 = ldexp(lmax, -ks);
  st->l2 = ks == 1 ? lmax : ldexp(lmax, -(ks - 1));
  st->lmid = st->l1;
  st->vol = vs;
  st->oc_pass += ks;
  st->oc_active = ((st->l2 - st->l1) / (st->l1 + st->l2) > st->oc_tol) ? 1 : 0;
}

template <int MODE0>
__global__ void __launch_bounds__(kBlock)
k_oc_gpass(Geo g, DevState* st, int stage, double move, const double* __restrict__ x, const double* __restrict__ A,
           const double* __restrict__ dvf, double* partials, unsigned int* counter, int finish) {
  pdl_enter();
  if (!st->oc_active) return;
  double sc[kOcCand], vol[kOcCand];
#pragma unroll
  for (int k = 0; k < kOcCand; ++k) {
    sc[k] = 1.0 / sqrt(ldexp(st->l2, -oc_gk(st, stage, k)));   // l2 = lmax during phase 1
    vol[k] = 0.0;
  }
  const unsigned b0 = (unsigned)(g.H * g.eplane), e0 = (unsigned)((g.H + g.nex) * g.eplane);
  for (unsigned i = b0 + blockIdx.x * blockDim.x + threadIdx.x; i < e0; i += gridDim.x * blockDim.x) {
    const double xv = x[i], av = A[i], dv = MODE0 ? dvf[i] : 1.0;
    const double lo = fmax(0.0, xv - move), hi = fmin(1.0, xv + move);
#pragma unroll
    for (int k = 0; k < kOcCand; ++k) vol[k] = fma(dv, fmin(hi, fmax(lo, av * sc[k])), vol[k]);
  }
  __shared__ double tot[kOcCand];
  if (grid_reduce<kOcCand>(vol, partials, counter, tot) && threadIdx.x == 0) {
    if (finish) oc_gwalk(st, stage, tot);
    else
      for (int k = 0; k < kOcCand; ++k) st->sums[k] = tot[k];
  }
}
__global__ void k_oc_gfinish(DevState* st, int stage) {
  pdl_enter();
  if (!st->oc_active) return;
  oc_gwalk(st, stage, st->sums);
}

__global__ void k_oc_finish(DevState* st) {
  pdl_enter();
  if (!st->oc_active) return;
  oc_walk(st, st->sums);
}

// final: xnew at the last evaluated lmid, change = max |xnew - x| over design
// elements, design-volume sum of xnew (passive elements skipped; pads give 0).
__global__ void __launch_bounds__(kBlock)
k_oc_final(Geo g, DevState* st, double move, const double* __restrict__ x, const double* __restrict__ A,
           const uint8_t* __restrict__ passive, double* __restrict__ xnew, double* partials, unsigned int* counter) {
  pdl_enter();
  const double lmid = st->lmid;   // the last evaluated midpoint
  const int any = st->oc_pass > 0;
  const double sc = any ? 1.0 / sqrt(lmid) : 0.0;
  const unsigned b0 = (unsigned)(g.H * g.eplane), e0 = (unsigned)((g.H + g.nex) * g.eplane);
  double chg = 0.0, vsum = 0.0;
  for (unsigned i = b0 + blockIdx.x * blockDim.x + threadIdx.x; i < e0; i += gridDim.x * blockDim.x) {
    const double xo = x[i];
    const double xn = any ? oc_xnew(xo, A[i], sc, move) : xo;
    xnew[i] = xn;
    if (passive[i]) continue;   // design elements only (passive solid holds 1, R27)
    chg = fmax(chg, fabs(xn - xo));
    vsum += xn;
  }
  __shared__ double tot[2];
  double v[2] = {vsum, chg};
  if (grid_reduce<2, 1>(v, partials, counter, tot) && threadIdx.x == 0) {
    st->sums[2] = tot[0];
    st->sums[3] = tot[1];
  }
}

// sum over owned elements of class `want` (0 design, kSolid ...) of a field
// (design volume of xPhys; the passive-solid volume floor sum dv~ over solid)
__global__ void __launch_bounds__(kBlock)
k_design_sum(Geo g, DevState* st, const double* __restrict__ a, const uint8_t* __restrict__ passive,
             int slot, double* partials, unsigned int* counter, int want = 0) {
  pdl_enter();
  const long long b0 = (long long)g.H * g.eplane, e0 = (long long)(g.H + g.nex) * g.eplane;
  double s = 0.0;
  for (long long i = b0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e0;
       i += (long long)gridDim.x * blockDim.x) {
    int ex, ey, ez;
    if (!decode_elem(g, i, ex, ey, ez) || passive[i] != want) continue;
    s += a[i];
  }
  __shared__ double tot[1];
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter, tot) && threadIdx.x == 0) st->sums[slot] = tot[0];
}

// ---------------------------------------------------------------------------
// Layout kernels: external (host order) <-> internal, for the owned range.
// ---------------------------------------------------------------------------
// nodes: ext[3*n + c] <-> SoA internal, for the owned node planes [ix0, ix0+nix).
// ext_global = 0: ext holds only that sub-block in external order (iz, ix, iy)
// (host staging); 1: ext is the whole external array (S:45 numbering, device
// pointer of a _d call) and n is the node's global external index.
__device__ __forceinline__ long long ext_node(const Geo& g, long long k, int ixr, int iy, int iz, int ix0,
                                              int ext_global) {
  return ext_global ? (long long)iz * (g.nelx + 1) * (g.nely + 1) + (long long)(ix0 + ixr) * (g.nely + 1) + iy : k;
}
__global__ void k_nodes_in(Geo g, const double* __restrict__ ext, double* __restrict__ in, int ix0,
                           int nix, int ext_global) {
  pdl_enter();
  const long long tot = (long long)nix * (g.nelz + 1) * (g.nely + 1);
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    // k enumerates the external sub-block in external order (iz, ix, iy)
    const int iy = (int)(k % (g.nely + 1));
    const long long t = k / (g.nely + 1);
    const int ixr = (int)(t % nix), iz = (int)(t / nix);
    const long long i = node_idx(g, ix0 + ixr, iy, iz), e = ext_node(g, k, ixr, iy, iz, ix0, ext_global);
#pragma unroll
    for (int c = 0; c < 3; ++c) in[i + c * g.ncomp] = ext[3 * e + c];
  }
}
__global__ void k_nodes_out(Geo g, const double* __restrict__ in, double* __restrict__ ext, int ix0,
                            int nix, int ext_global) {
  pdl_enter();
  const long long tot = (long long)nix * (g.nelz + 1) * (g.nely + 1);
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    const int iy = (int)(k % (g.nely + 1));
    const long long t = k / (g.nely + 1);
    const int ixr = (int)(t % nix), iz = (int)(t / nix);
    const long long i = node_idx(g, ix0 + ixr, iy, iz), e = ext_node(g, k, ixr, iy, iz, ix0, ext_global);
#pragma unroll
    for (int c = 0; c < 3; ++c) ext[3 * e + c] = in[i + c * g.ncomp];
  }
}
// per-node scalar (Jacobi inverse diagonal) -> per-DOF external array, 0 on fixed DOFs
__global__ void k_invd_out(Geo g, const double* __restrict__ in, const uint8_t* __restrict__ fixm,
                           double* __restrict__ ext, int ix0, int nix, int ext_global) {
  pdl_enter();
  const long long tot = (long long)nix * (g.nelz + 1) * (g.nely + 1);
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    const int iy = (int)(k % (g.nely + 1));
    const long long t = k / (g.nely + 1);
    const int ixr = (int)(t % nix), iz = (int)(t / nix);
    const long long i = node_idx(g, ix0 + ixr, iy, iz), e = ext_node(g, k, ixr, iy, iz, ix0, ext_global);
    const uint8_t fm = fixm[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) ext[3 * e + c] = (fm >> c) & 1 ? 0.0 : in[i];
  }
}
// elements: ext[(ez*nex + exr)*nely + ey] (owned sub-block, ext_global = 0) or
// ext[ez*nelx*nely + ex*nely + ey] (whole external array, ext_global = 1)
__device__ __forceinline__ long long ext_elem(const Geo& g, long long k, int exr, int ey, int ez, int ext_global) {
  return ext_global ? (long long)ez * g.nelx * g.nely + (long long)(g.ex0 + exr) * g.nely + ey : k;
}
__global__ void k_elems_in(Geo g, const double* __restrict__ ext, double* __restrict__ in, int ext_global) {
  pdl_enter();
  const long long tot = (long long)g.nex * g.nelz * g.nely;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    const int ey = (int)(k % g.nely);
    const long long t = k / g.nely;
    const int exr = (int)(t % g.nex), ez = (int)(t / g.nex);
    in[elem_idx(g, g.ex0 + exr, ey, ez)] = ext[ext_elem(g, k, exr, ey, ez, ext_global)];
  }
}
__global__ void k_elems_out(Geo g, const double* __restrict__ in, double* __restrict__ ext, int ext_global) {
  pdl_enter();
  const long long tot = (long long)g.nex * g.nelz * g.nely;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < tot;
       k += (long long)gridDim.x * blockDim.x) {
    const int ey = (int)(k % g.nely);
    const long long t = k / g.nely;
    const int exr = (int)(t % g.nex), ez = (int)(t / g.nex);
    ext[ext_elem(g, k, exr, ey, ez, ext_global)] = in[elem_idx(g, g.ex0 + exr, ey, ez)];
  }
}

// loopback allreduce: dst[g]->sums[k] = sum_g src ... (fixed slab order)
struct StatePtrs { DevState* s[16]; };
__global__ void k_slab_allreduce(StatePtrs sp, int nslab, int k0, int nk, int maxmask) {
  pdl_enter();
  // thread t owns slot k0+t: reads it on every slab, then writes it back
  const int k = k0 + threadIdx.x;
  if (threadIdx.x >= nk) return;
  double a = sp.s[0]->sums[k];
  const bool mx = (maxmask >> threadIdx.x) & 1;
  for (int s = 1; s < nslab; ++s) {
    const double v = sp.s[s]->sums[k];
    a = mx ? fmax(a, v) : a + v;
  }
  for (int s = 0; s < nslab; ++s) sp.s[s]->sums[k] = a;
}

}  // namespace topo

namespace topo {
// ---------------------------------------------------------------------------
// small state / utility kernels
// ---------------------------------------------------------------------------
__global__ void k_cg_init(DevState* st, double tol2, double bb, long long max_it) {
  pdl_enter();
  st->pending = 0;
  st->alpha_prev = 0.0;
  st->solo = tol2 < 0.0;   // TOPO_DIST_SOLO: a fixed iteration count, never a breakdown exit
  st->tol2 = tol2;
  st->bb = bb;
  st->max_it = max_it;
  st->it = 0;
  st->status = 0;
  st->fresh = 1;
  st->done = 0;
  st->alpha = st->beta = 0.0;
}
// after k_residual(write_r) + allreduce: rz, rr from sums; restart semantics
__global__ void k_cg_start(DevState* st) {
  pdl_enter();
  st->rz = st->sums[0];
  st->rr = st->sums[1];
  st->fresh = 1;
  st->status = 0;
  st->done = (!st->solo && st->rr <= st->tol2 * st->bb) ? 1 : 0;
}
__global__ void k_oc_init(DevState* st, double lmax, double target, double tol) {
  pdl_enter();
  st->l1 = 0.0;
  st->l2 = lmax;
  st->target = target;
  st->oc_tol = tol;
  st->oc_pass = 0;
  st->vol = 0.0;
  st->oc_frozen = 0.0;
  st->oc_lin = 0.0;
  st->oc_nact = 0;
  st->oc_glo = st->oc_ghi = 0;
  st->oc_gvhi = 0.0;
  st->oc_active = ((st->l2 - st->l1) / (st->l1 + st->l2) > tol) ? 1 : 0;
  st->lmid = 0.5 * (st->l2 + st->l1);
}
// zero the fixed DOFs of a node vector (owned planes)
__global__ void k_mask_fixed(Geo g, const uint8_t* __restrict__ fixm, double* __restrict__ v) {
  pdl_enter();
  const long long b = g.nplane, e = (long long)(g.nown + 1) * g.nplane;
  for (long long i = b + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e;
       i += (long long)gridDim.x * blockDim.x) {
    const uint8_t fm = fixm[i];
    if (!fm) continue;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if ((fm >> c) & 1) v[i + c * g.ncomp] = 0.0;
  }
}
// a = v * dv over the whole local element array (x0 = volfrac on design elements)
__global__ void k_fill_design(Geo g, const double* __restrict__ dv, double v, double* __restrict__ a) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.nelloc;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = v * dv[i];
}
// force passive elements to their value (0 void, 1 solid; R27) over the whole local element array
__global__ void k_apply_passive(Geo g, const uint8_t* __restrict__ passive, double* __restrict__ a) {
  pdl_enter();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.nelloc;
       i += (long long)gridDim.x * blockDim.x)
    if (passive[i]) a[i] = passive[i] == kSolid ? 1.0 : 0.0;
}
}  // namespace topo
