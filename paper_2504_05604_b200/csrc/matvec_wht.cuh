// A2 (+A3/A4 fusion): element-centric, x-marching EbE matvec on the exact
// Walsh-Hadamard block form of KE.
//
// KE = H^T B H, where H is the unnormalised tensor-product (+-1) transform of
// the 8 element corners (per displacement component) and B = H KE H^T / 64 is
// block-diagonal with eight 3x3 blocks indexed by the parity pi = m ^ e_c of
// (component c, mode m) (verified on the host at init).  With
// cubic symmetry the blocks have only 8 distinct entries:
//   pi = 000, 111 : full, diag d, off-diag o    -> Q_i = (d-o) P_i + o (P_0+P_1+P_2)
//   pi = one bit  : translation row is 0, 2x2 [[a,b],[b,a]]
//   pi = two bits : 2x2 [[r,r],[r,r]] plus a singleton s
// so q_e = E_e H^T B H p_e costs ~175 fp64 ops instead of 576 DFMA.
//
// Mapping: a CTA of 32 (y) x TZ (z) threads owns 31 x (TZ-1) nodes of a y-z
// tile and marches along x over a chunk of node planes.  Thread (ty,tz)
// handles the element column (y0-1+ty, z0-1+tz) and owns its base node
// (y0-1+ty, z0-1+tz) when ty,tz >= 1.  The y-z transform of a node plane
// (4 corners) is computed once and shared by the two elements left and right
// of the plane (x stage = sum/difference of consecutive planes); element
// contributions to a node plane are accumulated in the transformed domain,
// inverse-transformed once per plane, and summed over the 4 elements of the
// y-z neighbourhood with one shuffle pair (y) and one shared-memory exchange
// (z).  Every output node is written by exactly one thread; sums are in a
// fixed order (deterministic).
//
// kFused: p_new = M^{-1} r + beta p_old is computed while loading (Jacobi
// preconditioner + PCG direction update, A3/A4), written once by the owner,
// and the matvec runs on p_new; p_old / p_new are ping-pong buffers.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace topo {

struct WhtK { double k0, o0, k7, o7, a, b, r, s; };
__constant__ WhtK c_wht;

__device__ __forceinline__ void wht4(const double v[4], double G[4]) {
  // G[k], k = my + 2 mz, from corners v[a], a = ay + 2 az
  const double s0 = v[0] + v[1], d0 = v[0] - v[1], s1 = v[2] + v[3], d1 = v[2] - v[3];
  G[0] = s0 + s1;
  G[1] = d0 + d1;
  G[2] = s0 - s1;
  G[3] = d0 - d1;
}

// Q = E * B * P  (P, Q indexed [c][m], m = mx + 2 my + 4 mz)
__device__ __forceinline__ void wht_block(const double P[3][8], double Ee, double Q[3][8]) {
  const WhtK& K = c_wht;
  double t;
  t = K.o0 * (P[0][1] + P[1][2] + P[2][4]);
  Q[0][1] = fma(K.k0, P[0][1], t);
  Q[1][2] = fma(K.k0, P[1][2], t);
  Q[2][4] = fma(K.k0, P[2][4], t);
  t = K.o7 * (P[0][6] + P[1][5] + P[2][3]);
  Q[0][6] = fma(K.k7, P[0][6], t);
  Q[1][5] = fma(K.k7, P[1][5], t);
  Q[2][3] = fma(K.k7, P[2][3], t);
  Q[0][0] = Q[1][0] = Q[2][0] = 0.0;   // rigid translations carry no energy
  Q[1][3] = fma(K.a, P[1][3], K.b * P[2][5]);
  Q[2][5] = fma(K.b, P[1][3], K.a * P[2][5]);
  Q[0][3] = fma(K.a, P[0][3], K.b * P[2][6]);
  Q[2][6] = fma(K.b, P[0][3], K.a * P[2][6]);
  Q[0][5] = fma(K.a, P[0][5], K.b * P[1][6]);
  Q[1][6] = fma(K.b, P[0][5], K.a * P[1][6]);
  t = K.r * (P[0][2] + P[1][1]);
  Q[0][2] = t;
  Q[1][1] = t;
  Q[2][7] = K.s * P[2][7];
  t = K.r * (P[0][4] + P[2][1]);
  Q[0][4] = t;
  Q[2][1] = t;
  Q[1][7] = K.s * P[1][7];
  t = K.r * (P[1][4] + P[2][2]);
  Q[1][4] = t;
  Q[2][2] = t;
  Q[0][7] = K.s * P[0][7];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 1; m < 8; ++m) Q[c][m] *= Ee;
}

// Tensor maps of one matvec launch (TMA descriptors, kernel-parameter space).
struct MvMaps {
  CUtensorMap vin;    // 4D {NY, NZ, NXL, 3}: p (plain) or r (fused)
  CUtensorMap pold;   // 4D, fused only
  CUtensorMap invd;   // 3D {NY, NZ, NXL}, fused only
  CUtensorMap E;      // 3D {EY, EZ, NEXL}
};

constexpr int kMvStages = 4;
template <int TZ> struct MvSmem {
  static constexpr int YW = 34;                                   // 33 nodes, box width padded to 16 B
  static constexpr int V = 3 * (TZ + 1) * YW * 8;                 // bytes of one 3-component node tile
  static constexpr int I = (TZ + 1) * YW * 8;                     // one scalar node tile
  static constexpr int EB = TZ * YW * 8;                          // element tile (box width 34 as well)
  static constexpr int VA = (V + 127) / 128 * 128, IA = (I + 127) / 128 * 128, EA = (EB + 127) / 128 * 128;
  __host__ __device__ static constexpr int stage(bool fused) { return fused ? 2 * VA + IA + EA : VA + EA; }
  __host__ __device__ static constexpr int bytes(bool fused) { return kMvStages * stage(fused) + 128; }
};

template <int TZ, bool kFused, bool kDot>
__global__ void __launch_bounds__(32 * TZ, (TZ <= 8 ? 2 : 1))
k_mv_wht(const __grid_constant__ MvMaps maps, Geo g, DevState* st, int gate, int CX,
         const uint8_t* __restrict__ fixm, double* __restrict__ pnew, double* __restrict__ q,
         double* partials, unsigned int* counter, int finish) {
  if (gate && st->done) return;
  using L = MvSmem<TZ>;
  const double beta = (kFused && !st->fresh) ? st->beta : 0.0;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ double xch[2][TZ][32][3];
  __shared__ __align__(8) uint64_t full[kMvStages];

  const int ty = threadIdx.x, tz = threadIdx.y;
  const bool leader = (ty == 0 && tz == 0);
  const int y0 = blockIdx.x * 31, z0 = blockIdx.y * (TZ - 1);   // stored coords of the tile's (ty,tz) = (0,0)
  // TMA boxes start at an even stored y (16-byte aligned row start); yoff in {0,1}
  const int yb = y0 & ~1, yoff = y0 - yb;
  const int iyb = y0 - 1 + ty, izb = z0 - 1 + tz;                 // base node of this thread
  const int chunk = blockIdx.z;
  const int xend_slab = g.ex0 + g.nown;
  const int xs = g.ex0 + chunk * CX;
  const int xe = min(xs + CX, xend_slab);
  const bool first_chunk = chunk == 0, last_chunk = (xe == xend_slab);
  const bool owned = ty >= 1 && tz >= 1 && iyb <= g.nely && izb <= g.nelz;
  const long long ob = (long long)(izb + 1) * g.NY + (iyb + 1);
  const long long ncomp = g.ncomp, nplane = g.nplane;
  const int nunits = xe - xs + 2;           // node planes xs-1 .. xe

  auto slot = [&](int s) { return dsm + s * L::stage(kFused); };
  auto issue = [&](int t) {                 // unit t: node plane j = xs-1+t, element plane j-1
    const int s = t % kMvStages;
    unsigned char* b = slot(s);
    const int j = xs - 1 + t;
    const int ixl = j - g.ex0 + 1;
    const uint32_t bytes = (kFused ? 2 * L::V + L::I : L::V) + (t > 0 ? L::EB : 0);
    mbar_arrive_expect_tx(&full[s], bytes);
    tma_load_4d(b, &maps.vin, &full[s], yb, z0, ixl, 0);
    if (kFused) {
      tma_load_4d(b + L::VA, &maps.pold, &full[s], yb, z0, ixl, 0);
      tma_load_3d(b + 2 * L::VA, &maps.invd, &full[s], yb, z0, ixl);
    }
    if (t > 0) tma_load_3d(b + (kFused ? 2 * L::VA + L::IA : L::VA), &maps.E, &full[s], yb, z0, j - 1 - g.ex0 + g.H);
  };
  if (leader) {
    tma_prefetch_desc(&maps.vin);
    tma_prefetch_desc(&maps.E);
    if (kFused) { tma_prefetch_desc(&maps.pold); tma_prefetch_desc(&maps.invd); }
    for (int s = 0; s < kMvStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (leader)
    for (int t = 0; t < min(kMvStages, nunits); ++t) issue(t);

  // corners (k = ay + 2 az) of this thread's element column from unit t; returns E_e
  auto consume = [&](int t, double v[3][4], double pb[3]) -> double {
    const int s = t % kMvStages;
    mbar_wait(&full[s], (uint32_t)((t / kMvStages) & 1));
    const double* sv = reinterpret_cast<const double*>(slot(s));
    const double* sp = reinterpret_cast<const double*>(slot(s) + L::VA);
    const double* si = reinterpret_cast<const double*>(slot(s) + 2 * L::VA);
    const double* se = reinterpret_cast<const double*>(slot(s) + (kFused ? 2 * L::VA + L::IA : L::VA));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int o = (tz + (k >> 1)) * L::YW + ty + yoff + (k & 1);
      const double iv = kFused ? si[o] : 1.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int oc = c * (TZ + 1) * L::YW + o;
        v[c][k] = kFused ? fma(beta, sp[oc], iv * sv[oc]) : sv[oc];
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) pb[c] = v[c][0];
    if (kFused) {
      const int j = xs - 1 + t;
      if (owned && ((j >= xs && j < xe) || (j == xs - 1 && first_chunk) || (j == xe && last_chunk))) {
        const long long i = (long long)(j - g.ex0 + 1) * nplane + ob;
#pragma unroll
        for (int c = 0; c < 3; ++c) pnew[i + c * ncomp] = v[c][0];
      }
    }
    return t > 0 ? se[tz * L::YW + ty + yoff] : 0.0;
  };
  auto release = [&](int t) {               // all threads have read unit t (caller synced)
    if (leader && t + kMvStages < nunits) {
      fence_proxy_async();
      issue(t + kMvStages);
    }
  };

  double G0[3][4], A[3][4], pb_prev[3];
  {
    double v[3][4];
    consume(0, v, pb_prev);
#pragma unroll
    for (int c = 0; c < 3; ++c) wht4(v[c], G0[c]);
    __syncthreads();
    release(0);
  }
  double dot = 0.0;
  int buf = 0;
  for (int t = 1; t < nunits; ++t) {
    const int ex = xs - 2 + t;              // element plane of this step (node planes ex, ex+1)
    double v[3][4], pb[3], G1[3][4];
    const double Ee = consume(t, v, pb);
#pragma unroll
    for (int c = 0; c < 3; ++c) wht4(v[c], G1[c]);
    double P[3][8], Q[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        P[c][2 * k] = G0[c][k] + G1[c][k];
        P[c][2 * k + 1] = G0[c][k] - G1[c][k];
      }
    wht_block(P, Ee, Q);
    if (ex >= xs) {
      // complete node plane ex: A (from element ex-1) + R0 (element ex)
      double C[3][4];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double Ac[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) Ac[k] = A[c][k] + (Q[c][2 * k] + Q[c][2 * k + 1]);
        wht4(Ac, C[c]);
      }
      // y-z neighbourhood: owner(ty,tz) = C0(ty,tz) + C1(ty-1,tz) + C2(ty,tz-1) + C3(ty-1,tz-1)
      double S[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double T = C[c][2] + __shfl_up_sync(0xffffffffu, C[c][3], 1);
        S[c] = C[c][0] + __shfl_up_sync(0xffffffffu, C[c][1], 1);
        xch[buf][tz][ty][c] = T;
      }
      __syncthreads();
      release(t);
      if (owned) {
        const long long i = (long long)(ex - g.ex0 + 1) * nplane + ob;
        const uint8_t fm = fixm[i];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double qv = (fm >> c) & 1 ? 0.0 : S[c] + xch[buf][tz - 1][ty][c];
          q[i + c * ncomp] = qv;
          if (kDot) dot = fma(pb_prev[c], qv, dot);
        }
      }
      buf ^= 1;
    } else {
      __syncthreads();
      release(t);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        A[c][k] = Q[c][2 * k] - Q[c][2 * k + 1];   // R1: element ex -> node plane ex+1
        G0[c][k] = G1[c][k];
      }
      pb_prev[c] = pb[c];
    }
  }

  if (kDot) {
    __shared__ double tot[1];
    double vv[1] = {dot};
    if (grid_reduce<1>(vv, partials, counter, tot) && leader) {
      if (finish) {
        st->pq = tot[0];
        if (!(tot[0] > 0.0) || !isfinite(tot[0])) {
          st->status = 3;
          st->done = 1;
        } else {
          st->alpha = st->rz / tot[0];
        }
      } else {
        st->sums[0] = tot[0];
      }
    }
  }
}

}  // namespace topo
