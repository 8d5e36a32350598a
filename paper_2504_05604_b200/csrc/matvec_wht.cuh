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
// kPre (PCG direction update fused into the load, A3/A4; p_new is written
// once by the owner and the matvec runs on it; p_old / p_new are ping-pong):
//   kPre = 0: plain q = K v
//   kPre = 1: p_new = M^{-1} r + beta p_old   (Jacobi preconditioner, vin = r)
//   kPre = 2: p_new = z + beta p_old          (z = V(r) from the multigrid
//             preconditioner already in HBM, vin = z; no M^{-1} stream)
//   kPre = 3: p_new = w M^{-1} b               (first damped-Jacobi sweep of the
//             multigrid V-cycle from x = 0, w = *scale; vin = b)
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace topo {

template <typename T> struct WhtKT { T k0, o0, k7, o7, a, b, r, s; };
using WhtK = WhtKT<double>;
__constant__ WhtK c_wht;

template <typename T>
__device__ __forceinline__ void wht4(const T v[4], T G[4]) {
  // G[k], k = my + 2 mz, from corners v[a], a = ay + 2 az
  const T s0 = v[0] + v[1], d0 = v[0] - v[1], s1 = v[2] + v[3], d1 = v[2] - v[3];
  G[0] = s0 + s1;
  G[1] = d0 + d1;
  G[2] = s0 - s1;
  G[3] = d0 - d1;
}

// Q = E * B * P  (P, Q indexed [c][m], m = mx + 2 my + 4 mz).  E is folded
// into the 8 block constants (8 DMUL) instead of scaling the 21 outputs.
// Lambda^-1 B Lambda^-1, Lambda = diag(2^|m|): level-1 multigrid (mg.cuh), fp64 and fp32
__constant__ WhtK c_wht1;
__constant__ WhtKT<float> c_wht1f;
__constant__ WhtKT<float> c_whtf;   // c_wht in fp32: the multigrid smoothing matvecs with mg_fp32

template <typename T>
__device__ __forceinline__ void wht_block_k(const WhtKT<T>& K, const T P[3][8], T Ee, T Q[3][8]);
__device__ __forceinline__ void wht_block(const double P[3][8], double Ee, double Q[3][8]) {
  wht_block_k<double>(c_wht, P, Ee, Q);
}
__device__ __forceinline__ void wht_block(const float P[3][8], float Ee, float Q[3][8]) {
  wht_block_k<float>(c_whtf, P, Ee, Q);
}
template <typename T>
__device__ __forceinline__ void wht_block_k(const WhtKT<T>& K, const T P[3][8], T Ee, T Q[3][8]) {
  const T k0 = Ee * K.k0, o0 = Ee * K.o0, k7 = Ee * K.k7, o7 = Ee * K.o7;
  const T a = Ee * K.a, b = Ee * K.b, r = Ee * K.r, s = Ee * K.s;
  T t;
  t = o0 * (P[0][1] + P[1][2] + P[2][4]);
  Q[0][1] = fma(k0, P[0][1], t);
  Q[1][2] = fma(k0, P[1][2], t);
  Q[2][4] = fma(k0, P[2][4], t);
  t = o7 * (P[0][6] + P[1][5] + P[2][3]);
  Q[0][6] = fma(k7, P[0][6], t);
  Q[1][5] = fma(k7, P[1][5], t);
  Q[2][3] = fma(k7, P[2][3], t);
  Q[0][0] = Q[1][0] = Q[2][0] = T(0);   // rigid translations carry no energy
  Q[1][3] = fma(a, P[1][3], b * P[2][5]);
  Q[2][5] = fma(b, P[1][3], a * P[2][5]);
  Q[0][3] = fma(a, P[0][3], b * P[2][6]);
  Q[2][6] = fma(b, P[0][3], a * P[2][6]);
  Q[0][5] = fma(a, P[0][5], b * P[1][6]);
  Q[1][6] = fma(b, P[0][5], a * P[1][6]);
  t = r * (P[0][2] + P[1][1]);
  Q[0][2] = t;
  Q[1][1] = t;
  Q[2][7] = s * P[2][7];
  t = r * (P[0][4] + P[2][1]);
  Q[0][4] = t;
  Q[2][1] = t;
  Q[1][7] = s * P[1][7];
  t = r * (P[1][4] + P[2][2]);
  Q[1][4] = t;
  Q[2][2] = t;
  Q[0][7] = s * P[0][7];
}

// Tensor maps of one matvec launch (TMA descriptors, kernel-parameter space).
struct MvMaps {
  CUtensorMap vin;    // 4D {NY, NZ, NXL, 3}: p (plain) or r (fused)
  CUtensorMap pold;   // 4D, fused only
  CUtensorMap invd;   // 3D {NY, NZ, NXL}, fused only
  CUtensorMap E;      // 3D {EY, EZ, NEXL}
};

// Epilogue operands (multigrid V-cycle, b = r of the PCG):
//   kEpi = 1: out = mask(v + w M^-1 (b - K v)) and rho = b . out (last sweep)
//   kEpi = 2: out = mask(b - K v)  (the residual the restriction reads)
//   kEpi = 3: out = mask(K v)      (power steps of the smoother-weight estimate)
struct MvEpi {
  const double* b;          // 3 * ncomp
  const double* invd;       // per node
  const uint8_t* fixm;      // per node
  float* out32;             // kEpi = 2: if set, the residual is written here in fp32 (the
                            // restriction input of an fp32 multigrid hierarchy)
  float* w32;               // kEpi = 1: if set, the result is written here in fp32 (the
                            // fp32 multigrid's V-cycle output, read by the PCG matvec as a
                            // float TMA tile) instead of the double `q` output
  const double* qk;         // kEpi = 1: if set, the PCG's q = K p of this iteration; the
                            // epilogue also reduces q.out for the flexible (Polak-Ribiere)
                            // beta = -alpha (q.z)/rz of the K-cycle PCG (reading M9)
  // fp32 Krylov vectors: if set, b is read from b32 (r in fp32), the
  // flexible beta's q from qk32, and the PCG matvec (kEpi = 0) writes q to q32
  const float* b32;
  const float* qk32;
  float* q32;
};

constexpr int kMvStages = 3;   // raw TMA stages in flight ahead of the pre-pass
// TV: element type of the vin tile (double; float for the post-smoothing
// matvec's z, which the fp32 operator rounds to float anyway).  A float box
// row must be a multiple of 16 B (36 values) and starts at a y multiple of 4.
template <int TZ, typename TV = double> struct MvSmem {
  static constexpr int YW = 34;                                   // 33 nodes, box width padded to 16 B
  static constexpr int YWV = sizeof(TV) == 8 ? 34 : 36;           // vin box width
  static constexpr int V = 3 * (TZ + 1) * YW * 8;                 // bytes of one 3-component node tile
  static constexpr int VV = 3 * (TZ + 1) * YWV * (int)sizeof(TV); // bytes of the vin tile
  static constexpr int I = (TZ + 1) * YW * 8;                     // one scalar node tile
  static constexpr int EB = TZ * YW * 8;                          // element tile (box width 34 as well)
  static constexpr int VA = (V + 127) / 128 * 128, IA = (I + 127) / 128 * 128, EA = (EB + 127) / 128 * 128;
  static constexpr int VAV = (VV + 127) / 128 * 128;
  // stage = [vin][p_old (pre 1,2)][M^-1 (pre 1,3)][E]
  __host__ __device__ static constexpr int ioff(int pre) { return pre == 1 ? VAV + VA : VAV; }
  __host__ __device__ static constexpr int eoff(int pre) {
    return VAV + (pre == 1 || pre == 2 ? VA : 0) + (pre == 1 || pre == 3 ? IA : 0);
  }
  __host__ __device__ static constexpr int stage(int pre) { return eoff(pre) + EA; }
  // raw stages + 3 rotating p-planes (pre-pass output) + alignment slack
  __host__ __device__ static constexpr int bytes(int pre) { return kMvStages * stage(pre) + 3 * VA + 128; }
};

// TC: arithmetic type of the element operator (double; float for the
// multigrid smoothing matvecs with mg_fp32 -- the TMA operands stay fp64, the
// p-planes and the Walsh-domain work are fp32, the epilogue finishes in fp64).
template <int TZ, int kPre, bool kDot, int kEpi, typename TC, typename TV = double>
__global__ void __launch_bounds__(32 * TZ, (TZ <= 8 ? (sizeof(TC) == 4 ? 3 : 2) : 1))
k_mv_wht(const __grid_constant__ MvMaps maps, Geo g, DevState* st, int gate, int CX,
         double* __restrict__ pnew, double* __restrict__ q,
         double* partials, unsigned int* counter, int finish, const double* __restrict__ scale, MvEpi epi) {
  pdl_enter();
  if (gate && st->done) return;
  constexpr bool kFused = kPre != 0;
  constexpr bool kInvd = kPre == 1 || kPre == 3;
  using L = MvSmem<TZ, TV>;
  static_assert(sizeof(TV) == 8 || kPre == 0 || kPre == 2 || kPre == 3,
                "a float vin tile is not used by the Jacobi pre-pass");
  const double beta = (kPre == 1 || kPre == 2) && !st->fresh ? st->beta : 0.0;
  const double wsc = (kPre == 3 || kEpi == 1) ? *scale : 1.0;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ TC xch[2][3][TZ][32];   // lanes contiguous: conflict-free
  __shared__ __align__(8) uint64_t full[kMvStages];

  const int ty = threadIdx.x, tz = threadIdx.y;
  const bool leader = (ty == 0 && tz == 0);
  const int y0 = blockIdx.x * 31, z0 = blockIdx.y * (TZ - 1);   // stored coords of the tile's (ty,tz) = (0,0)
  // TMA boxes start at an even stored y (16-byte aligned row start); yoff in {0,1}
  const int yb = y0 & ~1, yoff = y0 - yb;
  const int ybv = sizeof(TV) == 8 ? yb : (y0 & ~3);   // vin box start (16-byte aligned)
  constexpr int CSV = (TZ + 1) * L::YWV;              // vin tile component stride
  const int iyb = y0 - 1 + ty, izb = z0 - 1 + tz;                 // base node of this thread
  const int chunk = blockIdx.z;
  const int xend_slab = g.ex0 + g.nown;
  const int xs = g.ex0 + chunk * CX;
  const int xe = min(xs + CX, xend_slab);
  const bool first_chunk = chunk == 0, last_chunk = (xe == xend_slab);
  const bool owned = ty >= 1 && tz >= 1 && iyb <= g.nely && izb <= g.nelz;
  // 32-bit in-array offsets (init validates 3*ncomp < 2^31)
  const int ob = (izb + 1) * g.NY + (iyb + 1);
  const int ncomp = (int)g.ncomp, nplane = (int)g.nplane;
  const int nunits = xe - xs + 2;           // node planes xs-1 .. xe
  // running output pointers at the base node (advanced by nplane per step)
  double* qp = q + (size_t)(xs - g.ex0 + 1) * nplane + ob;

  auto slot = [&](int s) { return dsm + s * L::stage(kPre); };
  TC* pbuf = reinterpret_cast<TC*>(dsm + kMvStages * L::stage(kPre));           // [3][3][TZ+1][YW]
  constexpr int PB = L::VA / (int)sizeof(TC);                                        // entries per p-plane
  constexpr int CS = (TZ + 1) * L::YW;                                               // component stride
  auto issue = [&](int t) {                 // unit t: node plane j = xs-1+t, element plane j-1
    const int s = t % kMvStages;
    unsigned char* b = slot(s);
    const int j = xs - 1 + t;
    const int ixl = j - g.ex0 + 1;
    const uint32_t bytes = L::VV + (kPre == 1 || kPre == 2 ? L::V : 0) + (kInvd ? L::I : 0) + (t > 0 ? L::EB : 0);
    mbar_arrive_expect_tx(&full[s], bytes);
    tma_load_4d(b, &maps.vin, &full[s], ybv, z0, ixl, 0);
    if (kPre == 1 || kPre == 2) tma_load_4d(b + L::VAV, &maps.pold, &full[s], yb, z0, ixl, 0);
    if (kInvd) tma_load_3d(b + L::ioff(kPre), &maps.invd, &full[s], yb, z0, ixl);
    if (t > 0) tma_load_3d(b + L::eoff(kPre), &maps.E, &full[s], yb, z0, j - 1 - g.ex0 + g.H);
  };
  if (leader) {
    tma_prefetch_desc(&maps.vin);
    tma_prefetch_desc(&maps.E);
    if (kPre == 1 || kPre == 2) tma_prefetch_desc(&maps.pold);
    if (kInvd) tma_prefetch_desc(&maps.invd);
    for (int s = 0; s < kMvStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (leader)
    for (int t = 0; t < min(kMvStages, nunits); ++t) issue(t);

  // Pre-pass of unit t: p = M^{-1} r + beta p_old once per node of the (TZ+1) x 34
  // tile plane into p-plane t%3 (plain variant: copy), owner nodes write p to
  // global; returns this thread's E_e for element plane j-1.  The raw stage is
  // fully consumed here.
  // Pre-pass node mapping (fixed per thread): nodes tid and tid + 32*TZ of the tile plane
  const int tid = tz * 32 + ty;
  constexpr int NPN = (CS + 32 * TZ - 1) / (32 * TZ);       // nodes per thread (2 for TZ = 8)
  int pn_idx[NPN];
  long long pn_off[NPN];                                      // global offset in a plane, -1 if not owned
#pragma unroll
  for (int u = 0; u < NPN; ++u) {
    const int n = tid + u * 32 * TZ;
    pn_idx[u] = n < CS ? n : -1;
    pn_off[u] = -1;
    if (n < CS) {
      const int row = n / L::YW, col = n - row * L::YW;
      const int cty = col - yoff, iy = yb + col - 1, iz = z0 + row - 1;
      if (cty >= 1 && cty <= 31 && row >= 1 && row <= TZ - 1 && iy <= g.nely && iz <= g.nelz)
        pn_off[u] = (long long)(z0 + row) * g.NY + (yb + col);
    }
  }
  // Pre-pass of unit t: p = M^{-1} r + beta p_old once per node of the (TZ+1) x 34
  // tile plane into p-plane t%3 (plain variant: copy), owner nodes write p to
  // global; returns this thread's E_e for element plane j-1.  The raw stage is
  // fully consumed here.
  auto prepass = [&](int t) -> TC {
    const int s = t % kMvStages;
    mbar_wait(&full[s], (uint32_t)((t / kMvStages) & 1));
    const double* sv = reinterpret_cast<const double*>(slot(s));
    const TV* svv = reinterpret_cast<const TV*>(slot(s));
    const double* sp = reinterpret_cast<const double*>(slot(s) + L::VAV);
    const double* si = reinterpret_cast<const double*>(slot(s) + L::ioff(kPre));
    const double* se = reinterpret_cast<const double*>(slot(s) + L::eoff(kPre));
    TC* pb = pbuf + (t % 3) * PB;
    const bool wr_plane = kFused && pnew != nullptr &&
                          ((t >= 1 && t < nunits - 1) || (t == 0 && first_chunk) || (t == nunits - 1 && last_chunk));
    double* pplane = pnew + (size_t)(xs + t - g.ex0) * nplane;     // node plane j = xs-1+t
#pragma unroll
    for (int u = 0; u < NPN; ++u) {
      const int n = pn_idx[u];
      if (n < 0) continue;
      double v[3];
      if (kPre == 1) {
        const double iv = si[n];
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = fma(beta, sp[c * CS + n], iv * sv[c * CS + n]);
      } else if (kPre == 2 && sizeof(TV) == 8) {
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = fma(beta, sp[c * CS + n], sv[c * CS + n]);
      } else if (kPre == 2) {   // V-cycle output w in fp32 (float vin tile, row stride YWV)
        const int row = n / L::YW, nv = row * L::YWV + (n - row * L::YW) + (yb - ybv);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = fma(beta, sp[c * CS + n], (double)svv[c * CSV + nv]);
      } else if (kPre == 3 && sizeof(TV) == 8) {
        const double iv = wsc * si[n];
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = iv * sv[c * CS + n];
      } else if (kPre == 3) {   // fp32 Krylov residual r (float vin tile)
        const double iv = wsc * si[n];
        const int row = n / L::YW, nv = row * L::YWV + (n - row * L::YW) + (yb - ybv);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = iv * (double)svv[c * CSV + nv];
      } else if (sizeof(TV) == 8) {
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = sv[c * CS + n];
      } else {   // float vin tile: row stride YWV, columns shifted by yb - ybv
        const int row = n / L::YW, nv = row * L::YWV + (n - row * L::YW) + (yb - ybv);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = (double)svv[c * CSV + nv];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) pb[c * CS + n] = (TC)v[c];
      if (wr_plane && pn_off[u] >= 0) {
        double* o = pplane + pn_off[u];
#pragma unroll
        for (int c = 0; c < 3; ++c) o[(size_t)c * ncomp] = v[c];
      }
    }
    return t > 0 ? (TC)se[tz * L::YW + ty + yoff] : TC(0);
  };
  // corners (k = ay + 2 az) of this thread's element column in p-plane t%3
  auto corners_wht = [&](int t, TC G[3][4]) {
    const TC* pb = pbuf + (t % 3) * PB;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      TC v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = pb[c * CS + (tz + (k >> 1)) * L::YW + ty + yoff + (k & 1)];
      wht4(v, G[c]);
    }
  };
  auto release = [&](int t) {               // all threads are past the pre-pass of unit t
    if (leader && t + kMvStages < nunits) {
      fence_proxy_async();
      issue(t + kMvStages);
    }
  };

  TC G0[3][4], A[3][4];
  TC Ecur = TC(0);
  // kEpi: the owner's epilogue operands (b, M^-1, mask) for the next node plane it
  // writes are loaded one x-step ahead, so the global loads overlap the compute
  double eb[3] = {0.0, 0.0, 0.0}, einv = 0.0, eq[3] = {0.0, 0.0, 0.0};
  uint8_t efm = 0;
  auto epi_load = [&](long long go) {
    if (kEpi != 0 && owned) {
      efm = epi.fixm[go];
      if (kEpi == 1) einv = epi.invd[go];
      if (kEpi == 1 || kEpi == 2)
#pragma unroll
        for (int c = 0; c < 3; ++c) eb[c] = epi.b32 ? (double)epi.b32[go + c * ncomp] : epi.b[go + c * ncomp];
      if (kEpi == 1 && epi.qk32)
#pragma unroll
        for (int c = 0; c < 3; ++c) eq[c] = (double)epi.qk32[go + c * ncomp];
      else if (kEpi == 1 && epi.qk)
#pragma unroll
        for (int c = 0; c < 3; ++c) eq[c] = epi.qk[go + c * ncomp];
    }
  };
  if (nunits > 2) epi_load(qp - q);
  prepass(0);
  if (nunits > 1) Ecur = prepass(1);
  __syncthreads();
  release(0);
  if (nunits > 1) release(1);
  corners_wht(0, G0);
  double dot = 0.0, dot2 = 0.0;
  for (int t = 1; t < nunits; ++t) {
    const int ex = xs - 2 + t;              // element plane of this step (node planes ex, ex+1)
    (void)ex;
    TC G1[3][4];
    corners_wht(t, G1);
    const TC Ee = Ecur;
    if (t + 1 < nunits) Ecur = prepass(t + 1);
    TC Q[3][8];
    {
      TC P[3][8];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          P[c][2 * k] = G0[c][k] + G1[c][k];
          P[c][2 * k + 1] = G0[c][k] - G1[c][k];
        }
      wht_block(P, Ee, Q);
    }
    if (t >= 2) {                           // ex >= xs: complete node plane ex
      const int buf = t & 1;
      TC S[3];
      double pbase[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        TC Ac[4], C[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) Ac[k] = A[c][k] + (Q[c][2 * k] + Q[c][2 * k + 1]);
        wht4(Ac, C);
        // y-z neighbourhood: owner(ty,tz) = C0(ty,tz) + C1(ty-1,tz) + C2(ty,tz-1) + C3(ty-1,tz-1)
        xch[buf][c][tz][ty] = C[2] + __shfl_up_sync(0xffffffffu, C[3], 1);
        S[c] = C[0] + __shfl_up_sync(0xffffffffu, C[1], 1);
        // p at the owner's node of plane ex (p-plane (t-1)%3 is rewritten only after this barrier)
        pbase[c] = (kDot || kEpi) ? (double)pbuf[((t - 1) % 3) * PB + c * CS + tz * L::YW + ty + yoff] : 0.0;
      }
      __syncthreads();
      if (owned && kEpi == 0) {
        // q is NOT masked here: the fixed-DOF mask is applied by the consumers
        // (k_update, k_residual, k_mask_fixed); p is exactly 0 on fixed DOFs, so
        // p.q is unaffected.  Keeps a latency-bound byte load off this loop.
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double qv = (double)(S[c] + xch[buf][c][tz - 1][ty]);
          if (epi.q32) {   // fp32 Krylov q: p.q of exactly the rounded q the update uses
            const float qf = (float)qv;
            epi.q32[(qp - q) + c * ncomp] = qf;
            qv = (double)qf;
          } else {
            qp[c * ncomp] = qv;
          }
          if (kDot) dot = fma(pbase[c], qv, dot);
        }
      } else if (owned && (kEpi == 2 || kEpi == 3)) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double qv = (double)(S[c] + xch[buf][c][tz - 1][ty]);
          const double o = ((efm >> c) & 1) ? 0.0 : (kEpi == 2 ? eb[c] - qv : qv);
          if (kEpi == 2 && epi.out32) epi.out32[(qp - q) + c * ncomp] = (float)o;
          else qp[c * ncomp] = o;
        }
      } else if (owned) {
        // damped-Jacobi sweep on the owner's node: out = v + w D^-1 (b - K v)
        const double wd = wsc * einv;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double qv = (double)(S[c] + xch[buf][c][tz - 1][ty]);
          double zn = ((efm >> c) & 1) ? 0.0 : fma(wd, eb[c] - qv, pbase[c]);
          if (epi.w32) {   // the V-cycle output stored in fp32 (its precision is the fp32 hierarchy's)
            const float zf = (float)zn;
            epi.w32[(qp - q) + c * ncomp] = zf;
            zn = (double)zf;   // rho and q.w of exactly what the PCG will read
          } else {
            qp[c * ncomp] = zn;
          }
          dot = fma(eb[c], zn, dot);
          dot2 = fma(eq[c], zn, dot2);
        }
      }
      qp += nplane;
      if (t + 1 < nunits) epi_load(qp - q);
    } else {
      __syncthreads();
    }
    if (t + 1 < nunits) release(t + 1);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        A[c][k] = Q[c][2 * k] - Q[c][2 * k + 1];   // R1: element ex -> node plane ex+1
        G0[c][k] = G1[c][k];
      }
  }

  if (kEpi == 1) {
    __shared__ double tot[2];
    double vv[2] = {dot, dot2};
    if (grid_reduce<2>(vv, partials, counter, tot) && leader) {
      const double rho = tot[0];
      if (!finish) {                         // x-slabs: allreduced, then k_finish_rho
        st->sums[0] = rho;
        st->sums[1] = tot[1];
      } else if (!(rho > 0.0) || !isfinite(rho)) {
        st->status = 3;
        st->done = 1;
      } else {
        // flexible (K-cycle, M9): z.(r_new - r_old) = -alpha z.q
        st->beta = st->fresh ? 0.0 : epi.qk ? -st->alpha * tot[1] / st->rz : rho / st->rz;
        st->rz = rho;
      }
    }
  } else if (kDot) {
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
