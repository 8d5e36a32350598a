// A6: rmin cone filter (§2.4) as an x-marching 2.5D stencil.
//
// out_i = post_i( sum_j H_ij v_j ),  H_ij = max(0, rmin - |c_i - c_j|) on the
// (2R+1)^3 offset box (zero weights outside the ball), v = the zero-padded
// operand of k_filt_prep (kernels.cuh), post as in k_filt_apply.
//
// Mapping: a CTA of 32 (y) x 8 (z-groups) threads owns a 32 x 32 (y, z) output
// tile and marches along x over a chunk of output planes.  Each input plane is
// staged ONCE in shared memory by TMA (a (32+2R) x (32+2R) box of the padded
// operand, 3-stage mbarrier ring, zero fill beyond the padded array), and
// contributes to the 2R+1 output planes x-R..x+R, whose partial sums live in
// registers (acc[2R+1][4]: a thread owns one y column and 4 consecutive z
// outputs).  Per input plane a thread reads (4+2R)(2R+1) values from shared
// memory (lanes on consecutive y: conflict-free) and issues (2R+1)^3 * 4
// DFMAs, weights from constant memory at compile-time indices.  Each operand
// value is read from HBM once (halo columns / rows of neighbouring tiles come
// from L2), instead of the 93-tap gather per output of k_filt_apply.
// The box includes the zero-weight corners ((2R+1)^3 = 125 DFMA per output at
// R = 2 vs 93 taps): fp64-ALU bound by design.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace topo {

__constant__ double c_fw[7 * 7 * 7];   // [dx+R][dz+R][dy+R], rmin - |d| inside the ball, else 0
__constant__ double c_fw2[4 * 4 * 4];  // [|dx|][a][b], a = min(|dy|,|dz|) <= b = max: the same weights by class

constexpr int kF25Y = 32, kF25Z = 32, kF25TZ = 4, kF25Stages = 3;

template <int R> struct F25Smem {
  static constexpr int BY = kF25Y + 2 * R;                         // box width (y), 16-byte multiple
  static constexpr int BZ = kF25Z + 2 * R;
  static constexpr int STAGE = (BY * BZ * 8 + 127) / 128 * 128;
  static constexpr int BYTES = kF25Stages * STAGE + 128;
};

// Post-op of an output (k_filt_apply's arithmetic): X0 / PLAIN multiply by the
// precomputed 1/Hs (within 1 ulp of the division, whose inlined slow path in the
// march loop made the x filter 665 vs ~150 us at config 4); its operands are
// loaded before the step's TMA wait.

// kSym: the cone weights depend on |d| only, so per input plane a thread first sums
// its 4 z-outputs' inputs by (y, z) offset class {|dy|, |dz|} = {a, b} (1D y-pair
// sums per row, then z-pairs), and each output plane offset +-dx gets ONE value
// V_|dx| = sum_classes w(|dx|, a, b) T_ab: ~33 fp64 ops per output at R = 2
// instead of the 125 DFMA of the box -- the same sum, reassociated.
template <int R, int MODE, bool kSym>
__global__ void __launch_bounds__(kF25Y * (kF25Z / kF25TZ), R == 3 ? 1 : 2)
k_filt25(const __grid_constant__ CUtensorMap vmap, Geo g, FiltPad fp, int CX, const double* __restrict__ a,
         const double* __restrict__ hs, const uint8_t* __restrict__ passive, double* __restrict__ out) {
  pdl_enter();
  constexpr int P = 2 * R + 1;
  using L = F25Smem<R>;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kF25Stages];
  const int ty = threadIdx.x, tg = threadIdx.y;
  const bool leader = ty == 0 && tg == 0;
  const int y0 = blockIdx.x * kF25Y, z0 = blockIdx.y * kF25Z;
  const int x0 = g.ex0 + blockIdx.z * CX, x1 = min(x0 + CX, g.ex0 + g.nex);   // output planes [x0, x1)
  const int nout = x1 - x0;
  if (nout <= 0) return;
  const int nin = nout + 2 * R;                                                // input planes x0-R .. x1+R-1
  const int ey = y0 + ty, ez0 = z0 + tg * kF25TZ;                              // this thread's outputs
  auto stage = [&](int t) { return reinterpret_cast<const double*>(dsm + (t % kF25Stages) * L::STAGE); };
  auto issue = [&](int t) {
    const int s = t % kF25Stages;
    mbar_arrive_expect_tx(&full[s], L::BY * L::BZ * 8);
    // padded coordinates: column ey + R, row ez + R, plane exl = x - ex0 + H
    tma_load_3d(dsm + s * L::STAGE, &vmap, &full[s], y0, z0, x0 - R + t - g.ex0 + g.H);
  };
  if (leader) {
    tma_prefetch_desc(&vmap);
    for (int s = 0; s < kF25Stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (leader)
    for (int t = 0; t < min(kF25Stages, nin); ++t) issue(t);

  double acc[P][kF25TZ];
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int k = 0; k < kF25TZ; ++k) acc[p][k] = 0.0;
  const bool col_ok = ey < g.nely;

  for (int tb = 0; tb < nin; tb += P) {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int t = tb + j;
      if (t >= nin) break;
      // post-op operands of the output plane this step completes (t - 2R), loaded
      // before the TMA wait and the arithmetic so their latency is hidden
      double ph[kF25TZ];
      uint8_t pp[kF25TZ];
      if (MODE == F_X0 || MODE == F_PLAIN || MODE == F_XDC) {
        const int to0 = t - 2 * R;
#pragma unroll
        for (int k = 0; k < kF25TZ; ++k) {
          ph[k] = 1.0;
          pp[k] = 0;
          if (to0 >= 0 && col_ok && ez0 + k < g.nelz) {
            const long long i = elem_idx(g, x0 + to0, ey, ez0 + k);
            ph[k] = hs[i];
            if (MODE == F_X0) pp[k] = passive[i];
          }
        }
      }
      mbar_wait(&full[t % kF25Stages], (uint32_t)((t / kF25Stages) & 1));
      const double* sv = stage(t);
      if (kSym) {
        double Y[kF25TZ + 2 * R][R + 1];   // Y[jr][a] = v(y - a) + v(y + a) of row jr (a = 0: v(y))
#pragma unroll
        for (int jr = 0; jr < kF25TZ + 2 * R; ++jr) {
          const double* row = sv + (tg * kF25TZ + jr) * L::BY + ty;
          Y[jr][0] = row[R];
#pragma unroll
          for (int a = 1; a <= R; ++a) Y[jr][a] = row[R - a] + row[R + a];
        }
#pragma unroll
        for (int k = 0; k < kF25TZ; ++k) {
          const int c = R + k;             // row of output k
          double T[R + 1][R + 1];          // class sums, a <= b
#pragma unroll
          for (int a = 0; a <= R; ++a)
#pragma unroll
            for (int b = a; b <= R; ++b) {
              if (a == 0 && b == 0) T[0][0] = Y[c][0];
              else if (a == 0) T[0][b] = (Y[c - b][0] + Y[c + b][0]) + Y[c][b];
              else if (a == b) T[a][a] = Y[c - a][a] + Y[c + a][a];
              else T[a][b] = (Y[c - b][a] + Y[c + b][a]) + (Y[c - a][b] + Y[c + a][b]);
            }
#pragma unroll
          for (int dx = 0; dx <= R; ++dx) {
            double V = 0.0;
#pragma unroll
            for (int a = 0; a <= R; ++a)
#pragma unroll
              for (int b = a; b <= R; ++b)
                if (dx * dx + a * a + b * b < (R + 1) * (R + 1)) V = fma(c_fw2[(dx * 4 + a) * 4 + b], T[a][b], V);
            const int s0 = ((j - R - dx) % P + P) % P;
            acc[s0][k] += V;
            if (dx > 0) {
              const int s1 = ((j - R + dx) % P + P) % P;
              acc[s1][k] += V;
            }
          }
        }
      } else
#pragma unroll
      for (int jr = 0; jr < kF25TZ + 2 * R; ++jr) {
        const double* row = sv + (tg * kF25TZ + jr) * L::BY + ty;
#pragma unroll
        for (int dy = -R; dy <= R; ++dy) {
          const double v = row[dy + R];
#pragma unroll
          for (int k = 0; k < kF25TZ; ++k) {
            const int dz = jr - R - k;              // input row - output row
            if (dz < -R || dz > R) continue;
#pragma unroll
            for (int dx = -R; dx <= R; ++dx) {      // input plane t feeds output plane t - R - dx (relative)
              const int slot = ((j - R - dx) % P + P) % P;
              acc[slot][k] = fma(c_fw[((dx + R) * 7 + (dz + R)) * 7 + (dy + R)], v, acc[slot][k]);
            }
          }
        }
      }
      __syncthreads();                               // stage t consumed by every thread
      if (leader && t + kF25Stages < nin) {
        fence_proxy_async();
        issue(t + kF25Stages);
      }
      // output plane t - 2R is complete: its slot is (j - 2R) mod P = (j + 1) mod P
      const int to = t - 2 * R;
      constexpr int dummy = 0;
      (void)dummy;
      const int es = (j + 1) % P;
      if (to >= 0) {
        const int xo = x0 + to;
#pragma unroll
        for (int k = 0; k < kF25TZ; ++k) {
          const int ez = ez0 + k;
          if (col_ok && ez < g.nelz) {
            const long long i = elem_idx(g, xo, ey, ez);
            double r = acc[es][k];
            if (MODE == F_XDC) r = r / (ph[k] * fmax(1e-3, a[i]));
            else if (MODE != F_DIV) r = r * ph[k];   // X0 / PLAIN: hs = 1/Hs
            if (MODE == F_X0 && pp[k]) r = pp[k] == kSolid ? 1.0 : 0.0;
            out[i] = r;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kF25TZ; ++k) acc[es][k] = 0.0;
    }
  }
}

}  // namespace topo
