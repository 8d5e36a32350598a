// Host-side Hex8 element stiffness: unit cube, unit modulus, isotropic linear
// elasticity, 2x2x2 Gauss-Legendre quadrature (exact for the trilinear
// integrand).  PAPER P:42 §2.2 "Element stiffness matrices are pre-computed";
// SPEC S:117.  Local nodes in SPEC S:45 order; DOFs (ux,uy,uz) per node.
// Written independently of oracle/ke.py (no shared code).
#include <cmath>
#include <cstring>

namespace topo {

static const int kCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                  {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

// ke: 24x24 row-major.
void build_element_stiffness(double nu, double* ke) {
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = 1.0 / (2.0 * (1.0 + nu));
  const double g[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  std::memset(ke, 0, sizeof(double) * 576);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k) {
        const double s[3] = {g[i], g[j], g[k]};
        double grad[8][3];
        for (int a = 0; a < 8; ++a) {
          double N[3], dN[3];
          for (int d = 0; d < 3; ++d) {
            N[d] = kCorner[a][d] ? s[d] : 1.0 - s[d];
            dN[d] = kCorner[a][d] ? 1.0 : -1.0;
          }
          grad[a][0] = dN[0] * N[1] * N[2];
          grad[a][1] = N[0] * dN[1] * N[2];
          grad[a][2] = N[0] * N[1] * dN[2];
        }
        // Energy density of the bilinear form: for DOFs (a,c) and (b,d):
        //   lam * dNa_c dNb_d + mu * (dNa_d dNb_c + delta_cd * sum_k dNa_k dNb_k)
        for (int a = 0; a < 8; ++a)
          for (int b = 0; b < 8; ++b) {
            double dot = 0.0;
            for (int kk = 0; kk < 3; ++kk) dot += grad[a][kk] * grad[b][kk];
            for (int c = 0; c < 3; ++c)
              for (int d = 0; d < 3; ++d) {
                double v = lam * grad[a][c] * grad[b][d] + mu * grad[a][d] * grad[b][c];
                if (c == d) v += mu * dot;
                ke[(3 * a + c) * 24 + (3 * b + d)] += 0.125 * v;
              }
          }
      }
}

}  // namespace topo
