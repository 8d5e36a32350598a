// Host-side Hex8 element stiffness: unit cube, unit modulus, isotropic linear
// elasticity, 2x2x2 Gauss-Legendre quadrature (exact for the trilinear
// integrand).  PAPER P:42 §2.2 "Element stiffness matrices are pre-computed";
// SPEC S:117.  Local nodes in SPEC S:45 order; DOFs (ux,uy,uz) per node.
// Written independently of oracle/ke.py (no shared code).
#include <cmath>
#include <cstring>
#include <initializer_list>

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

namespace topo {
// Walsh-Hadamard block form of KE: B = H KE H^T / 64 with
// H[(c,m),(a,d)] = delta_cd (-1)^{m.a} (m, a in {0,1}^3, m = mx + 2 my + 4 mz;
// transformed index 3m + c).  Extracts the 8 distinct entries used by the
// matvec kernel and verifies the block pattern the kernel assumes (every
// other entry zero, equal entries equal) to `tol` relative.  Returns false if
// the structure does not hold.
bool wht_constants(const double* ke, double out[8], double tol) {
  double H[24][24] = {};
  for (int c = 0; c < 3; ++c)
    for (int m = 0; m < 8; ++m)
      for (int a = 0; a < 8; ++a) {
        const int par = ((m & 1) * kCorner[a][0]) + (((m >> 1) & 1) * kCorner[a][1]) + ((m >> 2) * kCorner[a][2]);
        H[3 * m + c][3 * a + c] = (par & 1) ? -1.0 : 1.0;
      }
  double B[24][24];
  double T[24][24];
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) {
      double s = 0.0;
      for (int k = 0; k < 24; ++k) s += H[i][k] * ke[k * 24 + j];
      T[i][j] = s;
    }
  double bmax = 0.0;
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) {
      double s = 0.0;
      for (int k = 0; k < 24; ++k) s += T[i][k] * H[j][k];
      B[i][j] = s / 64.0;
      bmax = std::fmax(bmax, std::fabs(B[i][j]));
    }
  auto at = [&](int c, int m, int d, int n) { return B[3 * m + c][3 * n + d]; };
  const double d0 = at(0, 1, 0, 1), o0 = at(0, 1, 1, 2), d7 = at(0, 6, 0, 6), o7 = at(0, 6, 1, 5);
  const double a = at(1, 3, 1, 3), b = at(1, 3, 2, 5), r = at(0, 2, 0, 2), s = at(2, 7, 2, 7);
  // expected model of B, built from the 8 constants
  double M[24][24] = {};
  auto setp = [&](int c, int m, int d, int n, double v) { M[3 * m + c][3 * n + d] = v; };
  for (int pi : {0, 7}) {
    const double dd = pi == 0 ? d0 : d7, oo = pi == 0 ? o0 : o7;
    for (int c = 0; c < 3; ++c)
      for (int d = 0; d < 3; ++d) setp(c, pi ^ (1 << c), d, pi ^ (1 << d), c == d ? dd : oo);
  }
  for (int pi : {1, 2, 4}) {
    int cs[2], k = 0;
    for (int c = 0; c < 3; ++c)
      if ((1 << c) != pi) cs[k++] = c;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) setp(cs[i], pi ^ (1 << cs[i]), cs[j], pi ^ (1 << cs[j]), i == j ? a : b);
  }
  for (int pi : {3, 5, 6}) {
    int cs[2], k = 0, single = -1;
    for (int c = 0; c < 3; ++c) {
      if ((pi ^ (1 << c)) == 7) single = c;
      else cs[k++] = c;
    }
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) setp(cs[i], pi ^ (1 << cs[i]), cs[j], pi ^ (1 << cs[j]), r);
    setp(single, 7, single, 7, s);
  }
  double err = 0.0;
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) err = std::fmax(err, std::fabs(B[i][j] - M[i][j]));
  out[0] = d0 - o0;
  out[1] = o0;
  out[2] = d7 - o7;
  out[3] = o7;
  out[4] = a;
  out[5] = b;
  out[6] = r;
  out[7] = s;
  return err <= tol * bmax;
}
}  // namespace topo
