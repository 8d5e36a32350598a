// Host-side tables of the geometric multigrid preconditioner (SURVEY §8(f)
// NEXT f2; readings M1-M6).  Written independently of oracle/mg.py.
//
// Nested Hex8 grids: a coarse element is 2x2x2 fine elements.  Child c =
// cx + 2 cy + 4 cz of a coarse element covers the sub-cube [c/2, (c+1)/2]^3 of
// the coarse element's reference cube.  Trilinear interpolation from the coarse
// corners R to the child's corners A (SPEC S:45 local order) has the weights
//   w[c][A][R] = prod_d (R_d ? t_d : 1 - t_d),   t_d = (c_d + A_d) / 2,
// identical for the three displacement components.  Galerkin element matrices
// (P^T K P, P element-local for nested trilinear grids):
//   level 1 from fine moduli:   K1_e = sum_c E_c   M_c,   M_c = P_c^T KE P_c
//   level 2 from fine moduli:   K2_e = sum_g E_g   N_g,   N_g = P_g^T KE P_g,
//   P_g = P_d P_c for grandchild g = (child c of the coarse element, child d of c).
#include <cstring>

namespace topo {

static const int kCornerMg[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                    {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

void mg_child_weights(double w[8][8][8]) {
  for (int c = 0; c < 8; ++c) {
    const int cd[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
    for (int A = 0; A < 8; ++A)
      for (int R = 0; R < 8; ++R) {
        double v = 1.0;
        for (int d = 0; d < 3; ++d) {
          const double t = 0.5 * (cd[d] + kCornerMg[A][d]);
          v *= kCornerMg[R][d] ? t : 1.0 - t;
        }
        w[c][A][R] = v;
      }
  }
}

// out[3R+i][3S+j] = sum_{A,B} W[A][R] KE[3A+i][3B+j] W[B][S]
static void galerkin_node_weights(const double* ke, const double W[8][8], double* out) {
  for (int R = 0; R < 8; ++R)
    for (int S = 0; S < 8; ++S)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
          for (int A = 0; A < 8; ++A) {
            if (W[A][R] == 0.0) continue;
            for (int B = 0; B < 8; ++B) {
              if (W[B][S] == 0.0) continue;
              s += W[A][R] * ke[(3 * A + i) * 24 + 3 * B + j] * W[B][S];
            }
          }
          out[(3 * R + i) * 24 + 3 * S + j] = s;
        }
}

// tab8 [8][576] (child c), tab64 [64][576] (fine offset g = gx + 4 gy + 16 gz in
// [0,4)^3 of a level-2 element), diag8 [8][24] = diagonal of tab8.
void mg_galerkin_tables(const double* ke, double* tab8, double* tab64, double* diag8) {
  double w[8][8][8];
  mg_child_weights(w);
  for (int c = 0; c < 8; ++c) {
    galerkin_node_weights(ke, w[c], tab8 + 576 * c);
    for (int k = 0; k < 24; ++k) diag8[24 * c + k] = tab8[576 * c + 25 * k];
  }
  for (int gz = 0; gz < 4; ++gz)
    for (int gy = 0; gy < 4; ++gy)
      for (int gx = 0; gx < 4; ++gx) {
        const int c = (gx >> 1) + 2 * (gy >> 1) + 4 * (gz >> 1);
        const int d = (gx & 1) + 2 * (gy & 1) + 4 * (gz & 1);
        double W[8][8];
        for (int A = 0; A < 8; ++A)
          for (int R = 0; R < 8; ++R) {
            double s = 0.0;
            for (int Q = 0; Q < 8; ++Q) s += w[d][A][Q] * w[c][Q][R];
            W[A][R] = s;
          }
        galerkin_node_weights(ke, W, tab64 + 576 * (gx + 4 * gy + 16 * gz));
      }
}

}  // namespace topo
