// Gravity-anomaly post-processing ("better gravity anomaly
// solutions"; PAPER.md:39-44 gravity = gradient of the potential): g_z = -dPhi_h/dz of the glued FE
// potential on the horizontal plane z = z0 at every cell-centre column (x_c, y_c).  The point lies in
// hex cell (ci, cj, floor(z0/hz)) and in the Kuhn tet pi with xi_pi0 >= xi_pi1 >= xi_pi2 (ties broken
// by axis index, stable), where the P1/P2 gradient is evaluated exactly:
//   lambda = (1 - s0, s0 - s1, s1 - s2, s2) for the sorted local coordinates s,
//   grad phi_i = (4 lambda_i - 1) grad lambda_i, grad phi_ij = 4 (lambda_i grad lambda_j + lambda_j grad lambda_i).
#include <vector>

#include "ctx.h"

namespace osm {

struct GravTable {
  double g[6][4][3];  // physical barycentric gradients of tet t
  int8_t off[6][10][3];  // lattice offsets of the local nodes in the cell
  int perm[6][3];
};

namespace {

__global__ void k_gravity_z(GravTable T, int order, int64_t nx, int64_t ny, int64_t nz, int64_t Nx, int64_t Ny,
                            double hz, double z0, const double* __restrict__ phi, double* __restrict__ gz) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nx * ny) return;
  const int64_t ci = c % nx, cj = c / nx;
  int64_t ck = (int64_t)floor(z0 / hz);
  ck = ck < 0 ? 0 : (ck > nz - 1 ? nz - 1 : ck);
  const double xi[3] = {0.5, 0.5, z0 / hz - (double)ck};
  // stable descending sort of 3 values -> permutation
  int p[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && xi[p[j]] > xi[p[j - 1]]; --j) {
      const int t = p[j];
      p[j] = p[j - 1];
      p[j - 1] = t;
    }
  int t = 0;
  for (int k = 0; k < 6; ++k)
    if (T.perm[k][0] == p[0] && T.perm[k][1] == p[1] && T.perm[k][2] == p[2]) t = k;
  const double s0 = xi[p[0]], s1 = xi[p[1]], s2 = xi[p[2]];
  const double lam[4] = {1.0 - s0, s0 - s1, s1 - s2, s2};
  double gr[3] = {0.0, 0.0, 0.0};
  const int nloc = order == 1 ? 4 : 10;
  const int edge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (int a = 0; a < nloc; ++a) {
    const int64_t I = order * ci + T.off[t][a][0], J = order * cj + T.off[t][a][1], K = order * ck + T.off[t][a][2];
    const double v = phi[I + Nx * (J + Ny * K)];
    for (int d = 0; d < 3; ++d) {
      double gp;
      if (order == 1) {
        gp = T.g[t][a][d];
      } else if (a < 4) {
        gp = (4.0 * lam[a] - 1.0) * T.g[t][a][d];
      } else {
        const int i = edge[a - 4][0], j = edge[a - 4][1];
        gp = 4.0 * (lam[i] * T.g[t][j][d] + lam[j] * T.g[t][i][d]);
      }
      gr[d] += v * gp;
    }
  }
  gz[c] = -gr[2];
}

}  // namespace

void gravity_z(Ctx& c, double z0, double* d_out) {
  GravTable T{};
  const double h[3] = {c.mesh.lx / c.mesh.nx, c.mesh.ly / c.mesh.ny, c.mesh.lz / c.mesh.nz};
  static const int kPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  for (int t = 0; t < 6; ++t) {
    std::vector<double> g;
    tet_bary_gradients(t, h, g);
    for (int a = 0; a < 4; ++a)
      for (int d = 0; d < 3; ++d) T.g[t][a][d] = g[a * 3 + d];
    const auto offs = tet_local_offsets(t, c.mesh.order);
    for (size_t a = 0; a < offs.size(); ++a)
      for (int d = 0; d < 3; ++d) T.off[t][a][d] = (int8_t)offs[a][d];
    for (int d = 0; d < 3; ++d) T.perm[t][d] = kPerm[t][d];
  }
  const int o = c.mesh.order;
  const int64_t n = c.mesh.nx * c.mesh.ny;
  k_gravity_z<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(T, o, c.mesh.nx, c.mesh.ny, c.mesh.nz,
                                                                o * c.mesh.nx + 1, o * c.mesh.ny + 1, h[2], z0, c.phi,
                                                                d_out);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

}  // namespace osm
