// Host-side Kuhn-mesh geometry for libosm.  See lattice.h.
//
// step 1 (Kuhn tets: for each axis permutation pi,
// v0 = 0, v1 = e_pi0, v2 = v1 + e_pi1, v3 = (1,1,1)), step 2 (P2 nodes = refined
// lattice), step 3 (P1/P2 stiffness), step 4 (exact load weights), step 7 (plane
// mass on the Kuhn faces).  The integrals here are evaluated in closed form over
// barycentric monomials, not by quadrature.
#include "lattice.h"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <tuple>

namespace osm {

namespace {

const int kPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
const int kEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

void tet_vertices(int t, int v[4][3]) {
  for (int a = 0; a < 4; ++a)
    for (int d = 0; d < 3; ++d) v[a][d] = 0;
  v[1][kPerm[t][0]] = 1;
  for (int d = 0; d < 3; ++d) v[2][d] = v[1][d];
  v[2][kPerm[t][1]] = 1;
  for (int d = 0; d < 3; ++d) v[3][d] = 1;
}

// barycentric gradients g[4][3] and volume of the tet with vertices X[4][3]
void bary_gradients(const double X[4][3], double g[4][3], double& vol) {
  double J[3][3];  // columns X1-X0, X2-X0, X3-X0
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) J[r][c] = X[c + 1][r] - X[0][r];
  double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
               J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  // inverse via adjugate: row i of J^{-1} = grad lambda_{i+1}
  double inv[3][3];
  inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
  inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
  inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
  inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
  inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
  inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
  inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  for (int d = 0; d < 3; ++d) {
    g[1][d] = inv[0][d];
    g[2][d] = inv[1][d];
    g[3][d] = inv[2][d];
    g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
  }
  vol = std::fabs(det) / 6.0;
}

double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// grad phi_a = sum_m (A[a][m] + sum_k B[a][m][k] lam_k) grad lam_m  (P2)
void p2_gradient_coeffs(double A[10][4], double B[10][4][4]) {
  for (int a = 0; a < 10; ++a)
    for (int m = 0; m < 4; ++m) {
      A[a][m] = 0.0;
      for (int k = 0; k < 4; ++k) B[a][m][k] = 0.0;
    }
  for (int i = 0; i < 4; ++i) {  // phi_i = lam_i (2 lam_i - 1): grad = (4 lam_i - 1) grad lam_i
    A[i][i] = -1.0;
    B[i][i][i] = 4.0;
  }
  for (int e = 0; e < 6; ++e) {  // phi_ij = 4 lam_i lam_j: grad = 4 lam_j grad lam_i + 4 lam_i grad lam_j
    int i = kEdge[e][0], j = kEdge[e][1];
    B[4 + e][i][j] = 4.0;
    B[4 + e][j][i] = 4.0;
  }
}

// int_T (a + b.lam)(a' + b'.lam) / |T|
double lin_product_integral(double a, const double* b, double ap, const double* bp) {
  double sb = 0, sbp = 0, quad = 0;
  for (int k = 0; k < 4; ++k) {
    sb += b[k];
    sbp += bp[k];
    for (int l = 0; l < 4; ++l) quad += b[k] * bp[l] * (k == l ? 2.0 : 1.0) / 20.0;
  }
  return a * ap + (a * sbp + ap * sb) / 4.0 + quad;
}

// triangle polynomial in barycentric (l0,l1,l2), degree <= 4; index a + 5b + 25c
struct TriPoly {
  double c[125] = {0};
};
double factorial(int n) { return n <= 1 ? 1.0 : n * factorial(n - 1); }
// int_T l0^a l1^b l2^c / |T| = 2 a! b! c! / (a+b+c+2)!
double tri_monomial(int a, int b, int c) { return 2.0 * factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + 2); }
TriPoly tri_mul(const TriPoly& p, const TriPoly& q) {
  TriPoly r;
  for (int i = 0; i < 125; ++i) {
    if (p.c[i] == 0) continue;
    int a = i % 5, b = (i / 5) % 5, c = i / 25;
    for (int j = 0; j < 125; ++j) {
      if (q.c[j] == 0) continue;
      int a2 = a + j % 5, b2 = b + (j / 5) % 5, c2 = c + j / 25;
      if (a2 < 5 && b2 < 5 && c2 < 5) r.c[a2 + 5 * b2 + 25 * c2] += p.c[i] * q.c[j];
    }
  }
  return r;
}
double tri_integral(const TriPoly& p) {
  double s = 0;
  for (int i = 0; i < 125; ++i)
    if (p.c[i] != 0) s += p.c[i] * tri_monomial(i % 5, (i / 5) % 5, i / 25);
  return s;
}

// Triangle mass / area, basis order: P1 (v0,v1,v2); P2 (v0,v1,v2,e01,e12,e02)
std::vector<double> tri_mass_unit(int order) {
  std::vector<TriPoly> basis;
  auto mono = [](int a, int b, int c, double v) {
    TriPoly p;
    p.c[a + 5 * b + 25 * c] = v;
    return p;
  };
  auto add = [](TriPoly p, const TriPoly& q) {
    for (int i = 0; i < 125; ++i) p.c[i] += q.c[i];
    return p;
  };
  if (order == 1) {
    basis.push_back(mono(1, 0, 0, 1));
    basis.push_back(mono(0, 1, 0, 1));
    basis.push_back(mono(0, 0, 1, 1));
  } else {  // (v0, v1, v2, e01, e12, e02): lam_i (2 lam_i - 1), 4 lam_i lam_j
    basis.push_back(add(mono(2, 0, 0, 2), mono(1, 0, 0, -1)));
    basis.push_back(add(mono(0, 2, 0, 2), mono(0, 1, 0, -1)));
    basis.push_back(add(mono(0, 0, 2, 2), mono(0, 0, 1, -1)));
    basis.push_back(mono(1, 1, 0, 4));
    basis.push_back(mono(0, 1, 1, 4));
    basis.push_back(mono(1, 0, 1, 4));
  }
  int n = (int)basis.size();
  std::vector<double> M(n * n);
  for (int a = 0; a < n; ++a)
    for (int b = a; b < n; ++b) M[a * n + b] = M[b * n + a] = tri_integral(tri_mul(basis[a], basis[b]));
  return M;
}

// Plane-triangle stiffness (order P1/P2, basis order as tri_mass_unit) of the triangle with
// vertices Y[3][2]: closed form, int lam_i lam_j = |T|(1 + d_ij)/12, int lam_i = |T|/3.
std::vector<double> tri_stiffness(int order, const double Y[3][2]) {
  const double J[2][2] = {{Y[1][0] - Y[0][0], Y[2][0] - Y[0][0]}, {Y[1][1] - Y[0][1], Y[2][1] - Y[0][1]}};
  const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double area = std::fabs(det) / 2.0;
  double g[3][2];
  g[1][0] = J[1][1] / det;
  g[1][1] = -J[0][1] / det;
  g[2][0] = -J[1][0] / det;
  g[2][1] = J[0][0] / det;
  g[0][0] = -(g[1][0] + g[2][0]);
  g[0][1] = -(g[1][1] + g[2][1]);
  const int n = order == 1 ? 3 : 6;
  std::vector<double> K(n * n);
  if (order == 1) {
    for (int a = 0; a < 3; ++a)
      for (int b = a; b < 3; ++b) K[a * 3 + b] = K[b * 3 + a] = area * (g[a][0] * g[b][0] + g[a][1] * g[b][1]);
    return K;
  }
  // grad phi_a = sum_m (A[a][m] + sum_k B[a][m][k] lam_k) grad lam_m
  double A[6][3] = {}, B[6][3][3] = {};
  for (int i = 0; i < 3; ++i) {
    A[i][i] = -1.0;
    B[i][i][i] = 4.0;
  }
  const int e[3][2] = {{0, 1}, {1, 2}, {0, 2}};
  for (int k = 0; k < 3; ++k) {
    B[3 + k][e[k][0]][e[k][1]] = 4.0;
    B[3 + k][e[k][1]][e[k][0]] = 4.0;
  }
  auto lin = [](double a, const double* b, double ap, const double* bp) {
    double sb = 0, sbp = 0, qd = 0;
    for (int k = 0; k < 3; ++k) {
      sb += b[k];
      sbp += bp[k];
      for (int l = 0; l < 3; ++l) qd += b[k] * bp[l] * (k == l ? 2.0 : 1.0) / 12.0;
    }
    return a * ap + (a * sbp + ap * sb) / 3.0 + qd;
  };
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) {
      double s = 0.0;
      for (int m = 0; m < 3; ++m)
        for (int nn = 0; nn < 3; ++nn) {
          const double gg = g[m][0] * g[nn][0] + g[m][1] * g[nn][1];
          if (gg == 0.0) continue;
          s += gg * lin(A[a][m], B[a][m], A[b][nn], B[b][nn]);
        }
      K[a * 6 + b] = K[b * 6 + a] = area * s;
    }
  return K;
}

}  // namespace

std::vector<std::array<int, 3>> tet_local_offsets(int t, int order) {
  int v[4][3];
  tet_vertices(t, v);
  std::vector<std::array<int, 3>> out;
  if (order == 1) {
    for (int a = 0; a < 4; ++a) out.push_back({v[a][0], v[a][1], v[a][2]});
  } else {
    for (int a = 0; a < 4; ++a) out.push_back({2 * v[a][0], 2 * v[a][1], 2 * v[a][2]});
    for (int e = 0; e < 6; ++e) {
      int i = kEdge[e][0], j = kEdge[e][1];
      out.push_back({v[i][0] + v[j][0], v[i][1] + v[j][1], v[i][2] + v[j][2]});
    }
  }
  return out;
}

void element_stiffness(int order, const double h[3], std::vector<double>& Ke, double& vol) {
  const int nloc = order == 1 ? 4 : 10;
  Ke.assign(6 * nloc * nloc, 0.0);
  double A[10][4], B[10][4][4];
  p2_gradient_coeffs(A, B);
  for (int t = 0; t < 6; ++t) {
    int v[4][3];
    tet_vertices(t, v);
    double X[4][3], g[4][3];
    for (int a = 0; a < 4; ++a)
      for (int d = 0; d < 3; ++d) X[a][d] = v[a][d] * h[d];
    bary_gradients(X, g, vol);
    double* K = &Ke[t * nloc * nloc];
    for (int a = 0; a < nloc; ++a)
      for (int b = a; b < nloc; ++b) {
        double s = 0.0;
        if (order == 1) {
          s = vol * dot3(g[a], g[b]);
        } else {
          for (int m = 0; m < 4; ++m)
            for (int n = 0; n < 4; ++n) {
              double gg = dot3(g[m], g[n]);
              if (gg == 0.0) continue;
              s += gg * lin_product_integral(A[a][m], B[a][m], A[b][n], B[b][n]);
            }
          s *= vol;
        }
        K[a * nloc + b] = K[b * nloc + a] = s;
      }
  }
}

void tet_bary_gradients(int t, const double h[3], std::vector<double>& out) {
  int v[4][3];
  tet_vertices(t, v);
  double X[4][3], g[4][3], vol;
  for (int a = 0; a < 4; ++a)
    for (int d = 0; d < 3; ++d) X[a][d] = v[a][d] * h[d];
  bary_gradients(X, g, vol);
  out.assign(12, 0.0);
  for (int a = 0; a < 4; ++a)
    for (int d = 0; d < 3; ++d) out[a * 3 + d] = g[a][d];
}

StencilTables build_stencil_tables(int order, const double h[3]) {
  StencilTables T;
  T.order = order;
  T.nclass = order * order * order;
  const int nloc = order == 1 ? 4 : 10;
  std::vector<double> Ke;
  double vol;
  element_stiffness(order, h, Ke, vol);
  std::vector<std::vector<std::array<int, 3>>> offs(6);
  for (int t = 0; t < 6; ++t) offs[t] = tet_local_offsets(t, order);
  // int_T phi_a: P1 |T|/4; P2 vertex -|T|/20, edge |T|/5 (exact).
  std::vector<double> lw(nloc);
  for (int a = 0; a < nloc; ++a) lw[a] = order == 1 ? vol / 4.0 : (a < 4 ? -vol / 20.0 : vol / 5.0);

  T.col_begin.push_back(0);
  T.load_begin.push_back(0);
  for (int rz = 0; rz < order; ++rz)
    for (int ry = 0; ry < order; ++ry)
      for (int rx = 0; rx < order; ++rx) {
        const int r[3] = {rx, ry, rz};
        // incidences (dc, t, a) in element order: cells lexicographic (z, y, x), then tet
        struct Inc {
          int dc[3], t, a;
        };
        std::vector<Inc> inc;
        for (int dz = -1; dz <= 0; ++dz)
          for (int dy = -1; dy <= 0; ++dy)
            for (int dx = -1; dx <= 0; ++dx)
              for (int t = 0; t < 6; ++t)
                for (int a = 0; a < nloc; ++a) {
                  const int dc[3] = {dx, dy, dz};
                  bool hit = true;
                  for (int d = 0; d < 3; ++d) hit = hit && (order * dc[d] + offs[t][a][d] == r[d]);
                  if (hit) inc.push_back({{dx, dy, dz}, t, a});
                }
        // columns: every node of every incident tet, grouped by offset dQ
        struct Entry {
          int dq[3];
          StiffContrib c;
          int seq;
        };
        std::vector<Entry> ent;
        int seq = 0;
        for (const Inc& I : inc) {
          for (int b = 0; b < nloc; ++b) {
            Entry e;
            for (int d = 0; d < 3; ++d) e.dq[d] = order * I.dc[d] + offs[I.t][b][d] - r[d];
            e.c.dcx = (int8_t)I.dc[0];
            e.c.dcy = (int8_t)I.dc[1];
            e.c.dcz = (int8_t)I.dc[2];
            e.c.tet = (int8_t)I.t;
            e.c.pad = 0;
            e.c.val = Ke[I.t * nloc * nloc + I.a * nloc + b];
            e.seq = seq++;
            ent.push_back(e);
          }
          LoadContrib L;
          L.dcx = (int8_t)I.dc[0];
          L.dcy = (int8_t)I.dc[1];
          L.dcz = (int8_t)I.dc[2];
          L.tet = (int8_t)I.t;
          L.pad = 0;
          L.w = lw[I.a];
          T.loads.push_back(L);
        }
        // sort by column order (dz, dy, dx) -- contract numbering is x fastest -- keeping element order
        std::stable_sort(ent.begin(), ent.end(), [](const Entry& p, const Entry& q) {
          return std::make_tuple(p.dq[2], p.dq[1], p.dq[0], p.seq) < std::make_tuple(q.dq[2], q.dq[1], q.dq[0], q.seq);
        });
        size_t i = 0;
        int ncols = 0;
        while (i < ent.size()) {
          size_t j = i;
          StencilCol sc;
          sc.dx = (int8_t)ent[i].dq[0];
          sc.dy = (int8_t)ent[i].dq[1];
          sc.dz = (int8_t)ent[i].dq[2];
          sc.pad = 0;
          sc.c0 = (int32_t)T.contribs.size();
          while (j < ent.size() && ent[j].dq[0] == ent[i].dq[0] && ent[j].dq[1] == ent[i].dq[1] &&
                 ent[j].dq[2] == ent[i].dq[2]) {
            T.contribs.push_back(ent[j].c);
            ++j;
          }
          sc.c1 = (int32_t)T.contribs.size();
          T.cols.push_back(sc);
          ++ncols;
          i = j;
        }
        T.max_cols = std::max(T.max_cols, ncols);
        T.col_begin.push_back((int32_t)T.cols.size());
        T.load_begin.push_back((int32_t)T.loads.size());
      }
  return T;
}

void interface_mass(int order, int64_t ny, int64_t nz, double hy, double hz, std::vector<int32_t>& rowptr,
                    std::vector<int32_t>& col, std::vector<double>& val, std::vector<double>& sval) {
  const int64_t Ny = order * ny + 1, Nz = order * nz + 1;
  const int64_t nJ = Ny - 2, nK = Nz - 2, n = nJ * nK;
  const std::vector<double> Mu = tri_mass_unit(order);
  const int nl = order == 1 ? 3 : 6;
  const double area = 0.5 * hy * hz;
  const int tris[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{0, 0}, {0, 1}, {1, 1}}};
  struct Trip {
    int64_t r, c;
    double v, s;
  };
  std::vector<Trip> trip;
  for (int64_t ck = 0; ck < nz; ++ck)
    for (int64_t cj = 0; cj < ny; ++cj)
      for (int t = 0; t < 2; ++t) {
        double Y[3][2];
        for (int a = 0; a < 3; ++a) {
          Y[a][0] = tris[t][a][0] * hy;
          Y[a][1] = tris[t][a][1] * hz;
        }
        const std::vector<double> St = tri_stiffness(order, Y);
        int pts[6][2];
        for (int a = 0; a < 3; ++a) {
          pts[a][0] = order * tris[t][a][0];
          pts[a][1] = order * tris[t][a][1];
        }
        if (order == 2) {
          const int e[3][2] = {{0, 1}, {1, 2}, {0, 2}};
          for (int k = 0; k < 3; ++k)
            for (int d = 0; d < 2; ++d) pts[3 + k][d] = tris[t][e[k][0]][d] + tris[t][e[k][1]][d];
        }
        int64_t gid[6];
        bool fr[6];
        for (int a = 0; a < nl; ++a) {
          int64_t Jp = order * cj + pts[a][0], Kp = order * ck + pts[a][1];
          fr[a] = Jp >= 1 && Jp <= Ny - 2 && Kp >= 1 && Kp <= Nz - 2;
          gid[a] = (Jp - 1) + nJ * (Kp - 1);
        }
        for (int a = 0; a < nl; ++a)
          for (int b = 0; b < nl; ++b)
            if (fr[a] && fr[b]) trip.push_back({gid[a], gid[b], area * Mu[a * nl + b], St[a * nl + b]});
      }
  std::stable_sort(trip.begin(), trip.end(),
                   [](const Trip& p, const Trip& q) { return p.r != q.r ? p.r < q.r : p.c < q.c; });
  rowptr.assign(n + 1, 0);
  col.clear();
  val.clear();
  sval.clear();
  for (size_t i = 0; i < trip.size();) {
    size_t j = i;
    double s = 0.0, st = 0.0;
    while (j < trip.size() && trip[j].r == trip[i].r && trip[j].c == trip[i].c) {
      s += trip[j].v;
      st += trip[j].s;
      ++j;
    }
    col.push_back((int32_t)trip[i].c);
    val.push_back(s);
    sval.push_back(st);
    rowptr[trip[i].r + 1]++;
    i = j;
  }
  for (int64_t r = 0; r < n; ++r) rowptr[r + 1] += rowptr[r];
}

void plan_rank(int nsub, int nranks, int rank, int& s_begin, int& s_end, std::vector<PlanSide>& sides) {
  s_begin = (int)((int64_t)rank * nsub / nranks);
  s_end = (int)((int64_t)(rank + 1) * nsub / nranks);
  sides.clear();
  for (int s = s_begin; s < s_end; ++s)
    for (int plane = 0; plane < 2; ++plane) {  // 0: left plane, 1: right plane
      const bool has = plane == 0 ? s > 0 : s < nsub - 1;
      if (!has) continue;
      const int nbr = plane == 0 ? s - 1 : s + 1;
      PlanSide p;
      p.iface = plane == 0 ? s - 1 : s;
      p.which = plane == 0 ? 1 : 0;
      p.sub = s;
      p.remote = !(nbr >= s_begin && nbr < s_end);
      p.peer = (int)((int64_t)nbr * nranks / nsub);
      sides.push_back(p);
    }
}

std::vector<int64_t> partition_x(int64_t nx, int nsub) {
  std::vector<int64_t> c(nsub + 1, 0);
  int64_t base = nx / nsub, rem = nx % nsub;
  for (int s = 0; s < nsub; ++s) c[s + 1] = c[s] + base + (s < rem ? 1 : 0);
  return c;
}

}  // namespace osm
