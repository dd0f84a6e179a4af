// Host-side geometry of the Kuhn box mesh: element integrals, the per-parity-class
// stencil tables that drive the GPU assembly, the interface-plane mass matrix and
// the x-slab partition.  (PAPER.md:44, 156-157.)
#pragma once
#include <array>
#include <cstdint>
#include <vector>

namespace osm {

// One element contribution K_e[t][a][b] to row node a / column node b of tet t in
// the cell at offset (dcx,dcy,dcz) in {-1,0}^3 from the row's base cell.
struct StiffContrib {
  int8_t dcx, dcy, dcz, tet;
  int32_t pad;
  double val;
};
// One structural column offset dQ of a row class; its contributions are
// contribs[c0, c1) in element order (cell id ascending, then tet).
struct StencilCol {
  int8_t dx, dy, dz, pad;
  int32_t c0, c1;
};
// Load contribution: f_cell * w (w = int_T phi_a) from the tet t of the cell at offset dc.
struct LoadContrib {
  int8_t dcx, dcy, dcz, tet;
  int32_t pad;
  double w;
};

struct StencilTables {
  int order = 0;
  int nclass = 0;                   // order^3 lattice parity classes
  std::vector<int32_t> col_begin;   // nclass + 1
  std::vector<StencilCol> cols;
  std::vector<StiffContrib> contribs;
  std::vector<int32_t> load_begin;  // nclass + 1
  std::vector<LoadContrib> loads;
  int max_cols = 0;
};

// Lattice offsets of the local nodes of Kuhn tet t (t indexes the axis
// permutations in lexicographic order) inside its cell: P1 the 4 vertices
// (0..1), P2 the 4 vertices doubled then the 6 edge midpoints
// (01,02,03,12,13,23) on the refined lattice (0..2).
std::vector<std::array<int, 3>> tet_local_offsets(int t, int order);

// Element stiffness matrices of the 6 tets of a cell of size h (row-major
// nloc x nloc each) and the tet volume.  Exact integration in barycentric
// monomials (int lam_i lam_j = |T|(1+delta_ij)/20, int lam_i = |T|/4).
void element_stiffness(int order, const double h[3], std::vector<double>& Ke, double& vol);

StencilTables build_stencil_tables(int order, const double h[3]);

// Physical barycentric gradients (4 x 3, row-major) of Kuhn tet t of a cell of size h.
void tet_bary_gradients(int t, const double h[3], std::vector<double>& g);

// Interface-plane mass matrix M_Gamma on the free interior points of an x = const
// plane of the (Ny x Nz)-point lattice, CSR in plane-point order (j fastest).
// Triangles: each (j,k) square split along its (j,k)-(j+1,k+1) diagonal.
// Also the tangential stiffness S_Gamma = int grad_tau phi_i . grad_tau phi_j (the OO2 term),
// with exactly the same pattern (sval aligned with val).
void interface_mass(int order, int64_t ny, int64_t nz, double hy, double hz, std::vector<int32_t>& rowptr,
                    std::vector<int32_t>& col, std::vector<double>& val, std::vector<double>& sval);

// Cell starts c_0..c_S of the x-slabs (widths differ by <= 1, remainder to the left).
std::vector<int64_t> partition_x(int64_t nx, int nsub);

// Distribution plan of one rank (host only, no CUDA): subdomain s goes to rank
// floor(s * nranks / nsub); every slab plane that touches another slab is a "side".
struct PlanSide {
  int iface;   // interface index i (between slabs i and i+1)
  int which;   // 0: this slab is the left slab of the interface (its right plane), 1: the right slab
  int sub;     // global subdomain id owning the side
  int remote;  // neighbour on another rank
  int peer;    // rank of the neighbour slab
};
void plan_rank(int nsub, int nranks, int rank, int& s_begin, int& s_end, std::vector<PlanSide>& sides);

}  // namespace osm
