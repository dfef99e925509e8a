// Host basis construction (basis.cpp) -- internal header, not part of the C-ABI.
#pragma once
#include <stdint.h>

#include <vector>

namespace msim {

struct BasisInput {            // the GLOBAL mesh (every rank builds the same basis)
  int32_t nv = 0, nt = 0;
  const double *X = nullptr;   // (nv,3) rest positions
  const int32_t *tets = nullptr;
  const double *E = nullptr, *rho = nullptr;   // per tet
  std::vector<int32_t> dbc;    // Dirichlet vertices
};

struct BasisOutput {
  int32_t m = 0, n_cg = 20, n_holes = 0;
  double hop_radius = 0.0;
  std::vector<double> origins;           // (m,3)
  std::vector<int64_t> vptr;             // (nv+1)
  std::vector<int32_t> handle;
  std::vector<double> phi, phi_affine;
  double affine_origin[3] = {0, 0, 0};
  std::vector<int32_t> cluster, centroid_vertex;
  double t_kmeans = 0, t_connect = 0, t_solve = 0, t_total = 0;
};

void build_basis_host(const BasisInput &in, int32_t m, uint64_t seed, BasisOutput &out);

}  // namespace msim
