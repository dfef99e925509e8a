// ms_basis_build: the SMS / affine basis construction on the host (SURVEY §8(b)
// `ms_basis_build`; §3.5, §3.6, §3.7.2; readings
// Q14-Q17, R9, B1, B2 in DESIGN.md).  Native C++ with OpenMP over handles.
//
// The steps follow precompute/basis.py (the input generator the oracle uses) in the same order,
// with the same random draws and tie rules, so the two produce the same partition, centroid
// vertices and handle lists; the weights agree to the rounding of the subdomain solves:
//  1. tet volumes and barycentres; kmeans++ seeding on the barycentres weighted by volume with
//     draws k = 0..m-1 of the counter-based SplitMix64 stream of `seed`; Lloyd iterations
//     (exact squared distances, ties -> lowest centre) to an assignment fixed point or 100 rounds.
//  2. face-connectivity: keep the largest face-connected component of every cluster (ties ->
//     the component holding the lowest tet), move the others to the face-adjacent cluster with
//     the most shared faces (ties -> lowest cluster id); at most 20 rounds.  Empty clusters are
//     dropped.
//  3. centroid vertex c_i = cluster vertex nearest the volume-weighted barycentre (Q15); handles
//     relabelled in lexicographic (x, y, z) order of c_i.
//  4. subdomain T_i = cluster i + clusters sharing a vertex with it (R9); K = L_s M^-1 L_s with
//     L_s the P1 Laplacian weighted by E/median(E) and M the lumped volume (Q17); K u = 0 with
//     u(c_i) = 1, u = 0 at the neighbour centroids, on the internal boundary and at Dirichlet
//     vertices; the free block is solved by an envelope Cholesky in reverse
//     Cuthill-McKee order.  Clip u_pos = max(u, 0).
//  5. Dirichlet weight u_DBC, POU normalisation, coverage-hole
//     repair (B1), affine weight 1 - phi_DBC at the centre of mass (Q14).
//  6. N_cg = closer of 20 / 40 to the mean over partitions of the max edge-hop distance from the
//     centroid vertex (Q7).
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>

#include "common.cuh"
#include "basis.h"

namespace msim {

namespace {

double splitmix64_uniform(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

inline double sqd(const double *p, const double *c) {
  const double dx = p[0] - c[0], dy = p[1] - c[1], dz = p[2] - c[2];
  return (dx * dx + dy * dy) + dz * dz;
}

// index i with cdf[i-1] <= u cdf[n-1] < cdf[i] (cdf = sequential prefix sums of p)
int64_t weighted_pick(const std::vector<double> &p, double u, std::vector<double> &cdf) {
  const int64_t n = (int64_t)p.size();
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) cdf[i] = (s += p[i]);
  const double t = u * cdf[n - 1];
  const int64_t idx = std::upper_bound(cdf.begin(), cdf.end(), t) - cdf.begin();
  return std::min(idx, n - 1);
}

// uniform grid over the centres for exact nearest-centre queries
struct CentreGrid {
  double lo[3], h;
  int n[3];
  std::vector<int32_t> start, ids;
  void build(const std::vector<double> &C, int m) {
    double hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = 1e300;
      hi[d] = -1e300;
    }
    for (int i = 0; i < m; ++i)
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], C[3 * i + d]);
        hi[d] = std::max(hi[d], C[3 * i + d]);
      }
    double vol = 1.0;
    for (int d = 0; d < 3; ++d) vol *= std::max(hi[d] - lo[d], 1e-12);
    h = std::cbrt(vol / std::max(m, 1)) * 1.5;
    for (int d = 0; d < 3; ++d) n[d] = std::max(1, std::min(256, (int)std::ceil((hi[d] - lo[d]) / h) + 1));
    start.assign((size_t)n[0] * n[1] * n[2] + 1, 0);
    std::vector<int64_t> cell(m);
    for (int i = 0; i < m; ++i) {
      int q[3];
      for (int d = 0; d < 3; ++d) q[d] = std::min(n[d] - 1, std::max(0, (int)((C[3 * i + d] - lo[d]) / h)));
      cell[i] = ((int64_t)q[0] * n[1] + q[1]) * n[2] + q[2];
      start[cell[i] + 1]++;
    }
    for (size_t k = 0; k + 1 < start.size(); ++k) start[k + 1] += start[k];
    ids.resize(m);
    std::vector<int32_t> fill(start.begin(), start.end() - 1);
    for (int i = 0; i < m; ++i) ids[fill[cell[i]]++] = i;   // ascending ids within a cell
  }
  // exact nearest (squared distance, ties -> lowest id): search cube shells until the shell's
  // lower distance bound exceeds the best found
  int nearest(const double *p, const std::vector<double> &C) const {
    int q[3];
    for (int d = 0; d < 3; ++d) q[d] = (int)std::floor((p[d] - lo[d]) / h);
    double best = INFINITY;
    int bi = -1;
    const int rmax = std::max(n[0], std::max(n[1], n[2])) + 1;
    for (int r = 0; r <= rmax; ++r) {
      if (bi >= 0) {
        // every cell at Chebyshev ring r is at least (r-1) h away along some axis
        const double lb = (r - 1) * h;
        if (lb > 0 && lb * lb > best) break;
      }
      for (int a = q[0] - r; a <= q[0] + r; ++a) {
        if (a < 0 || a >= n[0]) continue;
        for (int b = q[1] - r; b <= q[1] + r; ++b) {
          if (b < 0 || b >= n[1]) continue;
          for (int cc = q[2] - r; cc <= q[2] + r; ++cc) {
            if (cc < 0 || cc >= n[2]) continue;
            if (std::max(std::abs(a - q[0]), std::max(std::abs(b - q[1]), std::abs(cc - q[2]))) != r) continue;
            const int64_t cell = ((int64_t)a * n[1] + b) * n[2] + cc;
            for (int32_t k = start[cell]; k < start[cell + 1]; ++k) {
              const int i = ids[k];
              const double dd = sqd(p, &C[3 * (size_t)i]);
              if (dd < best || (dd == best && i < bi)) {
                best = dd;
                bi = i;
              }
            }
          }
        }
      }
    }
    return bi;
  }
};

// ---------------------------------------------------------------- sparse symmetric solve
// Envelope Cholesky of an SPD matrix given in CSR (full symmetric pattern), RCM-ordered.
struct EnvelopeSolver {
  int n = 0;
  std::vector<int32_t> perm, iperm;   // perm[new] = old
  std::vector<int64_t> rstart;        // row i stored for columns first[i]..i at rstart[i]
  std::vector<int32_t> first;
  std::vector<double> L;

  void rcm(const std::vector<int32_t> &rp, const std::vector<int32_t> &ci) {
    perm.clear();
    std::vector<int32_t> deg(n);
    for (int i = 0; i < n; ++i) deg[i] = rp[i + 1] - rp[i];
    std::vector<char> seen(n, 0);
    std::vector<int32_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return deg[a] < deg[b]; });
    std::vector<int32_t> nb;
    for (int s : order) {
      if (seen[s]) continue;
      size_t head = perm.size();
      perm.push_back(s);
      seen[s] = 1;
      while (head < perm.size()) {
        const int v = perm[head++];
        nb.clear();
        for (int32_t k = rp[v]; k < rp[v + 1]; ++k)
          if (!seen[ci[k]]) {
            seen[ci[k]] = 1;
            nb.push_back(ci[k]);
          }
        std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
        perm.insert(perm.end(), nb.begin(), nb.end());
      }
    }
    std::reverse(perm.begin(), perm.end());
    iperm.assign(n, 0);
    for (int i = 0; i < n; ++i) iperm[perm[i]] = i;
  }

  // returns false if a pivot is not positive
  bool factor(const std::vector<int32_t> &rp, const std::vector<int32_t> &ci, const std::vector<double> &val) {
    rcm(rp, ci);
    first.assign(n, 0);
    for (int i = 0; i < n; ++i) {
      const int o = perm[i];
      int f = i;
      for (int32_t k = rp[o]; k < rp[o + 1]; ++k) f = std::min(f, (int)iperm[ci[k]]);
      first[i] = f;
    }
    rstart.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) rstart[i + 1] = rstart[i] + (i - first[i] + 1);
    L.assign(rstart[n], 0.0);
    for (int i = 0; i < n; ++i) {
      const int o = perm[i];
      for (int32_t k = rp[o]; k < rp[o + 1]; ++k) {
        const int j = iperm[ci[k]];
        if (j <= i) L[rstart[i] + (j - first[i])] += val[k];
      }
    }
    for (int i = 0; i < n; ++i) {
      double *Li = &L[rstart[i]];
      const int fi = first[i];
      for (int j = fi; j < i; ++j) {
        const int fj = first[j];
        const int k0 = std::max(fi, fj);
        const double *Lj = &L[rstart[j]];
        double s = Li[j - fi];
        const double *a = Li + (k0 - fi), *b = Lj + (k0 - fj);
        const int len = j - k0;
        double acc = 0.0;
        for (int k = 0; k < len; ++k) acc += a[k] * b[k];
        s -= acc;
        Li[j - fi] = s / Lj[j - fj];
      }
      double d = Li[i - fi];
      double acc = 0.0;
      for (int k = 0; k < i - fi; ++k) acc += Li[k] * Li[k];
      d -= acc;
      if (!(d > 0.0)) return false;
      Li[i - fi] = std::sqrt(d);
    }
    return true;
  }

  void solve(const std::vector<double> &b, std::vector<double> &x) const {
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int i = 0; i < n; ++i) {   // L y = b
      const double *Li = &L[rstart[i]];
      double s = y[i];
      for (int k = first[i]; k < i; ++k) s -= Li[k - first[i]] * y[k];
      y[i] = s / Li[i - first[i]];
    }
    for (int i = n - 1; i >= 0; --i) {   // L^T x = y (column sweep)
      const double *Li = &L[rstart[i]];
      y[i] /= Li[i - first[i]];
      const double yi = y[i];
      for (int k = first[i]; k < i; ++k) y[k] -= Li[k - first[i]] * yi;
    }
    x.assign(n, 0.0);
    for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
  }
};

// Solve K u = 0 (K = L M^-1 L on the sub-mesh `tsub`) with u = 1 on `ones`, u = 0 on `zeros`;
// verts: sorted global vertex ids of the sub-mesh.  Returns u over verts.
bool constrained_bilaplacian(const std::vector<int32_t> &verts, const std::vector<int32_t> &tsub,
                             const int32_t *tets, const std::vector<double> &Kl, const std::vector<double> &vol,
                             const std::vector<int32_t> &ones, const std::vector<int32_t> &zeros,
                             std::vector<double> &u) {
  const int n = (int)verts.size();
  auto loc = [&](int32_t g) { return (int)(std::lower_bound(verts.begin(), verts.end(), g) - verts.begin()); };
  // L_s (CSR, summed in tet order) and lumped M
  std::vector<std::vector<std::pair<int, double>>> rows(n);
  std::vector<double> M(n, 0.0);
  for (int32_t e : tsub) {
    int l[4];
    for (int a = 0; a < 4; ++a) l[a] = loc(tets[4 * (size_t)e + a]);
    for (int a = 0; a < 4; ++a) {
      M[l[a]] += vol[e] / 4.0;
      for (int b = 0; b < 4; ++b) rows[l[a]].push_back({l[b], Kl[16 * (size_t)e + 4 * a + b]});
    }
  }
  std::vector<int32_t> Lp(n + 1, 0), Lc;
  std::vector<double> Lv;
  for (int i = 0; i < n; ++i) {
    auto &r = rows[i];
    std::stable_sort(r.begin(), r.end(), [](const auto &a, const auto &b) { return a.first < b.first; });
    for (size_t k = 0; k < r.size(); ++k) {
      if (k > 0 && r[k].first == r[k - 1].first) {
        Lv.back() += r[k].second;
      } else {
        Lc.push_back(r[k].first);
        Lv.push_back(r[k].second);
      }
    }
    Lp[i + 1] = (int32_t)Lc.size();
    std::vector<std::pair<int, double>>().swap(r);
  }
  // constraints
  std::vector<char> cons(n, 0);
  std::vector<double> uc(n, 0.0);
  for (int32_t g : zeros) cons[loc(g)] = 1;
  for (int32_t g : ones) {
    cons[loc(g)] = 1;
    uc[loc(g)] = 1.0;
  }
  std::vector<int32_t> fidx(n, -1);
  int nf = 0;
  for (int i = 0; i < n; ++i)
    if (!cons[i]) fidx[i] = nf++;
  u.assign(n, 0.0);
  for (int i = 0; i < n; ++i) u[i] = uc[i];
  if (nf == 0) return true;
  // K = L M^-1 L row by row (dense accumulator); split into Kff and rhs = -Kfc uc
  std::vector<int32_t> Kp(nf + 1, 0), Kc;
  std::vector<double> Kv, rhs(nf, 0.0);
  std::vector<double> acc(n, 0.0);
  std::vector<int32_t> mark(n, -1), nz;
  for (int i = 0; i < n; ++i) {
    if (cons[i]) continue;
    nz.clear();
    for (int32_t a = Lp[i]; a < Lp[i + 1]; ++a) {
      const int k = Lc[a];
      const double lik = Lv[a] / M[k];
      for (int32_t b = Lp[k]; b < Lp[k + 1]; ++b) {
        const int j = Lc[b];
        if (mark[j] != i) {
          mark[j] = i;
          acc[j] = 0.0;
          nz.push_back(j);
        }
        acc[j] += lik * Lv[b];
      }
    }
    std::sort(nz.begin(), nz.end());
    double r = 0.0;
    for (int j : nz) {
      if (cons[j]) {
        r -= acc[j] * uc[j];
      } else {
        Kc.push_back(fidx[j]);
        Kv.push_back(acc[j]);
      }
    }
    rhs[fidx[i]] = r;
    Kp[fidx[i] + 1] = (int32_t)Kc.size();
  }
  EnvelopeSolver es;
  es.n = nf;
  if (!es.factor(Kp, Kc, Kv)) return false;
  std::vector<double> xf;
  es.solve(rhs, xf);
  for (int i = 0; i < n; ++i)
    if (!cons[i]) u[i] = xf[fidx[i]];
  return true;
}

double median_of(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return (n % 2) ? v[n / 2] : (v[n / 2 - 1] + v[n / 2]) / 2.0;
}

}  // namespace

void build_basis_host(const BasisInput &in, int32_t m_req, uint64_t seed, BasisOutput &out) {
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  const int32_t nv = in.nv, nt = in.nt;
  const double *X = in.X;
  const int32_t *tets = in.tets;
  MS_REQUIRE(m_req > 0 && m_req <= nt, MS_ERR_ARG, "ms_basis_build: need 0 < m <= n_tets");

  // ---- 1. volumes, barycentres, kmeans++, Lloyd
  std::vector<double> vol(nt), P(3 * (size_t)nt);
#pragma omp parallel for schedule(static)
  for (int32_t e = 0; e < nt; ++e) {
    const int32_t *t = tets + 4 * (size_t)e;
    double a[3], b[3], c[3];
    for (int d = 0; d < 3; ++d) {
      a[d] = X[3 * t[1] + d] - X[3 * t[0] + d];
      b[d] = X[3 * t[2] + d] - X[3 * t[0] + d];
      c[d] = X[3 * t[3] + d] - X[3 * t[0] + d];
    }
    const double det = a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) +
                       a[2] * (b[0] * c[1] - b[1] * c[0]);
    vol[e] = det / 6.0;
    for (int d = 0; d < 3; ++d)
      P[3 * (size_t)e + d] = (((X[3 * t[0] + d] + X[3 * t[1] + d]) + X[3 * t[2] + d]) + X[3 * t[3] + d]) / 4.0;
  }
  int32_t m = m_req;
  std::vector<double> C(3 * (size_t)m);
  {
    std::vector<double> cdf(nt), p(nt), d2(nt);
    int64_t idx = weighted_pick(vol, splitmix64_uniform(seed, 0), cdf);
    for (int d = 0; d < 3; ++d) C[d] = P[3 * idx + d];
#pragma omp parallel for schedule(static)
    for (int32_t e = 0; e < nt; ++e) d2[e] = sqd(&P[3 * (size_t)e], &C[0]);
    for (int k = 1; k < m; ++k) {
#pragma omp parallel for schedule(static)
      for (int32_t e = 0; e < nt; ++e) p[e] = vol[e] * d2[e];
      idx = weighted_pick(p, splitmix64_uniform(seed, k), cdf);
      for (int d = 0; d < 3; ++d) C[3 * k + d] = P[3 * idx + d];
      const double *ck = &C[3 * k];
#pragma omp parallel for schedule(static)
      for (int32_t e = 0; e < nt; ++e) d2[e] = std::min(d2[e], sqd(&P[3 * (size_t)e], ck));
    }
  }
  std::vector<int32_t> assign(nt, -1), a_new(nt);
  for (int it = 0; it < 100; ++it) {
    CentreGrid grid;
    grid.build(C, m);
#pragma omp parallel for schedule(static)
    for (int32_t e = 0; e < nt; ++e) a_new[e] = grid.nearest(&P[3 * (size_t)e], C);
    if (it > 0 && a_new == assign) break;
    assign = a_new;
    std::vector<double> W(m, 0.0), S(3 * (size_t)m, 0.0);
    for (int32_t e = 0; e < nt; ++e) W[assign[e]] += vol[e];
    for (int d = 0; d < 3; ++d)
      for (int32_t e = 0; e < nt; ++e) S[3 * (size_t)assign[e] + d] += vol[e] * P[3 * (size_t)e + d];
    for (int i = 0; i < m; ++i)
      if (W[i] > 0)
        for (int d = 0; d < 3; ++d) C[3 * i + d] = S[3 * i + d] / W[i];
  }
  const auto t_kmeans = clk::now();

  // ---- 2. face connectivity
  std::vector<int32_t> fa, fb;   // face-adjacent tet pairs
  {
    std::vector<std::pair<uint64_t, int64_t>> faces((size_t)4 * nt);
    static const int loc3[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
#pragma omp parallel for schedule(static)
    for (int32_t e = 0; e < nt; ++e)
      for (int f = 0; f < 4; ++f) {
        int64_t v[3] = {tets[4 * (size_t)e + loc3[f][0]], tets[4 * (size_t)e + loc3[f][1]], tets[4 * (size_t)e + loc3[f][2]]};
        std::sort(v, v + 3);
        faces[4 * (size_t)e + f] = {(uint64_t)(((v[0] << 21) + v[1]) << 21) + (uint64_t)v[2], 4 * (int64_t)e + f};
      }
    std::sort(faces.begin(), faces.end());
    for (size_t k = 0; k + 1 < faces.size(); ++k)
      if (faces[k].first == faces[k + 1].first) {
        fa.push_back((int32_t)(faces[k].second / 4));
        fb.push_back((int32_t)(faces[k + 1].second / 4));
      }
  }
  std::vector<int32_t> fptr(nt + 1, 0), fadj(2 * fa.size());
  for (size_t k = 0; k < fa.size(); ++k) {
    fptr[fa[k] + 1]++;
    fptr[fb[k] + 1]++;
  }
  for (int32_t e = 0; e < nt; ++e) fptr[e + 1] += fptr[e];
  {
    std::vector<int32_t> fill(fptr.begin(), fptr.end() - 1);
    for (size_t k = 0; k < fa.size(); ++k) {
      fadj[fill[fa[k]]++] = fb[k];
      fadj[fill[fb[k]]++] = fa[k];
    }
  }
  for (int round = 0; round < 20; ++round) {
    // components of the same-cluster face graph, labelled in order of their lowest tet
    std::vector<int32_t> comp(nt, -1), stack;
    int32_t ncomp = 0;
    for (int32_t s = 0; s < nt; ++s) {
      if (comp[s] >= 0) continue;
      comp[s] = ncomp;
      stack.assign(1, s);
      while (!stack.empty()) {
        const int32_t e = stack.back();
        stack.pop_back();
        for (int32_t k = fptr[e]; k < fptr[e + 1]; ++k) {
          const int32_t f = fadj[k];
          if (comp[f] < 0 && assign[f] == assign[e]) {
            comp[f] = ncomp;
            stack.push_back(f);
          }
        }
      }
      ncomp++;
    }
    std::vector<int64_t> size(ncomp, 0);
    std::vector<int32_t> ccl(ncomp);
    for (int32_t e = 0; e < nt; ++e) {
      size[comp[e]]++;
      ccl[comp[e]] = assign[e];
    }
    std::vector<int32_t> keep_comp(m, -1);   // per cluster: the kept (largest, lowest-id) component
    for (int32_t q = 0; q < ncomp; ++q) {
      const int32_t cl = ccl[q];
      if (keep_comp[cl] < 0 || size[q] > size[keep_comp[cl]]) keep_comp[cl] = q;
    }
    bool any_bad = false;
    std::map<std::pair<int32_t, int32_t>, int64_t> votes;
    for (int32_t e = 0; e < nt; ++e) {
      if (keep_comp[assign[e]] == comp[e]) continue;
      any_bad = true;
      for (int32_t k = fptr[e]; k < fptr[e + 1]; ++k) {
        const int32_t f = fadj[k];
        if (assign[f] != assign[e]) votes[{comp[e], assign[f]}]++;
      }
    }
    if (!any_bad) break;
    std::map<int32_t, std::pair<int32_t, int64_t>> target;
    for (const auto &kv : votes) {   // sorted by (component, cluster): ties -> lowest cluster
      auto it = target.find(kv.first.first);
      if (it == target.end() || kv.second > it->second.second) target[kv.first.first] = {kv.first.second, kv.second};
    }
    std::vector<int32_t> old = assign;
    for (int32_t e = 0; e < nt; ++e) {
      if (keep_comp[old[e]] == comp[e]) continue;
      auto it = target.find(comp[e]);
      if (it != target.end()) assign[e] = it->second.first;
    }
  }
  {   // drop empty clusters
    std::vector<int32_t> used(m, 0), remap(m, -1);
    for (int32_t e = 0; e < nt; ++e) used[assign[e]] = 1;
    int32_t k = 0;
    for (int i = 0; i < m; ++i)
      if (used[i]) remap[i] = k++;
    for (int32_t e = 0; e < nt; ++e) assign[e] = remap[assign[e]];
    m = k;
  }
  const auto t_conn = clk::now();

  // ---- 3. centroid vertices, relabelling
  std::vector<int32_t> cv(m);
  {
    std::vector<double> W(m, 0.0), B(3 * (size_t)m, 0.0);
    for (int32_t e = 0; e < nt; ++e) W[assign[e]] += vol[e];
    for (int d = 0; d < 3; ++d)
      for (int32_t e = 0; e < nt; ++e) B[3 * (size_t)assign[e] + d] += vol[e] * P[3 * (size_t)e + d];
    for (int i = 0; i < m; ++i)
      for (int d = 0; d < 3; ++d) B[3 * i + d] /= W[i];
    std::vector<double> best(m, INFINITY);
    std::vector<int32_t> bv(m, INT32_MAX);
    for (int32_t e = 0; e < nt; ++e) {
      const int i = assign[e];
      for (int a = 0; a < 4; ++a) {
        const int32_t v = tets[4 * (size_t)e + a];
        const double dd = sqd(&X[3 * (size_t)v], &B[3 * i]);
        if (dd < best[i] || (dd == best[i] && v < bv[i])) {
          best[i] = dd;
          bv[i] = v;
        }
      }
    }
    std::vector<int32_t> order(m);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      const double *pa = &X[3 * (size_t)bv[a]], *pb = &X[3 * (size_t)bv[b]];
      if (pa[0] != pb[0]) return pa[0] < pb[0];
      if (pa[1] != pb[1]) return pa[1] < pb[1];
      return pa[2] < pb[2];
    });
    std::vector<int32_t> newid(m);
    for (int k = 0; k < m; ++k) newid[order[k]] = k;
    for (int32_t e = 0; e < nt; ++e) assign[e] = newid[assign[e]];
    for (int k = 0; k < m; ++k) cv[k] = bv[order[k]];
  }

  // ---- 4. subdomains and bilaplacian solves
  // vertex -> clusters (sorted unique), cluster -> vertex-sharing clusters (incl. itself)
  std::vector<int32_t> vtc_ptr(nv + 1, 0), vtc;
  {
    std::vector<std::vector<int32_t>> vc(nv);
    for (int32_t e = 0; e < nt; ++e)
      for (int a = 0; a < 4; ++a) vc[tets[4 * (size_t)e + a]].push_back(assign[e]);
    for (int32_t v = 0; v < nv; ++v) {
      auto &l = vc[v];
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
      vtc.insert(vtc.end(), l.begin(), l.end());
      vtc_ptr[v + 1] = (int32_t)vtc.size();
      std::vector<int32_t>().swap(l);
    }
  }
  std::vector<std::vector<int32_t>> nbrs(m);
  for (int32_t v = 0; v < nv; ++v)
    for (int32_t a = vtc_ptr[v]; a < vtc_ptr[v + 1]; ++a)
      for (int32_t b = vtc_ptr[v]; b < vtc_ptr[v + 1]; ++b) nbrs[vtc[a]].push_back(vtc[b]);
  for (auto &l : nbrs) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  std::vector<int32_t> vert_tet_count(nv, 0);
  for (int64_t k = 0; k < 4 * (int64_t)nt; ++k) vert_tet_count[tets[k]]++;
  // weighted P1 Laplacians per tet: V w G G^T (G rows: barycentric gradients)
  std::vector<double> Kl(16 * (size_t)nt);
  {
    std::vector<double> E(in.E, in.E + nt);
    const double Emed = median_of(E);
#pragma omp parallel for schedule(static)
    for (int32_t e = 0; e < nt; ++e) {
      const int32_t *t = tets + 4 * (size_t)e;
      double D[3][3];   // rows = edge vectors
      for (int r = 0; r < 3; ++r)
        for (int d = 0; d < 3; ++d) D[r][d] = X[3 * t[r + 1] + d] - X[3 * t[0] + d];
      const double det = D[0][0] * (D[1][1] * D[2][2] - D[1][2] * D[2][1]) -
                         D[0][1] * (D[1][0] * D[2][2] - D[1][2] * D[2][0]) +
                         D[0][2] * (D[1][0] * D[2][1] - D[1][1] * D[2][0]);
      double Inv[3][3];   // D^-1 by the adjugate
      Inv[0][0] = (D[1][1] * D[2][2] - D[1][2] * D[2][1]) / det;
      Inv[0][1] = (D[0][2] * D[2][1] - D[0][1] * D[2][2]) / det;
      Inv[0][2] = (D[0][1] * D[1][2] - D[0][2] * D[1][1]) / det;
      Inv[1][0] = (D[1][2] * D[2][0] - D[1][0] * D[2][2]) / det;
      Inv[1][1] = (D[0][0] * D[2][2] - D[0][2] * D[2][0]) / det;
      Inv[1][2] = (D[0][2] * D[1][0] - D[0][0] * D[1][2]) / det;
      Inv[2][0] = (D[1][0] * D[2][1] - D[1][1] * D[2][0]) / det;
      Inv[2][1] = (D[0][1] * D[2][0] - D[0][0] * D[2][1]) / det;
      Inv[2][2] = (D[0][0] * D[1][1] - D[0][1] * D[1][0]) / det;
      double G[4][3];   // gradient of barycentric k (k = 1..3) = column k-1 of D^-1; g0 = -sum
      for (int k = 0; k < 3; ++k)
        for (int d = 0; d < 3; ++d) G[k + 1][d] = Inv[d][k];
      for (int d = 0; d < 3; ++d) G[0][d] = -(G[1][d] + G[2][d] + G[3][d]);
      const double s = (det / 6.0) * (in.E[e] / Emed);
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b)
          Kl[16 * (size_t)e + 4 * a + b] = (G[a][0] * G[b][0] + G[a][1] * G[b][1] + G[a][2] * G[b][2]) * s;
    }
  }
  std::vector<char> dbc_mask(nv, 0);
  for (int32_t v : in.dbc) dbc_mask[v] = 1;
  // tets per cluster
  std::vector<int32_t> ctp(m + 1, 0), ctets(nt);
  for (int32_t e = 0; e < nt; ++e) ctp[assign[e] + 1]++;
  for (int i = 0; i < m; ++i) ctp[i + 1] += ctp[i];
  {
    std::vector<int32_t> fill(ctp.begin(), ctp.end() - 1);
    for (int32_t e = 0; e < nt; ++e) ctets[fill[assign[e]]++] = e;
  }
  auto subdomain = [&](const std::vector<int32_t> &cls, std::vector<int32_t> &tsub, std::vector<int32_t> &verts,
                       std::vector<int32_t> &inner) {
    tsub.clear();
    for (int32_t c : cls) tsub.insert(tsub.end(), ctets.begin() + ctp[c], ctets.begin() + ctp[c + 1]);
    std::sort(tsub.begin(), tsub.end());
    verts.clear();
    for (int32_t e : tsub)
      for (int a = 0; a < 4; ++a) verts.push_back(tets[4 * (size_t)e + a]);
    std::sort(verts.begin(), verts.end());
    std::vector<int32_t> cnt;
    {   // local incidence counts
      std::vector<int32_t> all = verts;
      verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
      cnt.assign(verts.size(), 0);
      size_t k = 0;
      for (size_t q = 0; q < all.size(); ++q) {
        while (verts[k] != all[q]) ++k;
        cnt[k]++;
      }
    }
    inner.clear();   // internal boundary: vertices also used by tets outside the subdomain
    for (size_t k = 0; k < verts.size(); ++k)
      if (vert_tet_count[verts[k]] > cnt[k]) inner.push_back(verts[k]);
  };
  std::vector<std::vector<int32_t>> res_v(m);
  std::vector<std::vector<double>> res_u(m);
  int bad_solve = -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < m; ++i) {
    std::vector<int32_t> tsub, verts, inner;
    subdomain(nbrs[i], tsub, verts, inner);
    std::vector<int32_t> zeros = inner;
    for (int32_t j : nbrs[i])
      if (j != i) zeros.push_back(cv[j]);
    for (int32_t v : verts)
      if (dbc_mask[v]) zeros.push_back(v);
    std::sort(zeros.begin(), zeros.end());
    zeros.erase(std::unique(zeros.begin(), zeros.end()), zeros.end());
    zeros.erase(std::remove(zeros.begin(), zeros.end(), cv[i]), zeros.end());
    std::vector<double> u;
    if (!constrained_bilaplacian(verts, tsub, tets, Kl, vol, {cv[i]}, zeros, u)) {
#pragma omp critical
      bad_solve = i;
    }
    res_v[i] = std::move(verts);
    res_u[i] = std::move(u);
  }
  MS_REQUIRE(bad_solve < 0, MS_ERR_NOT_SPD, "ms_basis_build: subdomain bilaplacian not SPD");
  std::vector<double> u_dbc(nv, 0.0);
  if (!in.dbc.empty()) {
    std::vector<int32_t> cls;
    for (int32_t v : in.dbc)
      for (int32_t a = vtc_ptr[v]; a < vtc_ptr[v + 1]; ++a) cls.push_back(vtc[a]);
    std::sort(cls.begin(), cls.end());
    cls.erase(std::unique(cls.begin(), cls.end()), cls.end());
    std::vector<int32_t> sub;
    for (int32_t c : cls) sub.insert(sub.end(), nbrs[c].begin(), nbrs[c].end());
    std::sort(sub.begin(), sub.end());
    sub.erase(std::unique(sub.begin(), sub.end()), sub.end());
    std::vector<int32_t> tsub, verts, inner;
    subdomain(sub, tsub, verts, inner);
    std::vector<int32_t> ones(in.dbc.begin(), in.dbc.end());
    std::sort(ones.begin(), ones.end());
    ones.erase(std::unique(ones.begin(), ones.end()), ones.end());
    std::vector<int32_t> zeros = inner;
    for (int32_t c : cls) zeros.push_back(cv[c]);
    std::sort(zeros.begin(), zeros.end());
    zeros.erase(std::unique(zeros.begin(), zeros.end()), zeros.end());
    std::vector<int32_t> z2;
    std::set_difference(zeros.begin(), zeros.end(), ones.begin(), ones.end(), std::back_inserter(z2));
    std::vector<double> u;
    MS_REQUIRE(constrained_bilaplacian(verts, tsub, tets, Kl, vol, ones, z2, u), MS_ERR_NOT_SPD,
               "ms_basis_build: Dirichlet bilaplacian not SPD");
    for (size_t k = 0; k < verts.size(); ++k) u_dbc[verts[k]] = std::max(u[k], 0.0);
  }
  const auto t_solve = clk::now();

  // ---- 5. POU normalisation with coverage-hole repair (B1)
  std::vector<int32_t> rows;
  std::vector<int32_t> hid;
  std::vector<double> uraw;
  for (int i = 0; i < m; ++i) {
    rows.insert(rows.end(), res_v[i].begin(), res_v[i].end());
    hid.insert(hid.end(), res_v[i].size(), i);
    uraw.insert(uraw.end(), res_u[i].begin(), res_u[i].end());
  }
  auto denominators = [&](std::vector<double> &den) {
    den = u_dbc;
    std::vector<double> s(nv, 0.0);
    for (size_t k = 0; k < rows.size(); ++k) s[rows[k]] += std::max(uraw[k], 0.0);
    for (int32_t v = 0; v < nv; ++v) den[v] = s[v] + u_dbc[v];
  };
  std::vector<double> den;
  denominators(den);
  int32_t n_holes = 0;
  {
    std::vector<int64_t> best(nv, -1);
    for (size_t k = 0; k < rows.size(); ++k) {
      const int32_t v = rows[k];
      if (den[v] > 0 || dbc_mask[v]) continue;
      if (best[v] < 0 || uraw[k] > uraw[best[v]]) best[v] = (int64_t)k;   // ties -> first (lowest handle)
    }
    for (int32_t v = 0; v < nv; ++v)
      if (best[v] >= 0) {
        uraw[best[v]] = 1.0;
        n_holes++;
      }
    if (n_holes) denominators(den);
  }
  for (int32_t v = 0; v < nv; ++v)
    MS_REQUIRE(den[v] > 0 || dbc_mask[v], MS_ERR_COVERAGE, "ms_basis_build: coverage hole at a free vertex");
  // vertex-major CSR, handles ascending
  std::vector<int64_t> vp(nv + 1, 0);
  for (size_t k = 0; k < rows.size(); ++k)
    if (uraw[k] > 0 && den[rows[k]] > 0) vp[rows[k] + 1]++;
  for (int32_t v = 0; v < nv; ++v) vp[v + 1] += vp[v];
  out.vptr = vp;
  out.handle.assign(vp[nv], 0);
  out.phi.assign(vp[nv], 0.0);
  {
    std::vector<int64_t> fill(vp.begin(), vp.end() - 1);
    for (size_t k = 0; k < rows.size(); ++k) {   // entries grouped by handle ascending
      const int32_t v = rows[k];
      if (!(uraw[k] > 0 && den[v] > 0)) continue;
      out.handle[fill[v]] = hid[k];
      out.phi[fill[v]++] = uraw[k] / den[v];
    }
  }
  out.phi_affine.assign(nv, 1.0);
  for (int32_t v = 0; v < nv; ++v) {
    const double pd = dbc_mask[v] ? 1.0 : (den[v] > 0 ? u_dbc[v] / den[v] : 0.0);
    out.phi_affine[v] = 1.0 - pd;
  }
  // ---- 6. affine origin (centre of mass), hop radius, N_cg
  {
    std::vector<double> mass(nv, 0.0);
    for (int32_t e = 0; e < nt; ++e)
      for (int a = 0; a < 4; ++a) mass[tets[4 * (size_t)e + a]] += in.rho[e] * vol[e] / 4.0;
    double msum = 0.0, mx[3] = {0, 0, 0};
    for (int32_t v = 0; v < nv; ++v) {
      msum += mass[v];
      for (int d = 0; d < 3; ++d) mx[d] += mass[v] * X[3 * (size_t)v + d];
    }
    for (int d = 0; d < 3; ++d) out.affine_origin[d] = mx[d] / msum;
  }
  {
    // mesh edges (CSR over vertices)
    std::vector<std::vector<int32_t>> adj(nv);
    for (int32_t e = 0; e < nt; ++e)
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b)
          if (a != b) adj[tets[4 * (size_t)e + a]].push_back(tets[4 * (size_t)e + b]);
    for (auto &l : adj) {
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
    }
    std::vector<double> radius(m, 0.0);
#pragma omp parallel for schedule(dynamic, 4)
    for (int i = 0; i < m; ++i) {
      std::vector<int32_t> pv;
      for (int32_t k = ctp[i]; k < ctp[i + 1]; ++k)
        for (int a = 0; a < 4; ++a) pv.push_back(tets[4 * (size_t)ctets[k] + a]);
      std::sort(pv.begin(), pv.end());
      pv.erase(std::unique(pv.begin(), pv.end()), pv.end());
      std::vector<int32_t> dist(pv.size(), -1);
      auto li = [&](int32_t g) {
        auto it = std::lower_bound(pv.begin(), pv.end(), g);
        return (it != pv.end() && *it == g) ? (int)(it - pv.begin()) : -1;
      };
      std::queue<int32_t> q;
      const int s = li(cv[i]);
      dist[s] = 0;
      q.push(s);
      int32_t dmax = 0;
      while (!q.empty()) {
        const int a = q.front();
        q.pop();
        dmax = std::max(dmax, dist[a]);
        for (int32_t g : adj[pv[a]]) {
          const int b = li(g);
          if (b >= 0 && dist[b] < 0) {
            dist[b] = dist[a] + 1;
            q.push(b);
          }
        }
      }
      radius[i] = dmax;
    }
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += radius[i];
    out.hop_radius = s / m;
    out.n_cg = std::fabs(out.hop_radius - 20.0) <= std::fabs(out.hop_radius - 40.0) ? 20 : 40;
  }
  out.m = m;
  out.n_holes = n_holes;
  out.origins.resize(3 * (size_t)m);
  for (int i = 0; i < m; ++i)
    for (int d = 0; d < 3; ++d) out.origins[3 * i + d] = X[3 * (size_t)cv[i] + d];
  out.cluster = assign;
  out.centroid_vertex = cv;
  const auto t_end = clk::now();
  auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  out.t_kmeans = sec(t_start, t_kmeans);
  out.t_connect = sec(t_kmeans, t_conn);
  out.t_solve = sec(t_conn, t_solve);
  out.t_total = sec(t_start, t_end);
}

}  // namespace msim
