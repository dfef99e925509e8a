// Slab partition, halo plan and collective backends (NCCL; in-process hub for one-GPU tests).
// SURVEY §8(e); see dist.h.
#include "dist.h"

#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <numeric>

#include "common.cuh"

namespace msim {

void make_partition(int rank, int world, int32_t nv, const double *X, int32_t nt, const int32_t *tets,
                    Partition &P, std::vector<int32_t> *owner_out) {
  MS_REQUIRE(world >= 1 && rank >= 0 && rank < world, MS_ERR_ARG, "bad rank / world");
  MS_REQUIRE(nv >= world, MS_ERR_ARG, "fewer vertices than ranks");
  P = Partition{};
  P.rank = rank;
  P.world = world;
  P.nv_glob = nv;
  P.nt_glob = nt;
  // owner: slabs along x (vertices in (x, id) order) balanced by element work: a vertex weighs
  // the tets it heads (vertex 0 of the tet, the energy owner) plus one, so slabs of a mesh with
  // density varying along x (the C3 lattice) carry equal numbers of owned tets; cuts never split
  // vertices of equal x (a cube layer stays on one rank)
  std::vector<int32_t> order(nv), owner(nv);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return X[3 * a] < X[3 * b]; });
  {
    std::vector<int64_t> wgt(nv, 1);
    for (int32_t e = 0; e < nt; ++e) wgt[tets[4 * (size_t)e]]++;
    int64_t total = 0;
    for (int32_t v = 0; v < nv; ++v) total += wgt[v];
    int64_t acc = 0;
    int32_t r = 0;
    for (int32_t k = 0; k < nv; ++k) {
      const int32_t v = order[k];
      // advance to the next rank once this rank's share is reached, but only between x values
      if (r < world - 1 && acc * world >= (int64_t)(r + 1) * total &&
          (k == 0 || X[3 * order[k - 1]] != X[3 * v]))
        ++r;
      owner[v] = r;
      acc += wgt[v];
    }
  }
  // local tets: owned first (vertex 0 owned), then the other tets with an owned vertex
  std::vector<int32_t> own_t, oth_t;
  for (int32_t e = 0; e < nt; ++e) {
    const int32_t *t = tets + 4 * (size_t)e;
    bool any = false;
    for (int a = 0; a < 4; ++a) any = any || owner[t[a]] == rank;
    if (!any) continue;
    (owner[t[0]] == rank ? own_t : oth_t).push_back(e);
  }
  P.nt_own = (int32_t)own_t.size();
  P.tet_l2g = own_t;
  P.tet_l2g.insert(P.tet_l2g.end(), oth_t.begin(), oth_t.end());
  P.nt_loc = (int32_t)P.tet_l2g.size();
  // local vertices: owned (by id), then ghosts (by id)
  P.g2l.assign(nv, -1);
  for (int32_t v = 0; v < nv; ++v)
    if (owner[v] == rank) {
      P.g2l[v] = (int32_t)P.l2g.size();
      P.l2g.push_back(v);
    }
  P.nv_own = (int32_t)P.l2g.size();
  std::vector<char> ghost(nv, 0);
  for (int32_t e : P.tet_l2g)
    for (int a = 0; a < 4; ++a) {
      const int32_t v = tets[4 * (size_t)e + a];
      if (owner[v] != rank) ghost[v] = 1;
    }
  for (int32_t v = 0; v < nv; ++v)
    if (ghost[v]) {
      P.g2l[v] = (int32_t)P.l2g.size();
      P.l2g.push_back(v);
    }
  P.nv_loc = (int32_t)P.l2g.size();
  P.tets_loc.resize(4 * (size_t)P.nt_loc);
  for (int32_t le = 0; le < P.nt_loc; ++le)
    for (int a = 0; a < 4; ++a) P.tets_loc[4 * (size_t)le + a] = P.g2l[tets[4 * (size_t)P.tet_l2g[le] + a]];
  // halo plan: a tet holding vertices of ranks r and q makes the r-owned ones ghosts on q
  std::vector<std::vector<int32_t>> send(world), recv(world);
  for (int32_t e = 0; e < nt; ++e) {
    const int32_t *t = tets + 4 * (size_t)e;
    int32_t ow[4];
    bool mine = false;
    for (int a = 0; a < 4; ++a) {
      ow[a] = owner[t[a]];
      mine = mine || ow[a] == rank;
    }
    if (!mine) continue;
    for (int a = 0; a < 4; ++a) {
      if (ow[a] == rank) {
        for (int b = 0; b < 4; ++b)
          if (ow[b] != rank) send[ow[b]].push_back(t[a]);
      } else {
        recv[ow[a]].push_back(t[a]);
      }
    }
  }
  for (int q = 0; q < world; ++q) {
    auto &S = send[q], &R = recv[q];
    std::sort(S.begin(), S.end());
    S.erase(std::unique(S.begin(), S.end()), S.end());
    std::sort(R.begin(), R.end());
    R.erase(std::unique(R.begin(), R.end()), R.end());
    if (S.empty() && R.empty()) continue;
    HaloPeer hp{q, (int32_t)S.size(), (int32_t)R.size(), (int64_t)P.send_idx.size(), (int64_t)P.recv_idx.size()};
    for (int32_t v : S) P.send_idx.push_back(P.g2l[v]);
    for (int32_t v : R) P.recv_idx.push_back(P.g2l[v]);
    P.peers.push_back(hp);
  }
  if (owner_out) *owner_out = owner;
}

// ------------------------------------------------------------------ NCCL
#define MS_NCCL(call)                                                                          \
  do {                                                                                         \
    ncclResult_t _r = (call);                                                                  \
    if (_r != ncclSuccess) throw ::msim::Error{MS_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(_r)}; \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  bool capturable() const override { return true; }
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  void allreduce_sum(double *dev, int64_t n, cudaStream_t s) override {
    MS_NCCL(ncclAllReduce(dev, dev, (size_t)n, ncclFloat64, ncclSum, comm, s));
  }
  void allreduce_min(double *dev, int64_t n, cudaStream_t s) override {
    MS_NCCL(ncclAllReduce(dev, dev, (size_t)n, ncclFloat64, ncclMin, comm, s));
  }
  void exchange(const std::vector<HaloPeer> &peers, const double *send, double *recv, cudaStream_t s) override {
    MS_NCCL(ncclGroupStart());
    for (const auto &p : peers) {
      if (p.n_send) MS_NCCL(ncclSend(send + 3 * p.send_off, 3 * (size_t)p.n_send, ncclFloat64, p.rank, comm, s));
      if (p.n_recv) MS_NCCL(ncclRecv(recv + 3 * p.recv_off, 3 * (size_t)p.n_recv, ncclFloat64, p.rank, comm, s));
    }
    MS_NCCL(ncclGroupEnd());
  }
};

Comm *make_nccl_comm(const uint8_t id[128], int rank, int world, int device) {
  MS_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
  std::copy(id, id + 128, reinterpret_cast<uint8_t *>(uid.internal));
  auto *c = new NcclComm();
  try {
    MS_NCCL(ncclCommInitRank(&c->comm, world, uid, rank));
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId uid;
  MS_NCCL(ncclGetUniqueId(&uid));
  std::copy(reinterpret_cast<const uint8_t *>(uid.internal), reinterpret_cast<const uint8_t *>(uid.internal) + 128, out);
}

// ------------------------------------------------------------------ in-process hub
struct Hub {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<std::vector<double>> slot;                 // per rank
  std::vector<const std::vector<HaloPeer> *> peers;      // per rank (exchange)
  explicit Hub(int w) : world(w), slot(w), peers(w, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

Hub *hub_create(int world) { return new Hub(world); }
void hub_destroy(Hub *h) { delete h; }

struct HubComm : Comm {
  Hub *hub;
  int rank;
  HubComm(Hub *h, int r) : hub(h), rank(r) {}
  template <typename Op>
  void reduce(double *dev, int64_t n, cudaStream_t s, Op op) {
    auto &mine = hub->slot[rank];
    mine.resize(n);
    MS_CUDA(cudaMemcpyAsync(mine.data(), dev, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    MS_CUDA(cudaStreamSynchronize(s));
    hub->barrier();
    std::vector<double> acc(hub->slot[0]);   // fixed rank order: identical result on every rank
    for (int q = 1; q < hub->world; ++q)
      for (int64_t k = 0; k < n; ++k) acc[k] = op(acc[k], hub->slot[q][k]);
    hub->barrier();
    MS_CUDA(cudaMemcpyAsync(dev, acc.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
    MS_CUDA(cudaStreamSynchronize(s));
  }
  void allreduce_sum(double *dev, int64_t n, cudaStream_t s) override {
    reduce(dev, n, s, [](double a, double b) { return a + b; });
  }
  void allreduce_min(double *dev, int64_t n, cudaStream_t s) override {
    reduce(dev, n, s, [](double a, double b) { return std::min(a, b); });
  }
  void exchange(const std::vector<HaloPeer> &peers, const double *send, double *recv, cudaStream_t s) override {
    int64_t ns = 0, nr = 0;
    for (const auto &p : peers) {
      ns += p.n_send;
      nr += p.n_recv;
    }
    auto &mine = hub->slot[rank];
    mine.resize(3 * ns);
    if (ns) MS_CUDA(cudaMemcpyAsync(mine.data(), send, sizeof(double) * 3 * ns, cudaMemcpyDeviceToHost, s));
    MS_CUDA(cudaStreamSynchronize(s));
    hub->peers[rank] = &peers;
    hub->barrier();
    std::vector<double> in(3 * nr);
    for (const auto &p : peers) {
      if (!p.n_recv) continue;
      const HaloPeer *src = nullptr;
      for (const auto &qp : *hub->peers[p.rank])
        if (qp.rank == rank) src = &qp;
      MS_REQUIRE(src && src->n_send == p.n_recv, MS_ERR_STATE, "inconsistent halo plans");
      std::copy(hub->slot[p.rank].begin() + 3 * src->send_off,
                hub->slot[p.rank].begin() + 3 * (src->send_off + src->n_send), in.begin() + 3 * p.recv_off);
    }
    hub->barrier();
    if (nr) MS_CUDA(cudaMemcpyAsync(recv, in.data(), sizeof(double) * 3 * nr, cudaMemcpyHostToDevice, s));
    MS_CUDA(cudaStreamSynchronize(s));
  }
};

Comm *make_hub_comm(Hub *hub, int rank) { return new HubComm(hub, rank); }

}  // namespace msim
