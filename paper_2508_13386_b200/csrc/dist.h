// Multi-GPU slab partition of the mesh: one rank per GPU, SPMD.
//
// Every rank receives the full mesh and basis (ms_upload_mesh / ms_basis_upload) and keeps
//   * owned vertices: a contiguous slab along x (vertices sorted by (x, id), split into equal
//     counts), numbered first in the local numbering;
//   * local tets: every tet with an owned vertex (so the rows of owned vertices -- gradient,
//     Hessian, Galerkin contributions -- are complete); owned tets (vertex 0 owned) first, they
//     alone count in energies;
//   * ghost vertices: the other vertices of the local tets, numbered after the owned ones.
// Ghost values are refreshed from their owners by a halo exchange of the vectors whose ghost
// entries are read (the PCG search vector z once per iteration, the Newton direction d before
// the line search); reductions (energies, dots, B^T r, S = B^T H B) cover owned entries and
// are summed across ranks; the coarse factorisation is replicated.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace msim {

struct HaloPeer {
  int rank;
  int32_t n_send, n_recv;          // vertices
  int64_t send_off, recv_off;      // into the concatenated index lists
};

struct Partition {
  int rank = 0, world = 1;
  int32_t nv_glob = 0, nt_glob = 0;
  int32_t nv_own = 0, nv_loc = 0, nt_own = 0, nt_loc = 0;
  std::vector<int32_t> l2g;        // local vertex -> global id
  std::vector<int32_t> g2l;        // global id -> local vertex (-1: not local)
  std::vector<int32_t> tet_l2g;    // local tet -> global tet
  std::vector<int32_t> tets_loc;   // local connectivity (n_loc x 4)
  std::vector<HaloPeer> peers;
  std::vector<int32_t> send_idx, recv_idx;   // local vertex ids, concatenated by peer
};

// Host-only: the partition of rank `rank` of `world` (deterministic; identical plans on all
// ranks).  owner[v] = slab of vertex v.
void make_partition(int rank, int world, int32_t nv, const double *X, int32_t nt, const int32_t *tets,
                    Partition &P, std::vector<int32_t> *owner_out = nullptr);

// Collective backend.  All operations are enqueued on / synchronised with `stream`.
struct Comm {
  virtual ~Comm() = default;
  // true if the operations can be recorded into a CUDA graph (NCCL; not the host-side hub)
  virtual bool capturable() const { return false; }
  virtual void allreduce_sum(double *dev, int64_t n, cudaStream_t stream) = 0;
  virtual void allreduce_min(double *dev, int64_t n, cudaStream_t stream) = 0;
  // send[peer] -> recv[peer] for every peer (3 doubles per vertex), buffers on the device
  virtual void exchange(const std::vector<HaloPeer> &peers, const double *send, double *recv,
                        cudaStream_t stream) = 0;
};

Comm *make_nccl_comm(const uint8_t id[128], int rank, int world, int device);   // throws on error
void nccl_unique_id(uint8_t out[128]);

// In-process hub (tests on one GPU): W contexts driven by W host threads exchange through host
// memory; every collective synchronises the calling stream first (no device-side waiting).
struct Hub;
Hub *hub_create(int world);
void hub_destroy(Hub *);
Comm *make_hub_comm(Hub *hub, int rank);

}  // namespace msim
