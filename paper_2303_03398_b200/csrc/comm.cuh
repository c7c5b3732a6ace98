// comm.cuh -- communication layer of libmaspcg: the phi-slab halo exchange
// and the scalar all-reduces of the PCG, behind one interface with two implementations:
//   * NcclComm      -- production: grouped ncclSend/ncclRecv and ncclAllReduce over NVLink /
//                      NVSwitch, one process per GPU (the CUDA-aware MPI halo exchange of
//                      PAPER.md:282, 290-292 re-done B200-first);
//   * LoopbackComm  -- test-only: several ranks in ONE process on ONE device (one host thread
//                      per rank), exchanging through device-to-device copies and fixed-order
//                      sums.  It lets the multi-rank decomposition (slabs, halos, split stencil,
//                      all-reduced scalars) be checked against the oracle on a single GPU.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "common.cuh"

namespace maspcg {

class Comm {
   public:
    virtual ~Comm() = default;
    int rank = 0, nranks = 1;
    int left() const { return (rank + nranks - 1) % nranks; }
    int right() const { return (rank + 1) % nranks; }
    // May the calls be captured into a CUDA graph?
    virtual bool capturable() const = 0;
    // Padded array buf[nloc+2][plane]: buf[0] <- left's plane nloc (its last local plane),
    // buf[nloc+1] <- right's plane 1 (its first local plane).
    virtual int halo_padded(double *buf, size_t plane, int nloc, cudaStream_t st, std::string &err) = 0;
    // lo_recv <- left's `last`, hi_recv <- right's `first` (each `count` doubles).
    virtual int halo_planes(const double *first, const double *last, double *lo_recv, double *hi_recv, size_t count,
                            cudaStream_t st, std::string &err) = 0;
    // recv[count] <- left's send[count] (ring shift towards higher ranks).
    virtual int shift_right(const double *send, double *recv, size_t count, cudaStream_t st, std::string &err) = 0;
    // recv[r * count + i] <- rank r's send[i] (all-gather).
    virtual int allgather(const double *send, double *recv, int count, cudaStream_t st, std::string &err) = 0;
    // In-place sum / max over ranks; every rank receives identical bits.
    virtual int allreduce_sum(double *dev, int count, cudaStream_t st, std::string &err) = 0;
    virtual int allreduce_max(int *dev, int count, cudaStream_t st, std::string &err) = 0;
    // Global value of `npairs` Dot2 (p, s) pairs in place, combined in rank order, in ONE device step
    // (peer communicator); false: the caller all-gathers and combines with its own kernel.
    // Peer communicator: the halo exchange of a padded buffer split in three, so a producing kernel can
    // store its boundary planes itself (fused): the neighbours' halo addresses and flags, a push of the
    // current planes (without waiting), and the wait (returns at once when *done is set).
    virtual bool fusable_halo() const { return false; }
    virtual int halo_targets(double *, size_t, int, double **, double **, unsigned long long **,
                             unsigned long long **, std::string &err) {
        err = "fused halo exchange not implemented by this communicator";
        return ST_E_INVALID;
    }
    virtual int halo_push(double *, size_t, int, cudaStream_t, std::string &err) {
        err = "fused halo exchange not implemented by this communicator";
        return ST_E_INVALID;
    }
    virtual int halo_wait(const int *, cudaStream_t, std::string &err) {
        err = "fused halo exchange not implemented by this communicator";
        return ST_E_INVALID;
    }
    virtual bool has_pair_allreduce() const { return false; }
    // peer communicator: every rank's staging area (for kernels that push their own LL words)
    virtual int ll_targets(double **, std::string &err) {
        err = "LL staging not available on this communicator";
        return ST_E_INVALID;
    }
    virtual int allreduce_pairs(double *, int, bool, cudaStream_t, std::string &err) {
        err = "pair all-reduce not implemented by this communicator";
        return ST_E_INVALID;
    }
};

// Returns nullptr and sets *status / err on failure.
Comm *make_nccl_comm(const void *unique_id, int rank, int nranks, int *status, std::string &err);

struct LoopbackGroup;
LoopbackGroup *loopback_group_create(int nranks);
void loopback_group_destroy(LoopbackGroup *g);
Comm *make_loopback_comm(LoopbackGroup *g, int rank, int nranks, int *status, std::string &err);

// ---- peer-memory communicator (peer.cu) ----
// Every rank's workspaces (region 0: the base workspace, 1: the vector-viscosity workspace) have the same
// layout; a local address inside a region maps to the same offset in the peer's region.
struct PeerTable {
    char *base[kP2PRegions][kP2PMaxRanks] = {};
    size_t bytes[kP2PRegions] = {};
    void *mapping[kP2PRegions][kP2PMaxRanks] = {};   // CUDA IPC mappings to close
    P2PArea *area = nullptr;                         // this rank's flags / epochs / staging (in region 0)
};
Comm *make_peer_comm(PeerTable *tab, int rank, int nranks, int *status, std::string &err);
// CUDA IPC: export a region (handle of its allocation + offset + size: kP2PHandleBytes), import a peer's.
int peer_export(const void *base, size_t bytes, void *out, std::string &err);
int peer_import(const void *in, char **base, size_t *bytes, void **mapping, std::string &err);
void peer_close(void *mapping);

}  // namespace maspcg
