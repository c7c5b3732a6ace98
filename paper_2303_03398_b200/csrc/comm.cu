// comm.cu -- NCCL and in-process loopback implementations of the communication layer.
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "comm.cuh"

namespace maspcg {

// ============================================================== NCCL
class NcclComm final : public Comm {
   public:
    ncclComm_t comm = nullptr;        // collectives (all-gather of Dot2 pairs, validation all-reduce)
    ncclComm_t halo = nullptr;        // point-to-point halo planes: its own communicator (ncclCommSplit), so a
                                      // halo on the communication stream may overlap a collective on the
                                      // compute stream without two streams sharing one communicator
    ~NcclComm() override {
        if (halo) ncclCommDestroy(halo);
        if (comm) ncclCommDestroy(comm);
    }
    bool capturable() const override { return true; }

    static int fail(ncclResult_t r, const char *what, std::string &err) {
        err = std::string(what) + ": " + ncclGetErrorString(r);
        return ST_E_NCCL;
    }

    // Ops to the same peer are matched in issue order, so this order is also right when
    // left == right (P = 2): the first send / receive between a pair carries "first plane -> hi halo".
    int halo_planes(const double *first, const double *last, double *lo_recv, double *hi_recv, size_t count,
                    cudaStream_t st, std::string &err) override {
        ncclResult_t r;
        if ((r = ncclGroupStart()) != ncclSuccess) return fail(r, "ncclGroupStart", err);
        r = ncclSend(first, count, ncclDouble, left(), halo, st);                          // my first plane
        if (r == ncclSuccess) r = ncclRecv(hi_recv, count, ncclDouble, right(), halo, st);  // right's first
        if (r == ncclSuccess) r = ncclSend(last, count, ncclDouble, right(), halo, st);     // my last plane
        if (r == ncclSuccess) r = ncclRecv(lo_recv, count, ncclDouble, left(), halo, st);   // left's last
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess) return fail(r, "halo send/recv", err);
        if (r2 != ncclSuccess) return fail(r2, "ncclGroupEnd", err);
        return ST_OK;
    }

    int halo_padded(double *buf, size_t pl, int nloc, cudaStream_t st, std::string &err) override {
        return halo_planes(buf + pl, buf + (size_t)nloc * pl, buf, buf + (size_t)(nloc + 1) * pl, pl, st, err);
    }

    int shift_right(const double *send, double *recv, size_t count, cudaStream_t st, std::string &err) override {
        ncclResult_t r;
        if ((r = ncclGroupStart()) != ncclSuccess) return fail(r, "ncclGroupStart", err);
        r = ncclSend(send, count, ncclDouble, right(), halo, st);
        if (r == ncclSuccess) r = ncclRecv(recv, count, ncclDouble, left(), halo, st);
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess) return fail(r, "shift send/recv", err);
        if (r2 != ncclSuccess) return fail(r2, "ncclGroupEnd", err);
        return ST_OK;
    }

    int allgather(const double *send, double *recv, int count, cudaStream_t st, std::string &err) override {
        ncclResult_t r = ncclAllGather(send, recv, count, ncclDouble, comm, st);
        return r == ncclSuccess ? ST_OK : fail(r, "ncclAllGather", err);
    }

    int allreduce_sum(double *dev, int count, cudaStream_t st, std::string &err) override {
        ncclResult_t r = ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, comm, st);
        return r == ncclSuccess ? ST_OK : fail(r, "ncclAllReduce(sum)", err);
    }

    int allreduce_max(int *dev, int count, cudaStream_t st, std::string &err) override {
        ncclResult_t r = ncclAllReduce(dev, dev, count, ncclInt32, ncclMax, comm, st);
        return r == ncclSuccess ? ST_OK : fail(r, "ncclAllReduce(max)", err);
    }
};

Comm *make_nccl_comm(const void *unique_id, int rank, int nranks, int *status, std::string &err) {
    auto *c = new NcclComm();
    c->rank = rank;
    c->nranks = nranks;
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
        c->comm = nullptr;
        delete c;
        *status = ST_E_NCCL;
        return nullptr;
    }
    r = ncclCommSplit(c->comm, 0, rank, &c->halo, nullptr);   // collective, same rank order
    if (r != ncclSuccess) {
        err = std::string("ncclCommSplit: ") + ncclGetErrorString(r);
        c->halo = nullptr;
        delete c;
        *status = ST_E_NCCL;
        return nullptr;
    }
    *status = ST_OK;
    return c;
}

// ============================================================== loopback (test-only)
constexpr int kLoopMaxRanks = 16;
constexpr int kLoopSlot = 16384;   // doubles per rank: the scalar dots and the vector operator's pole rings (4 nr)

struct LoopSlots {
    const double *d[kLoopMaxRanks];
    const int *i[kLoopMaxRanks];
};

__global__ void k_gather_sum(LoopSlots s, int nranks, int count, double *out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int r = 0; r < nranks; ++r) v += s.d[r][t];   // fixed rank order: identical bits everywhere
        out[t] = v;
    }
}

__global__ void k_gather_max(LoopSlots s, int nranks, int count, int *out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
        int v = s.i[0][t];
        for (int r = 1; r < nranks; ++r) v = max(v, s.i[r][t]);
        out[t] = v;
    }
}

struct LoopbackGroup {
    int n = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    struct Slot {
        const double *buf = nullptr;   // padded array / send buffer published for this exchange
        const double *buf2 = nullptr;  // second send buffer (halo_planes: last plane)
        double *dslot = nullptr;       // device scratch for sums
        int *islot = nullptr;
        cudaEvent_t e = nullptr, f = nullptr;
    };
    std::vector<Slot> slots;

    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long g = generation;
        if (++arrived == n) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != g; });
        }
    }
};

LoopbackGroup *loopback_group_create(int nranks) {
    if (nranks < 1 || nranks > kLoopMaxRanks) return nullptr;
    auto *g = new LoopbackGroup();
    g->n = nranks;
    g->slots.resize(nranks);
    return g;
}

void loopback_group_destroy(LoopbackGroup *g) { delete g; }


class LoopbackComm final : public Comm {
   public:
    LoopbackGroup *g = nullptr;
    ~LoopbackComm() override {
        // collective, like every loopback call: a peer may still be issuing cudaStreamWaitEvent on
        // this rank's events from the last exchange, so nobody destroys them before all arrive
        g->barrier();
        auto &s = g->slots[rank];
        if (s.dslot) cudaFree(s.dslot);
        if (s.islot) cudaFree(s.islot);
        if (s.e) cudaEventDestroy(s.e);
        if (s.f) cudaEventDestroy(s.f);
        s = LoopbackGroup::Slot{};
    }
    bool capturable() const override { return false; }

    static int ck(cudaError_t e, const char *what, std::string &err) {
        if (e == cudaSuccess) return ST_OK;
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return ST_E_CUDA;
    }
    LoopbackGroup::Slot &me() { return g->slots[rank]; }

    // publish (record e), rendezvous, wait for the peers' e
    int phase1(cudaStream_t st, const int *peers, int npeers, std::string &err) {
        if (int s = ck(cudaEventRecord(me().e, st), "record", err)) return s;
        g->barrier();
        for (int k = 0; k < npeers; ++k)
            if (int s = ck(cudaStreamWaitEvent(st, g->slots[peers[k]].e, 0), "wait", err)) return s;
        return ST_OK;
    }
    // record f after reading the peers' data, rendezvous, wait until the readers of MY data are done
    int phase2(cudaStream_t st, const int *peers, int npeers, std::string &err) {
        if (int s = ck(cudaEventRecord(me().f, st), "record", err)) return s;
        g->barrier();
        for (int k = 0; k < npeers; ++k)
            if (int s = ck(cudaStreamWaitEvent(st, g->slots[peers[k]].f, 0), "wait", err)) return s;
        return ST_OK;
    }

    int halo_padded(double *buf, size_t pl, int nloc, cudaStream_t st, std::string &err) override {
        me().buf = buf;
        const int peers[2] = {left(), right()};
        if (int s = phase1(st, peers, 2, err)) return s;
        const double *L = g->slots[left()].buf, *R = g->slots[right()].buf;
        if (int s = ck(cudaMemcpyAsync(buf, L + (size_t)nloc * pl, 8 * pl, cudaMemcpyDeviceToDevice, st), "copy", err))
            return s;
        if (int s = ck(cudaMemcpyAsync(buf + (size_t)(nloc + 1) * pl, R + pl, 8 * pl, cudaMemcpyDeviceToDevice, st),
                       "copy", err))
            return s;
        return phase2(st, peers, 2, err);
    }

    int halo_planes(const double *first, const double *last, double *lo_recv, double *hi_recv, size_t count,
                    cudaStream_t st, std::string &err) override {
        me().buf = first;
        me().buf2 = last;
        const int peers[2] = {left(), right()};
        if (int s = phase1(st, peers, 2, err)) return s;
        if (int s = ck(cudaMemcpyAsync(lo_recv, g->slots[left()].buf2, 8 * count, cudaMemcpyDeviceToDevice, st),
                       "copy", err))
            return s;
        if (int s = ck(cudaMemcpyAsync(hi_recv, g->slots[right()].buf, 8 * count, cudaMemcpyDeviceToDevice, st),
                       "copy", err))
            return s;
        return phase2(st, peers, 2, err);
    }

    int shift_right(const double *send, double *recv, size_t count, cudaStream_t st, std::string &err) override {
        me().buf = send;
        const int from[1] = {left()}, readers[1] = {right()};
        if (int s = phase1(st, from, 1, err)) return s;
        if (int s = ck(cudaMemcpyAsync(recv, g->slots[left()].buf, 8 * count, cudaMemcpyDeviceToDevice, st), "copy",
                       err))
            return s;
        return phase2(st, readers, 1, err);
    }

    int all_peers(int *p) const {
        for (int r = 0; r < nranks; ++r) p[r] = r;
        return nranks;
    }

    int allgather(const double *send, double *recv, int count, cudaStream_t st, std::string &err) override {
        if (count > kLoopSlot) {
            err = "loopback all-gather count too large";
            return ST_E_INVALID;
        }
        if (int s = ck(cudaMemcpyAsync(me().dslot, send, 8 * count, cudaMemcpyDeviceToDevice, st), "copy", err))
            return s;
        int peers[kLoopMaxRanks];
        const int np = all_peers(peers);
        if (int s = phase1(st, peers, np, err)) return s;
        for (int r = 0; r < nranks; ++r)
            if (int s = ck(cudaMemcpyAsync(recv + (size_t)r * count, g->slots[r].dslot, 8 * count,
                                           cudaMemcpyDeviceToDevice, st),
                           "copy", err))
                return s;
        return phase2(st, peers, np, err);
    }

    int allreduce_sum(double *dev, int count, cudaStream_t st, std::string &err) override {
        if (count > kLoopSlot) {
            err = "loopback all-reduce count too large";
            return ST_E_INVALID;
        }
        if (int s = ck(cudaMemcpyAsync(me().dslot, dev, 8 * count, cudaMemcpyDeviceToDevice, st), "copy", err))
            return s;
        int peers[kLoopMaxRanks];
        const int np = all_peers(peers);
        if (int s = phase1(st, peers, np, err)) return s;
        LoopSlots ls{};
        for (int r = 0; r < nranks; ++r) ls.d[r] = g->slots[r].dslot;
        k_gather_sum<<<(count + 255) / 256, 256, 0, st>>>(ls, nranks, count, dev);
        if (int s = ck(cudaGetLastError(), "k_gather_sum", err)) return s;
        return phase2(st, peers, np, err);
    }

    int allreduce_max(int *dev, int count, cudaStream_t st, std::string &err) override {
        if (count > kLoopSlot) {
            err = "loopback all-reduce count too large";
            return ST_E_INVALID;
        }
        if (int s = ck(cudaMemcpyAsync(me().islot, dev, 4 * count, cudaMemcpyDeviceToDevice, st), "copy", err))
            return s;
        int peers[kLoopMaxRanks];
        const int np = all_peers(peers);
        if (int s = phase1(st, peers, np, err)) return s;
        LoopSlots ls{};
        for (int r = 0; r < nranks; ++r) ls.i[r] = g->slots[r].islot;
        k_gather_max<<<(count + 255) / 256, 256, 0, st>>>(ls, nranks, count, dev);
        if (int s = ck(cudaGetLastError(), "k_gather_max", err)) return s;
        return phase2(st, peers, np, err);
    }
};

Comm *make_loopback_comm(LoopbackGroup *g, int rank, int nranks, int *status, std::string &err) {
    if (!g || rank < 0 || rank >= g->n || nranks != g->n) {
        err = "bad loopback group or rank";
        *status = ST_E_INVALID;
        return nullptr;
    }
    auto *c = new LoopbackComm();
    c->g = g;
    c->rank = rank;
    c->nranks = g->n;
    auto &s = g->slots[rank];
    cudaError_t e = cudaMalloc((void **)&s.dslot, 8 * kLoopSlot);
    if (e == cudaSuccess) e = cudaMalloc((void **)&s.islot, 4 * kLoopSlot);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.e, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.f, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        err = std::string("loopback init: ") + cudaGetErrorString(e);
        delete c;
        *status = ST_E_CUDA;
        return nullptr;
    }
    *status = ST_OK;
    return c;
}

}  // namespace maspcg
