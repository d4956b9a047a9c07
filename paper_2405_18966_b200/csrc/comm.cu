// comm.cu -- collectives of the row-partitioned multi-GPU solve (SURVEY.md
// 8(e); BASELINE.json north_star (e): all-gather of v, reduce of the partial
// A^T u, all-reduce of the Gram-Schmidt coefficient vectors).
//
// Two backends behind one interface (internal.h `Comm`):
//   * NCCL (one process per GPU, NVLink / NVSwitch), loaded with dlopen so the
//     library has no link-time NCCL dependency; every collective is enqueued on
//     the solve's stream.
//   * loopback: the ranks are threads of ONE process, each with its own handle
//     and stream (same or different devices).  Every collective synchronizes
//     the caller's stream, meets the other ranks at a host barrier and moves
//     the data with plain copies / a fixed-order summation kernel, so the
//     library's multi-rank host logic (partition, slicing, collective order,
//     status agreement) runs on a single GPU.  No kernel ever waits on another
//     rank's kernel.  Sums are over ranks 0..P-1 in order: every rank gets
//     bitwise identical results.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"

namespace svdsc {

// ---------------------------------------------------------------------------
// NCCL (runtime-loaded)
namespace {
typedef struct ncclComm *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclInt32 = 2, kNcclFloat64 = 8, kNcclSum = 0, kNcclMin = 3;

struct Nccl {
    bool tried = false, ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl g_nccl;
std::mutex g_nccl_mu;

bool nccl_load() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return false;
#define SYM(name, field) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(lib, name))
    SYM("ncclGetUniqueId", GetUniqueId);
    SYM("ncclCommInitRank", CommInitRank);
    SYM("ncclCommDestroy", CommDestroy);
    SYM("ncclCommAbort", CommAbort);
    SYM("ncclAllReduce", AllReduce);
    SYM("ncclReduceScatter", ReduceScatter);
    SYM("ncclReduce", Reduce);
    SYM("ncclAllGather", AllGather);
    SYM("ncclGetErrorString", GetErrorString);
#undef SYM
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.ReduceScatter && g_nccl.Reduce &&
                g_nccl.AllGather;
    return g_nccl.ok;
}

void ckn(ncclResult_t r, const char *what) {
    if (r != 0)
        throw CommError(SVDSC_ENCCL, std::string(what) + ": " +
                                         (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
}
void ckc(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw CommError(SVDSC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    int *dint = nullptr;
    // peer mailboxes (cgs2_peer): this rank's block (IPC-exported), the peers'
    // blocks opened through CUDA IPC (NVLink P2P mappings), the device PeerArgs
    bool peer_tried = false;
    void *mbox_block = nullptr;
    std::vector<void *> peer_blocks;
    PeerArgs *peer_dev = nullptr;
    ~NcclComm() override {
        peer_release();
        if (dint) cudaFree(dint);
        if (c && g_nccl.CommDestroy) g_nccl.CommDestroy(c);
    }
    void peer_release() {
        for (void *p : peer_blocks)
            if (p) cudaIpcCloseMemHandle(p);
        peer_blocks.clear();
        if (mbox_block) cudaFree(mbox_block);
        if (peer_dev) cudaFree(peer_dev);
        mbox_block = nullptr;
        peer_dev = nullptr;
        cudaGetLastError();
    }
    void peer_reset(cudaStream_t s) override {
        if (mbox_block) ckc(cudaMemsetAsync(mbox_block, 0, kPeerHdrBytes, s), "peer mailbox reset");
    }
    // first call: allocate and zero this rank's mailbox, all-gather
    // [ok, nsm, IPC handle] over NCCL, open every peer's block, agree (min) on
    // success; on any failure every rank returns NULL (the phased path runs)
    const PeerArgs *peer_setup(int nsm, cudaStream_t s) override {
        if (peer_tried) return peer_dev;
        peer_tried = true;
        const int P = nranks;
        if (P > kMaxPeers) return nullptr;
        const size_t bytes = peer_mailbox_bytes(P, kPeerPS);
        constexpr int kRec = 2 + (int)(sizeof(cudaIpcMemHandle_t) + 7) / 8;  // doubles per rank
        std::vector<double> mine(kRec, 0.0), all((size_t)kRec * P, 0.0);
        int ok = 1;
        cudaIpcMemHandle_t h{};
        if (cudaMalloc(&mbox_block, bytes) != cudaSuccess || cudaMemsetAsync(mbox_block, 0, bytes, s) != cudaSuccess ||
            (P > 1 && cudaIpcGetMemHandle(&h, mbox_block) != cudaSuccess))
            ok = 0;
        cudaGetLastError();
        mine[0] = ok;
        mine[1] = nsm;
        std::memcpy(mine.data() + 2, &h, sizeof(h));
        double *dbuf = nullptr;
        ckc(cudaMalloc(&dbuf, sizeof(double) * kRec * (P + 1)), "cudaMalloc");
        ckc(cudaMemcpyAsync(dbuf + (size_t)kRec * P, mine.data(), sizeof(double) * kRec, cudaMemcpyHostToDevice, s),
            "H2D");
        allgather(dbuf + (size_t)kRec * P, dbuf, kRec, s);
        ckc(cudaMemcpyAsync(all.data(), dbuf, sizeof(double) * kRec * P, cudaMemcpyDeviceToHost, s), "D2H");
        ckc(cudaStreamSynchronize(s), "sync");
        cudaFree(dbuf);
        PeerArgs pa{};
        pa.P = P;
        pa.rank = rank;
        pa.PS = kPeerPS;
        pa.expect = (unsigned)(P * nsm);
        for (int q = 0; q < P && ok; q++) {
            if (all[(size_t)q * kRec] != 1.0 || all[(size_t)q * kRec + 1] != (double)nsm) ok = 0;
        }
        peer_blocks.assign(P, nullptr);
        for (int q = 0; q < P && ok; q++) {
            char *base = nullptr;
            if (q == rank) {
                base = static_cast<char *>(mbox_block);
            } else {
                cudaIpcMemHandle_t hq;
                std::memcpy(&hq, all.data() + (size_t)q * kRec + 2, sizeof(hq));
                void *p = nullptr;
                if (cudaIpcOpenMemHandle(&p, hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    ok = 0;
                    break;
                }
                peer_blocks[q] = p;
                base = static_cast<char *>(p);
            }
            pa.ctr_peer[q] = reinterpret_cast<unsigned int *>(base);
            pa.mbox_peer[q] = reinterpret_cast<double *>(base + kPeerHdrBytes);
        }
        if (ok) {
            char *mb = static_cast<char *>(mbox_block);
            pa.ctr = reinterpret_cast<unsigned int *>(mb);
            pa.seq = reinterpret_cast<unsigned int *>(mb) + 2;
            pa.mbox = reinterpret_cast<double *>(mb + kPeerHdrBytes);
            if (cudaMalloc(&peer_dev, sizeof(PeerArgs)) != cudaSuccess ||
                cudaMemcpyAsync(peer_dev, &pa, sizeof(PeerArgs), cudaMemcpyHostToDevice, s) != cudaSuccess)
                ok = 0;
            cudaGetLastError();
        }
        if (allreduce_min_int(ok, s) != 1) {
            ckc(cudaStreamSynchronize(s), "sync");
            peer_release();
            return nullptr;
        }
        return peer_dev;
    }
    void allreduce_sum(double *buf, size_t n, cudaStream_t s) override {
        ckn(g_nccl.AllReduce(buf, buf, n, kNcclFloat64, kNcclSum, c, s), "ncclAllReduce");
    }
    void reduce_scatter_sum(const double *in, double *out, size_t n_each, cudaStream_t s) override {
        ckn(g_nccl.ReduceScatter(in, out, n_each, kNcclFloat64, kNcclSum, c, s), "ncclReduceScatter");
    }
    void reduce_sum(const double *in, double *out, size_t n, int root, cudaStream_t s) override {
        ckn(g_nccl.Reduce(in, out, n, kNcclFloat64, kNcclSum, root, c, s), "ncclReduce");
    }
    void allgather(const double *in, double *out, size_t n_each, cudaStream_t s) override {
        ckn(g_nccl.AllGather(in, out, n_each, kNcclFloat64, c, s), "ncclAllGather");
    }
    int allreduce_min_int(int v, cudaStream_t s) override {
        if (!dint) ckc(cudaMalloc(&dint, sizeof(int)), "cudaMalloc");
        ckc(cudaMemcpyAsync(dint, &v, sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
        ckn(g_nccl.AllReduce(dint, dint, 1, kNcclInt32, kNcclMin, c, s), "ncclAllReduce(min)");
        int r = 0;
        ckc(cudaMemcpyAsync(&r, dint, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
        ckc(cudaStreamSynchronize(s), "sync");
        return r;
    }
};

// ---------------------------------------------------------------------------
// loopback
constexpr int kMaxLoopRanks = 16;
struct RankPtrs {
    const double *p[kMaxLoopRanks];
};

// out[i] = sum_{q < P} p[q][off + i], q ascending (fixed order)
__global__ void k_sum_ranks(RankPtrs rp, int P, size_t off, size_t n, double *out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < P; q++) s += rp.p[q][off + i];
        out[i] = s;
    }
}
}  // namespace

struct LoopbackGroup {
    int P = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool failed = false;
    int refs = 1;  // the creator's reference + one per attached rank
    std::vector<const double *> ptr;
    std::vector<int> ival;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (failed) throw CommError(SVDSC_ECUDA, "loopback group: another rank failed");
        const uint64_t g = gen;
        if (++arrived == P) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g || failed; });
            if (failed && gen == g) throw CommError(SVDSC_ECUDA, "loopback group: another rank failed");
        }
    }
    void fail() {
        std::lock_guard<std::mutex> lk(mu);
        failed = true;
        cv.notify_all();
    }
};

namespace {
struct LoopbackComm : Comm {
    LoopbackGroup *g;
    double *tmp = nullptr;
    size_t tmp_n = 0;
    explicit LoopbackComm(LoopbackGroup *grp) : g(grp) {}
    ~LoopbackComm() override {
        if (tmp) cudaFree(tmp);
        loopback_group_release(g);
    }
    RankPtrs ptrs() const {
        RankPtrs r{};
        for (int q = 0; q < nranks; q++) r.p[q] = g->ptr[q];
        return r;
    }
    void sum_into(size_t off, size_t n, double *out, cudaStream_t s) {
        if (n == 0) return;
        const int blocks = (int)std::min<size_t>(1184, (n + 255) / 256);
        k_sum_ranks<<<blocks, 256, 0, s>>>(ptrs(), nranks, off, n, out);
        count_launch();
        ckc(cudaGetLastError(), "k_sum_ranks");
    }
    void publish(const double *p, cudaStream_t s) {
        ckc(cudaStreamSynchronize(s), "sync");  // p's producer is complete
        g->ptr[rank] = p;
        g->barrier();
    }
    void allreduce_sum(double *buf, size_t n, cudaStream_t s) override {
        if (n > tmp_n) {
            if (tmp) cudaFree(tmp);
            tmp = nullptr;
            ckc(cudaMalloc(&tmp, n * sizeof(double)), "cudaMalloc");
            tmp_n = n;
        }
        publish(buf, s);
        sum_into(0, n, tmp, s);
        ckc(cudaStreamSynchronize(s), "sync");
        g->barrier();  // every rank has read every buffer
        ckc(cudaMemcpyAsync(buf, tmp, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "D2D");
    }
    void reduce_sum(const double *in, double *out, size_t n, int root, cudaStream_t s) override {
        publish(in, s);
        if (rank == root) sum_into(0, n, out, s);
        ckc(cudaStreamSynchronize(s), "sync");
        g->barrier();
    }
    void reduce_scatter_sum(const double *in, double *out, size_t n_each, cudaStream_t s) override {
        publish(in, s);
        sum_into((size_t)rank * n_each, n_each, out, s);
        ckc(cudaStreamSynchronize(s), "sync");
        g->barrier();
    }
    void allgather(const double *in, double *out, size_t n_each, cudaStream_t s) override {
        publish(in, s);
        for (int q = 0; q < nranks; q++)
            ckc(cudaMemcpyAsync(out + (size_t)q * n_each, g->ptr[q], n_each * sizeof(double), cudaMemcpyDefault, s),
                "allgather copy");
        ckc(cudaStreamSynchronize(s), "sync");
        g->barrier();
    }
    int allreduce_min_int(int v, cudaStream_t) override {
        g->ival[rank] = v;
        g->barrier();
        int m = v;
        for (int q = 0; q < nranks; q++) m = std::min(m, g->ival[q]);
        g->barrier();
        return m;
    }
    void abort() override { g->fail(); }
};
}  // namespace

bool comm_nccl_available() { return nccl_load(); }

void comm_nccl_unique_id(unsigned char id[128]) {
    if (!nccl_load()) throw CommError(SVDSC_ENCCL, "libnccl.so.2 not loadable");
    ncclUniqueId u;
    ckn(g_nccl.GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
}

Comm *comm_nccl_create(const unsigned char id[128], int nranks, int rank) {
    if (!nccl_load()) throw CommError(SVDSC_ENCCL, "libnccl.so.2 not loadable");
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    NcclComm *c = new NcclComm();
    c->nranks = nranks;
    c->rank = rank;
    const ncclResult_t r = g_nccl.CommInitRank(&c->c, nranks, u, rank);
    if (r != 0) {
        c->c = nullptr;
        delete c;
        ckn(r, "ncclCommInitRank");
    }
    return c;
}

LoopbackGroup *loopback_group_create(int nranks) {
    if (nranks < 1 || nranks > kMaxLoopRanks) return nullptr;
    LoopbackGroup *g = new LoopbackGroup();
    g->P = nranks;
    g->ptr.assign(nranks, nullptr);
    g->ival.assign(nranks, 0);
    return g;
}

void loopback_group_release(LoopbackGroup *g) {
    if (!g) return;
    bool del = false;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        del = --g->refs == 0;
    }
    if (del) delete g;
}

Comm *comm_loopback_create(LoopbackGroup *g, int rank) {
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->refs++;
    }
    LoopbackComm *c = new LoopbackComm(g);
    c->nranks = g->P;
    c->rank = rank;
    return c;
}

}  // namespace svdsc
