// comm.cu -- the context's communicator for the particle-sharded pipeline
// (SURVEY 8(b) pifcm_dist, 8(e)): NCCL over NVLink / NVSwitch, loaded with
// dlopen (libnccl.so.2: the one torch already mapped, else the system's), or
// caller-supplied host collectives (gloo, MPI, ... -- tests share one GPU
// between ranks, which NCCL refuses).  The only exchanges of the method are
// the all-gather of the per-generation fitness vector (Alg. 1 step 4 -> 5,
// PAPER:98-99) and the broadcast of the gbest state before the final IFCM
// (Alg. 1 steps 10-11).
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <vector>

#include "pifcm_comm.h"

namespace pifcm {

namespace {
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errStr)(ncclResult_t) = nullptr;
    bool ok() const { return getUniqueId && commInitRank && commDestroy && allGather && broadcast && errStr; }
};

NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) api.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (api.h) {
            api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
            api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.h, "ncclCommInitRank"));
            api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.h, "ncclCommDestroy"));
            api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(api.h, "ncclAllGather"));
            api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(api.h, "ncclBroadcast"));
            api.errStr = reinterpret_cast<decltype(api.errStr)>(dlsym(api.h, "ncclGetErrorString"));
        }
    }
    return api;
}

// [world][maxl] padded all-gather buffer -> fit[0, P) in particle order
__global__ void k_unpack_fit(const double *recv, int maxl, int P, int world, double *fit) {
    const int base = P / world, rem = P % world;
    for (int r = 0; r < world; ++r) {
        const int p0 = r * base + (r < rem ? r : rem), n = base + (r < rem ? 1 : 0);
        for (int i = threadIdx.x; i < n; i += blockDim.x) fit[p0 + i] = recv[(long long)r * maxl + i];
    }
}
}  // namespace

void dist_range(int P, int world, int rank, int *p0, int *p1) {
    const int base = P / world, rem = P % world;
    *p0 = rank * base + (rank < rem ? rank : rem);
    *p1 = *p0 + base + (rank < rem ? 1 : 0);
}

int comm_unique_id(uint8_t *id, std::string &err) {
    NcclApi &a = nccl();
    if (!a.ok()) { err = "libnccl.so.2 not loadable"; return PIFCM_ENCCL; }
    ncclUniqueId u;
    const ncclResult_t r = a.getUniqueId(&u);
    if (r != ncclSuccess) { err = a.errStr(r); return PIFCM_ENCCL; }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id, &u, 128);
    return PIFCM_OK;
}

int comm_init(Comm &c, int device, const pifcm_dist *d, const pifcm_host_coll *hc, std::string &err) {
    comm_free(c);
    if (!d || d->world <= 1) return PIFCM_OK;
    if (d->rank < 0 || d->rank >= d->world) { err = "rank outside [0, world)"; return PIFCM_EINVAL; }
    if (d->shard != 0) { err = "pifcm_dist.shard: only 0 (particles) is supported by the C pipeline"; return PIFCM_EINVAL; }
    c.rank = d->rank;
    c.world = d->world;
    if (hc) {
        if (!hc->allgather || !hc->broadcast) { err = "host collectives need allgather and broadcast"; return PIFCM_EINVAL; }
        c.host = *hc;
        c.kind = Comm::HOST;
    } else {
        if (!d->nccl_unique_id) { err = "world > 1 needs an NCCL unique id or host collectives"; return PIFCM_EINVAL; }
        NcclApi &a = nccl();
        if (!a.ok()) { err = "libnccl.so.2 not loadable"; return PIFCM_ENCCL; }
        ncclUniqueId u;
        memcpy(&u, d->nccl_unique_id, 128);
        if (cudaSetDevice(device) != cudaSuccess) { err = "cudaSetDevice"; return PIFCM_ECUDA; }
        ncclComm_t comm = nullptr;
        const ncclResult_t r = a.commInitRank(&comm, d->world, u, d->rank);
        if (r != ncclSuccess) { err = std::string("ncclCommInitRank: ") + a.errStr(r); return PIFCM_ENCCL; }
        c.nccl = comm;
        c.kind = Comm::NCCL;
    }
    return PIFCM_OK;
}

void comm_free(Comm &c) {
    if (c.kind == Comm::NCCL && c.nccl) nccl().commDestroy(static_cast<ncclComm_t>(c.nccl));
    if (c.buf) cudaFree(c.buf);
    c = Comm{};
}

static int ensure_buf(Comm &c, size_t bytes, std::string &err) {
    if (c.buf_bytes >= bytes) return PIFCM_OK;
    if (c.buf) cudaFree(c.buf);
    c.buf = nullptr;
    c.buf_bytes = 0;
    if (cudaMalloc(&c.buf, bytes) != cudaSuccess) { err = "comm scratch cudaMalloc"; return PIFCM_ENOMEM; }
    c.buf_bytes = bytes;
    return PIFCM_OK;
}

// fit[P] (device fp64): on entry this rank's range holds its particles'
// fitness; on exit every entry holds its owner's value (rank order).
int comm_allgather_fitness(Comm &c, double *fit, int P, cudaStream_t st, std::string &err) {
    if (c.world <= 1) return PIFCM_OK;
    int p0, p1;
    dist_range(P, c.world, c.rank, &p0, &p1);
    const int maxl = (P + c.world - 1) / c.world;
    const size_t seg = sizeof(double) * (size_t)maxl;
    int r;
    if ((r = ensure_buf(c, seg * (c.world + 1), err))) return r;
    double *send = static_cast<double *>(c.buf), *recv = send + maxl;
    if (cudaMemsetAsync(send, 0, seg, st) != cudaSuccess ||
        cudaMemcpyAsync(send, fit + p0, sizeof(double) * (p1 - p0), cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
        err = "fitness staging";
        return PIFCM_ECUDA;
    }
    if (c.kind == Comm::NCCL) {
        NcclApi &a = nccl();
        const ncclResult_t e = a.allGather(send, recv, (size_t)maxl, ncclFloat64, static_cast<ncclComm_t>(c.nccl), st);
        if (e != ncclSuccess) { err = std::string("ncclAllGather: ") + a.errStr(e); return PIFCM_ENCCL; }
    } else {
        std::vector<double> hs(maxl), hr((size_t)maxl * c.world);
        if (cudaMemcpyAsync(hs.data(), send, seg, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) { err = "fitness D2H"; return PIFCM_ECUDA; }
        if (c.host.allgather(c.host.user, hs.data(), hr.data(), seg) != 0) { err = "host allgather failed"; return PIFCM_ENCCL; }
        if (cudaMemcpyAsync(recv, hr.data(), seg * c.world, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) { err = "fitness H2D"; return PIFCM_ECUDA; }
    }
    k_unpack_fit<<<1, 128, 0, st>>>(recv, maxl, P, c.world, fit);
    if (cudaGetLastError() != cudaSuccess) { err = "k_unpack_fit"; return PIFCM_ECUDA; }
    return PIFCM_OK;
}

// bytes of device memory `buf` from rank `root` to every rank
int comm_broadcast(Comm &c, void *buf, size_t bytes, int root, cudaStream_t st, std::string &err) {
    if (c.world <= 1) return PIFCM_OK;
    if (c.kind == Comm::NCCL) {
        NcclApi &a = nccl();
        const ncclResult_t e = a.broadcast(buf, buf, bytes, ncclUint8, root, static_cast<ncclComm_t>(c.nccl), st);
        if (e != ncclSuccess) { err = std::string("ncclBroadcast: ") + a.errStr(e); return PIFCM_ENCCL; }
        return PIFCM_OK;
    }
    std::vector<unsigned char> h(bytes);
    if (c.rank == root &&
        (cudaMemcpyAsync(h.data(), buf, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
         cudaStreamSynchronize(st) != cudaSuccess)) { err = "broadcast D2H"; return PIFCM_ECUDA; }
    if (c.host.broadcast(c.host.user, h.data(), bytes, root) != 0) { err = "host broadcast failed"; return PIFCM_ENCCL; }
    if (c.rank != root &&
        (cudaMemcpyAsync(buf, h.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
         cudaStreamSynchronize(st) != cudaSuccess)) { err = "broadcast H2D"; return PIFCM_ECUDA; }
    return PIFCM_OK;
}

}  // namespace pifcm
