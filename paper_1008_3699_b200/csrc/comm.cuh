// comm.cuh -- communicators of a slab decomposition (include/sweep.h sw_comm).
//
// The only data a decomposed sweep needs from another rank are the neighbours' previous-sweep
// values in the 2 layers beyond the slab ("halo points ... renewed (via communication) prior to a
// new iteration"); a PCG iteration adds 1-layer exchanges and the reductions.
// Along the slab axis (the slowest: y in 2D, z in 3D, x in 1D) w layers of a padded array are
// one contiguous block of w * L doubles (L = the padded layer size), so an exchange is one
// send/receive pair per neighbour straight from / into the library's arrays:
//   send layers [2, 2 + w) to rank - 1, receive its layers into the ghost layers [2 - w, 2);
//   send layers [2 + n - w, 2 + n) to rank + 1, receive into [2 + n, 2 + n + w).
// Transports: NCCL point-to-point / all-gather on the caller's stream (one process per GPU over
// NVLink), or a HOST transport of the caller's (callbacks on pinned staging buffers) for several
// processes or threads that share one GPU in tests.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

namespace sw {

// NCCL entry points, resolved at run time: the libnccl.so.2 already in the process (torch's) if
// there is one, else the system library.  No link-time dependency for single-GPU use.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

inline NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
#define SW_NCCL_SYM(f)                                                              \
    *(void **)(&api.f) = dlsym(h, "nccl" #f);                                       \
    if (!api.f) {                                                                   \
        api.why = "libnccl.so.2 lacks nccl" #f;                                     \
        return;                                                                     \
    }
        SW_NCCL_SYM(GetUniqueId)
        SW_NCCL_SYM(CommInitRank)
        SW_NCCL_SYM(CommDestroy)
        SW_NCCL_SYM(GroupStart)
        SW_NCCL_SYM(GroupEnd)
        SW_NCCL_SYM(Send)
        SW_NCCL_SYM(Recv)
        SW_NCCL_SYM(AllGather)
        SW_NCCL_SYM(GetErrorString)
#undef SW_NCCL_SYM
        api.ok = true;
    });
    return api;
}

}  // namespace sw

struct sw_comm {
    enum Kind { NCCL = 1, HOST = 2 } kind = HOST;
    int rank = 0, nranks = 1, dev = 0;
    ncclComm_t nc = nullptr;
    sw_exchange_fn xfn = nullptr;
    sw_allgather_fn gfn = nullptr;
    void *ctx = nullptr;
    unsigned char *stage = nullptr;   // pinned staging of the HOST transport
    size_t stage_bytes = 0;
};

namespace sw {

// status + message of a transport step (the caller turns it into sw_status / sw_last_error)
struct CommErr {
    int code = 0;   // 0 ok, 1 NCCL / host callback, 2 CUDA
    std::string msg;
};

inline CommErr comm_cuda(cudaError_t e, const char *what) {
    CommErr r;
    if (e != cudaSuccess) {
        r.code = 2;
        r.msg = std::string(what) + ": " + cudaGetErrorString(e);
    }
    return r;
}

inline CommErr comm_nccl(ncclResult_t e, const char *what) {
    CommErr r;
    if (e != ncclSuccess) {
        r.code = 1;
        r.msg = std::string(what) + ": " + nccl().GetErrorString(e);
    }
    return r;
}

inline CommErr stage_reserve(sw_comm *c, size_t bytes) {
    if (c->stage_bytes >= bytes) return {};
    if (c->stage) cudaFreeHost(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    CommErr e = comm_cuda(cudaMallocHost((void **)&c->stage, bytes), "cudaMallocHost (staging)");
    if (!e.code) c->stage_bytes = bytes;
    return e;
}

// Refresh the w ghost layers on both slab sides of the padded array `base` (L doubles per layer,
// n interior layers along the slab axis) from ranks -1 / +1, ordered on stream s.
inline CommErr comm_exchange(sw_comm *c, double *base, size_t L, int64_t n, int w, cudaStream_t s) {
    const bool lo = c->rank > 0, hi = c->rank < c->nranks - 1;
    const size_t cnt = (size_t)w * L, bytes = cnt * sizeof(double);
    double *send_lo = base + 2 * L, *recv_lo = base + (2 - w) * L;
    double *send_hi = base + (size_t)(2 + n - w) * L, *recv_hi = base + (size_t)(2 + n) * L;
    if (c->kind == sw_comm::NCCL) {
        NcclApi &N = nccl();
        CommErr e = comm_nccl(N.GroupStart(), "ncclGroupStart");
        if (e.code) return e;
        if (lo) {
            if ((e = comm_nccl(N.Send(send_lo, cnt, ncclFloat64, c->rank - 1, c->nc, s), "ncclSend")).code) return e;
            if ((e = comm_nccl(N.Recv(recv_lo, cnt, ncclFloat64, c->rank - 1, c->nc, s), "ncclRecv")).code) return e;
        }
        if (hi) {
            if ((e = comm_nccl(N.Send(send_hi, cnt, ncclFloat64, c->rank + 1, c->nc, s), "ncclSend")).code) return e;
            if ((e = comm_nccl(N.Recv(recv_hi, cnt, ncclFloat64, c->rank + 1, c->nc, s), "ncclRecv")).code) return e;
        }
        return comm_nccl(N.GroupEnd(), "ncclGroupEnd");
    }
    CommErr e = stage_reserve(c, 4 * bytes);
    if (e.code) return e;
    unsigned char *h_slo = c->stage, *h_rlo = c->stage + bytes, *h_shi = c->stage + 2 * bytes,
                  *h_rhi = c->stage + 3 * bytes;
    if (lo && (e = comm_cuda(cudaMemcpyAsync(h_slo, send_lo, bytes, cudaMemcpyDeviceToHost, s), "D2H halo")).code)
        return e;
    if (hi && (e = comm_cuda(cudaMemcpyAsync(h_shi, send_hi, bytes, cudaMemcpyDeviceToHost, s), "D2H halo")).code)
        return e;
    if ((e = comm_cuda(cudaStreamSynchronize(s), "halo staging")).code) return e;
    if (c->xfn(c->ctx, lo ? h_slo : nullptr, lo ? h_rlo : nullptr, lo ? bytes : 0, hi ? h_shi : nullptr,
               hi ? h_rhi : nullptr, hi ? bytes : 0) != 0) {
        e.code = 1;
        e.msg = "host exchange callback failed";
        return e;
    }
    if (lo && (e = comm_cuda(cudaMemcpyAsync(recv_lo, h_rlo, bytes, cudaMemcpyHostToDevice, s), "H2D halo")).code)
        return e;
    if (hi && (e = comm_cuda(cudaMemcpyAsync(recv_hi, h_rhi, bytes, cudaMemcpyHostToDevice, s), "H2D halo")).code)
        return e;
    return comm_cuda(cudaStreamSynchronize(s), "halo staging");   // the staging buffer is free again
}

// recv = every rank's `count` doubles of send, in rank order (device buffers, stream s)
inline CommErr comm_allgather(sw_comm *c, const double *send, double *recv, size_t count, cudaStream_t s) {
    if (c->kind == sw_comm::NCCL)
        return comm_nccl(nccl().AllGather(send, recv, count, ncclFloat64, c->nc, s), "ncclAllGather");
    const size_t bytes = count * sizeof(double);
    CommErr e = stage_reserve(c, bytes * (1 + (size_t)c->nranks));
    if (e.code) return e;
    if ((e = comm_cuda(cudaMemcpyAsync(c->stage, send, bytes, cudaMemcpyDeviceToHost, s), "D2H gather")).code)
        return e;
    if ((e = comm_cuda(cudaStreamSynchronize(s), "gather staging")).code) return e;
    if (c->gfn(c->ctx, c->stage, c->stage + bytes, bytes) != 0) {
        e.code = 1;
        e.msg = "host allgather callback failed";
        return e;
    }
    if ((e = comm_cuda(cudaMemcpyAsync(recv, c->stage + bytes, bytes * c->nranks, cudaMemcpyHostToDevice, s),
                       "H2D gather")).code)
        return e;
    return comm_cuda(cudaStreamSynchronize(s), "gather staging");
}

// out[j] = sum over ranks (in rank order) of the double-double pair j of every rank's block of k
// pairs (the all-gathered partial sums), rounded once: identical on every rank.
__global__ void k_rank_sum(const double *gath, int nranks, int k, double *o0, double *o1) {
    const int j = threadIdx.x;
    if (j >= k) return;
    double hi = 0.0, lo = 0.0;
    for (int r = 0; r < nranks; ++r) {
        const double h = gath[(2 * (size_t)r * k) + 2 * j], l = gath[(2 * (size_t)r * k) + 2 * j + 1];
        const double t = hi + h, bp = t - hi;
        const double err = (hi - (t - bp)) + (h - bp);
        hi = t;
        lo = lo + err + l;
    }
    (j == 0 ? o0 : o1)[0] = hi + lo;
}

// p ghost layers of the PCG direction (multi-rank): p_new = z + beta p_old, as every rank forms
// its own interior values (k_pupdate_r / k_pspmv*: fma(beta, p_old, z), p = z on the first
// iteration), on layer `lay` (L doubles) of the padded arrays; bitwise the neighbour's values.
__global__ void k_ghost_pupdate(const double *beta_dev, int first, const double *__restrict__ z,
                                const double *__restrict__ pold, double *__restrict__ pnew, size_t L, size_t lay0,
                                size_t lay1) {
    const double be = first ? 0.0 : *beta_dev;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < 2 * L; t += (size_t)gridDim.x * blockDim.x) {
        const size_t lay = t < L ? lay0 : lay1;   // SIZE_MAX: no neighbour on that side
        if (lay == (size_t)-1) continue;
        const size_t i = lay * L + (t % L);
        pnew[i] = first ? z[i] : fma(be, pold[i], z[i]);
    }
}

}  // namespace sw
