// comm.cu -- csrk_comm over NCCL for row-sharded multi-GPU steps (north_star
// "partial gradients combined by NCCL ... over NVLink").
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy torch already loaded in this
// process if there is one), so libcsrk.so has no link-time NCCL dependency and single-GPU users
// never touch it.  nccl.h supplies the types only.
//
//   allreduce_sum  ncclAllReduce(sum, fp64) in place on the caller's stream
//   halo GATHER    one NCCL group: for every peer q, send my owned range q holds as ghosts,
//                  receive my ghost range owned by q (straight into the extended vector)
//   halo REDUCE    one NCCL group: send my ghost range (my partial of q's rows), receive q's
//                  partial of my rows into scratch; then one kernel per peer adds it into the
//                  owned range.  Ghosts are left as they were (undefined by contract).
// All calls are stream-ordered and capturable in a CUDA graph (NCCL >= 2.9).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "csrk_internal.cuh"

namespace csrk {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    bool ok = false;
};

static NcclApi *nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        bool all = true;
        auto get = [&](auto &fp, const char *name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            all &= fp != nullptr;
        };
        get(api.GetUniqueId, "ncclGetUniqueId");
        get(api.CommInitRank, "ncclCommInitRank");
        get(api.CommDestroy, "ncclCommDestroy");
        get(api.AllReduce, "ncclAllReduce");
        get(api.Send, "ncclSend");
        get(api.Recv, "ncclRecv");
        get(api.GroupStart, "ncclGroupStart");
        get(api.GroupEnd, "ncclGroupEnd");
        api.ok = all;
    });
    return api.ok ? &api : nullptr;
}

struct NcclComm {
    ncclComm_t comm = nullptr;
    std::vector<int> peer;
    std::vector<int64_t> own_off, own_len, ghost_off, ghost_len, scr_off;
    double *scratch = nullptr;
};

#define NCCL_TRY(expr)                                  \
    do {                                                \
        if ((expr) != ncclSuccess) return CSRK_ERR_CUDA; \
    } while (0)

__global__ __launch_bounds__(256) void k_add_into(double *__restrict__ dst, const double *__restrict__ src, int64_t n)
{
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) dst[i] += src[i];
}

static int nccl_allreduce(void *ctx, double *buf, int64_t count, csrk_stream_t stream)
{
    NcclApi *api = nccl();
    NcclComm *c = static_cast<NcclComm *>(ctx);
    if (!api || count <= 0) return api ? CSRK_OK : CSRK_ERR_CUDA;
    NCCL_TRY(api->AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, c->comm, (cudaStream_t)stream));
    return CSRK_OK;
}

static int nccl_halo(void *ctx, double *v, int mode, csrk_stream_t stream)
{
    NcclApi *api = nccl();
    if (!api) return CSRK_ERR_CUDA;
    NcclComm *c = static_cast<NcclComm *>(ctx);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t np = c->peer.size();
    if (np == 0) return CSRK_OK;
    NCCL_TRY(api->GroupStart());
    for (size_t q = 0; q < np; ++q) {
        if (mode == 0) {   // gather: owners' values into my ghosts
            if (c->own_len[q]) NCCL_TRY(api->Send(v + c->own_off[q], (size_t)c->own_len[q], ncclFloat64, c->peer[q], c->comm, s));
            if (c->ghost_len[q])
                NCCL_TRY(api->Recv(v + c->ghost_off[q], (size_t)c->ghost_len[q], ncclFloat64, c->peer[q], c->comm, s));
        } else {           // reduce: my ghost partials to their owners, theirs into scratch
            if (c->ghost_len[q])
                NCCL_TRY(api->Send(v + c->ghost_off[q], (size_t)c->ghost_len[q], ncclFloat64, c->peer[q], c->comm, s));
            if (c->own_len[q])
                NCCL_TRY(api->Recv(c->scratch + c->scr_off[q], (size_t)c->own_len[q], ncclFloat64, c->peer[q], c->comm, s));
        }
    }
    NCCL_TRY(api->GroupEnd());
    if (mode == 1)
        for (size_t q = 0; q < np; ++q) {
            const int64_t n = c->own_len[q];
            if (!n) continue;
            const int64_t g = cdiv(n, 256);
            CSRK_LAUNCH(k_add_into, (unsigned)(g < kNumSMs * 4 ? g : kNumSMs * 4), 256, 0, s, v + c->own_off[q],
                        (const double *)(c->scratch + c->scr_off[q]), n);
        }
    return CSRK_OK;
}

}  // namespace csrk

using namespace csrk;

extern "C" {

int csrk_comm_nccl_unique_id(void *id128)
{
    NcclApi *api = nccl();
    if (!id128) return CSRK_ERR_INVALID_ARG;
    if (!api) return CSRK_ERR_CUDA;
    ncclUniqueId id;
    NCCL_TRY(api->GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id128, &id, sizeof(id));
    return CSRK_OK;
}

int csrk_comm_nccl_create(const void *id128, int rank, int world, const csrk_halo *halo, csrk_comm *out)
{
    if (!id128 || !out || !halo || world < 1 || rank < 0 || rank >= world || halo->npeers < 0) return CSRK_ERR_INVALID_ARG;
    if (halo->npeers > 0 && (!halo->peer || !halo->own_off || !halo->own_len || !halo->ghost_off || !halo->ghost_len))
        return CSRK_ERR_INVALID_ARG;
    NcclApi *api = nccl();
    if (!api) return CSRK_ERR_CUDA;
    NcclComm *c = new NcclComm();
    int64_t scr = 0;
    for (int q = 0; q < halo->npeers; ++q) {
        if (halo->peer[q] < 0 || halo->peer[q] >= world || halo->peer[q] == rank || halo->own_len[q] < 0 ||
            halo->ghost_len[q] < 0) {
            delete c;
            return CSRK_ERR_INVALID_ARG;
        }
        c->peer.push_back(halo->peer[q]);
        c->own_off.push_back(halo->own_off[q]);
        c->own_len.push_back(halo->own_len[q]);
        c->ghost_off.push_back(halo->ghost_off[q]);
        c->ghost_len.push_back(halo->ghost_len[q]);
        c->scr_off.push_back(scr);
        scr += halo->own_len[q];
    }
    if (scr > 0 && cudaMalloc(&c->scratch, sizeof(double) * (size_t)scr) != cudaSuccess) {
        delete c;
        return CSRK_ERR_CUDA;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    if (api->CommInitRank(&c->comm, world, id, rank) != ncclSuccess) {
        if (c->scratch) cudaFree(c->scratch);
        delete c;
        return CSRK_ERR_CUDA;
    }
    out->ctx = c;
    out->allreduce_sum = nccl_allreduce;
    out->halo = nccl_halo;
    out->capturable = 1;
    return CSRK_OK;
}

int csrk_comm_nccl_destroy(csrk_comm *comm)
{
    if (!comm || !comm->ctx) return CSRK_ERR_INVALID_ARG;
    NcclComm *c = static_cast<NcclComm *>(comm->ctx);
    NcclApi *api = nccl();
    if (api && c->comm) api->CommDestroy(c->comm);
    if (c->scratch) cudaFree(c->scratch);
    delete c;
    comm->ctx = nullptr;
    return CSRK_OK;
}

}  // extern "C"
