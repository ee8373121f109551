// halo.cu -- halo exchange of a slab rank and the
// one-call-per-step sub-step loop with the exchanges between the phases.
//
// Records are packed / unpacked by the engine's kernels (engine.cu k_pack /
// k_unpack) for all peers at once; NCCL moves each peer's contiguous slice
// with grouped ncclSend / ncclRecv on the engine's stream, so a sub-step is
// enqueued without a host round trip.  NCCL is opened with dlopen on first
// use (no link-time dependency): the copy already in the process (torch's)
// if there is one, else the system library.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>

#include "engine.cuh"

using namespace sph;

namespace {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl()
{
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = (decltype(api.get_unique_id))sym("ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))sym("ncclCommInitRank");
    api.comm_destroy = (decltype(api.comm_destroy))sym("ncclCommDestroy");
    api.group_start = (decltype(api.group_start))sym("ncclGroupStart");
    api.group_end = (decltype(api.group_end))sym("ncclGroupEnd");
    api.send = (decltype(api.send))sym("ncclSend");
    api.recv = (decltype(api.recv))sym("ncclRecv");
    api.all_reduce = (decltype(api.all_reduce))sym("ncclAllReduce");
    api.error_string = (decltype(api.error_string))sym("ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.group_start &&
             api.group_end && api.send && api.recv && api.all_reduce;
    return api;
}

int nccl_check(ncclResult_t r, const char* what)
{
    if (r == ncclSuccess) return SPH_OK;
    static char buf[256];
    const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
    snprintf(buf, sizeof(buf), "%s: NCCL error %d (%s)", what, (int)r, msg);
    set_error(buf);
    return SPH_ERR_CUDA;
}

int need_nccl()
{
    if (nccl().ok) return SPH_OK;
    set_error("NCCL (libnccl.so.2) not available");
    return SPH_ERR_UNSUPPORTED;
}

int plan_valid(const SphHaloPlan* p)
{
    if (!p || p->npeers < 0 || p->npeers > SPH_MAX_PEERS) {
        set_error("halo plan: bad peer count");
        return SPH_ERR_INVALID;
    }
    return SPH_OK;
}

}  // namespace

extern "C" int sph_halo_pack(const SphEngine* e, const SphHaloPlan* plan, int32_t kind,
                             int32_t cls, cudaStream_t s)
{
    int rc = plan_valid(plan);
    if (rc) return rc;
    if (cls < 0 || cls > 1) return SPH_ERR_INVALID;
    const int64_t n = plan->send_off[cls][plan->npeers];
    if (n <= 0) return SPH_OK;
    return sph_engine_pack(e, kind, plan->send_phys[cls], n, plan->send_buf, s);
}

extern "C" int sph_halo_unpack(SphEngine* e, const SphHaloPlan* plan, int32_t kind, int32_t cls,
                               cudaStream_t s)
{
    int rc = plan_valid(plan);
    if (rc) return rc;
    if (cls < 0 || cls > 1) return SPH_ERR_INVALID;
    const int64_t n = plan->recv_off[cls][plan->npeers];
    if (n <= 0) return SPH_OK;
    return sph_engine_unpack(e, kind, plan->recv_phys[cls], n, plan->recv_buf, s);
}

extern "C" size_t sph_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

extern "C" int sph_comm_unique_id(void* id_out)
{
    int rc = need_nccl();
    if (rc) return rc;
    return nccl_check(nccl().get_unique_id((ncclUniqueId*)id_out), "ncclGetUniqueId");
}

extern "C" int sph_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm_out)
{
    int rc = need_nccl();
    if (rc) return rc;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    rc = nccl_check(nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
    if (rc) return rc;
    *comm_out = (void*)c;
    return SPH_OK;
}

extern "C" int sph_comm_destroy(void* comm)
{
    if (!comm) return SPH_OK;
    int rc = need_nccl();
    if (rc) return rc;
    return nccl_check(nccl().comm_destroy((ncclComm_t)comm), "ncclCommDestroy");
}

extern "C" int sph_halo_exchange(SphEngine* e, void* comm, const SphHaloPlan* plan,
                                 int32_t kind, int32_t cls, cudaStream_t s)
{
    int rc = plan_valid(plan);
    if (rc || (rc = need_nccl())) return rc;
    const int w = sph_engine_halo_width(kind);
    if (w < 0 || cls < 0 || cls > 1) return SPH_ERR_INVALID;
    if ((rc = sph_halo_pack(e, plan, kind, cls, s))) return rc;
    const size_t es = e->f64 ? sizeof(double) : sizeof(float);
    const ncclDataType_t dt = e->f64 ? ncclFloat64 : ncclFloat32;
    NcclApi& api = nccl();
    if ((rc = nccl_check(api.group_start(), "ncclGroupStart"))) return rc;
    for (int p = 0; p < plan->npeers && !rc; p++) {
        const int64_t s0 = plan->send_off[cls][p], sn = plan->send_off[cls][p + 1] - s0;
        const int64_t r0 = plan->recv_off[cls][p], rn = plan->recv_off[cls][p + 1] - r0;
        if (sn > 0)
            rc = nccl_check(api.send((const char*)plan->send_buf + (size_t)s0 * w * es,
                                     (size_t)sn * w, dt, plan->peer[p], (ncclComm_t)comm, s),
                            "ncclSend");
        if (!rc && rn > 0)
            rc = nccl_check(api.recv((char*)plan->recv_buf + (size_t)r0 * w * es,
                                     (size_t)rn * w, dt, plan->peer[p], (ncclComm_t)comm, s),
                            "ncclRecv");
    }
    const int rc2 = nccl_check(api.group_end(), "ncclGroupEnd");
    if (rc || rc2) return rc ? rc : rc2;
    return sph_halo_unpack(e, plan, kind, cls, s);
}

// the step statistics of all ranks, reduced in place on the engine stream:
// order-preserving keys and non-negative f64 bits reduce as uint64 max / min,
// counters as sums; the NaN flags are split into one word per bit (max = OR)
__global__ void k_stats_split(SphStepStats* st, unsigned int* w)
{
    w[0] = st->overflow;
    w[1] = st->nfix;
    w[2] = st->nan_flags & 1u;
    w[3] = (st->nan_flags >> 1) & 1u;
}
__global__ void k_stats_merge(SphStepStats* st, const unsigned int* w, int flags)
{
    if (flags & 2) {
        st->overflow = w[0];
        st->nfix = w[1];
    }
    if (flags & 4) st->nan_flags = (w[2] ? 1u : 0u) | (w[3] ? 2u : 0u);
}

extern "C" int sph_stats_allreduce(SphEngine* e, void* comm, int32_t flags, cudaStream_t s)
{
    int rc = need_nccl();
    if (rc) return rc;
    if (!e || !e->stats || !comm || !e->ws || e->ws_bytes < 64) return SPH_ERR_INVALID;
    NcclApi& api = nccl();
    ncclComm_t c = (ncclComm_t)comm;
    SphStepStats* st = e->stats;
    unsigned int* w = reinterpret_cast<unsigned int*>(e->ws);   // free between calls
    const bool words = (flags & 6) != 0;
    if (words) note_launch(), k_stats_split<<<1, 1, 0, s>>>(st, w);
    auto ar = [&](void* p, size_t n, ncclDataType_t t, ncclRedOp_t op) {
        if (rc) return;
        rc = nccl_check(api.all_reduce(p, p, n, t, op, c, s), "ncclAllReduce");
    };
    if ((rc = nccl_check(api.group_start(), "ncclGroupStart"))) return rc;
    if (flags & 1) ar(&st->vmax_bits, 2, ncclUint64, ncclMax);   // vmax, amax (f64 bits >= 0)
    if (flags & 2) {
        ar(&st->interactions, 1, ncclUint64, ncclSum);
        ar(w, 2, ncclUint32, ncclSum);                          // overflow, nfix
    }
    if (flags & 4) {
        ar(&st->rho_min_key, 1, ncclUint64, ncclMin);
        ar(&st->v2max_key, 1, ncclUint64, ncclMax);
        ar(w + 2, 2, ncclUint32, ncclMax);                      // NaN flag bits
    }
    const int rc2 = nccl_check(api.group_end(), "ncclGroupEnd");
    if (rc || rc2) return rc ? rc : rc2;
    if (words) note_launch(), k_stats_merge<<<1, 1, 0, s>>>(st, w, flags);
    return check_launch("stats_allreduce");
}

extern "C" int sph_engine_substeps_slab(SphEngine* e, void* comm, const SphHaloPlan* plan,
                                        double half_dt, double full_dt, int32_t nsub,
                                        cudaStream_t s)
{
    int rc = plan_valid(plan);
    if (rc) return rc;
    for (int k = 0; k < nsub && !rc; k++) {
        if (!rc) rc = sph_engine_phase(e, SPH_PHASE_KICK_DRIFT, half_dt, full_dt, s);
        if (!rc) rc = sph_halo_exchange(e, comm, plan, SPH_HALO_XV, 0, s);
        if (!rc) rc = sph_engine_phase(e, SPH_PHASE_CONTINUITY, half_dt, full_dt, s);
        if (!rc) rc = sph_halo_exchange(e, comm, plan, SPH_HALO_RP_NEXT, 0, s);
        if (!rc) rc = sph_engine_phase(e, SPH_PHASE_WALL, half_dt, full_dt, s);
        if (!rc) rc = sph_halo_exchange(e, comm, plan, SPH_HALO_RP_NEXT, 1, s);
        // all but the last sub-step: the momentum sweep also applies the next
        // sub-step's kick + drift to owned fluid (its KICK_DRIFT phase is then
        // a no-op; the XV refresh after it still updates the ghosts)
        if (!rc) rc = sph_engine_phase(e, k + 1 < nsub ? SPH_PHASE_MOMENTUM_NEXT
                                                       : SPH_PHASE_MOMENTUM,
                                       half_dt, full_dt, s);
    }
    return rc;
}
