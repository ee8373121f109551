// layout.cu -- engine layout management: registry <-> SoA, the per-step CLL
// rebuild (fluid re-sort by cell), the reference-order mirror and the step
// reductions.
//
// physics.py:446-449 _rebuild_cll rebuilds the reference's cell linked list
// every advective step; on the device that IS a stable re-sort of the fluid
// segment by cell key (radix sort, sort.cu) followed by one fused gather of
// every per-particle field and a per-cell lower-bound for the offsets.
// Walls never move, so their segment is sorted once, at push.
#include <cstddef>

#include "engine.cuh"

namespace sph {

// push-time registry checks (the former host-side O(n) scans): ids must be
// a permutation of 0..n-1.  k_push_place flags an out-of-range id; the
// duplicate count runs in the second half of the push (k_id_count over the
// placed ids, off the path to the list build), so the first half needs no
// scratch that the list build reuses.
__global__ void k_id_count(const uint32_t* __restrict__ id, int64_t n,
                           uint32_t* __restrict__ cnt)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) atomicAdd(&cnt[id[r]], 1u);   // placed ids are in range
}

__global__ void k_id_check(const uint32_t* __restrict__ cnt, int64_t n, SphStepStats* st)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n && cnt[r] != 1u) st->push_error = 1;
}

// cell keys of the push (the wall flag above the cell bits), the clamp
// counts, and the fluid count the host checks against the allocation
template <class T, int D>
__global__ void k_push_keys(const T* __restrict__ x, const uint32_t* __restrict__ wall, int64_t n,
                            GridP<T> g, int key_bits, uint32_t* __restrict__ keys,
                            SphStepStats* __restrict__ st)
{
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int cl = 0;
    bool is_wall = false;
    if (r < n) {
        int c0 = cell_coord<T>(x[r * D], g.o[0], g.cs, g.s[0], cl);
        int c1 = cell_coord<T>(x[r * D + 1], g.o[1], g.cs, g.s[1], cl);
        uint32_t lin = (uint32_t)c0 * g.s[1] + c1;
        if (D == 3) lin = lin * g.s[2] + cell_coord<T>(x[r * D + 2], g.o[2], g.cs, g.s[2], cl);
        is_wall = wall[r] != 0;
        keys[r] = lin | (is_wall ? (1u << key_bits) : 0u);
    }
    unsigned b = __ballot_sync(0xffffffffu, cl && is_wall);
    if (lane_id() == 0 && b) atomicAdd(&st->oob_walls, (uint32_t)__popc(b));
    // fluid clamps: what this step's CLL build counts (k_fluid_keys) when the
    // push's cell order stands in for it
    b = __ballot_sync(0xffffffffu, cl && r < n && !is_wall);
    if (lane_id() == 0 && b) atomicAdd(&st->oob, (uint32_t)__popc(b));
    b = __ballot_sync(0xffffffffu, r < n && !is_wall);
    if (lane_id() == 0 && b) atomicAdd(&st->fluid_seen, (uint32_t)__popc(b));
}

// push, first half: the particle's place (cell order), position, identity;
// refpos[i] = its registry row, which the second half gathers by (the mass
// in pos.w comes with the second half: the list build does not read it)
template <class T, int D>
__global__ void k_push_place(Eng<T> E, const uint32_t* __restrict__ perm, const T* __restrict__ x,
                             const uint32_t* __restrict__ id, const uint32_t* __restrict__ wall)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    uint32_t r = perm[i];
    vec4<T> P4;
    P4.x = x[r * D]; P4.y = x[r * D + 1]; P4.z = D == 3 ? x[r * D + 2] : T(0); P4.w = T(0);
    E.pos[i] = P4; E.pos_next[i] = P4;   // walls stay valid in both buffers
    uint32_t pid = id[r];
    // an out-of-range id is reported (push_error, raised by the host before
    // the state is used) and stored as 0, so that the list build an
    // overlapped push queues before that check indexes in bounds
    if (pid >= (uint64_t)E.idr) {
        E.stats->push_error = 1;
        pid = 0;
    }
    E.id[i] = pid;
    E.refpos[i] = r;
    E.wall_id[pid] = wall[r];
}

// push, second half: every other field from registry row refpos[i]
template <class T, int D>
__global__ void k_push_fields(Eng<T> E, const T* __restrict__ v, const T* __restrict__ rho,
                              const T* __restrict__ p, const T* __restrict__ m,
                              const T* __restrict__ vol,
                              const T* __restrict__ drho, const T* __restrict__ dvdt,
                              const T* __restrict__ rho_scratch, const uint32_t* __restrict__ nnb,
                              const uint32_t* __restrict__ oflow)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    uint32_t r = E.refpos[i];
    vec4<T> V4, A4;
    V4.x = v[r * D]; V4.y = v[r * D + 1]; V4.z = D == 3 ? v[r * D + 2] : T(0); V4.w = T(0);
    A4.x = dvdt[r * D]; A4.y = dvdt[r * D + 1]; A4.z = D == 3 ? dvdt[r * D + 2] : T(0);
    A4.w = T(0);
    vec2<T> RP; RP.x = rho[r]; RP.y = p[r];
    reinterpret_cast<T*>(&E.pos[i])[3] = m[r];
    reinterpret_cast<T*>(&E.pos_next[i])[3] = m[r];
    E.vel[0][i] = V4; E.vel[1][i] = V4;
    E.rp[0][i] = RP; E.rp[1][i] = RP;
    E.dvdt[i] = A4;
    E.drho[i] = drho[r];
    E.nnb[i] = nnb[r];
    const uint32_t pid = E.id[i];   // in range (k_push_place)
    if (rho_scratch) E.rho_scratch_id[pid] = rho_scratch[r];   // else: sph_engine_push_tail
    if (oflow) E.oflow_id[pid] = oflow[r];
    if (vol) E.vol_id[pid] = vol[r];
}

// the by-id fields a push deferred (registry order in, by id out): oflow
// keeps the flags the step's sweeps set meanwhile
template <class T>
__global__ void k_push_tail(Eng<T> E, const uint32_t* __restrict__ id, int64_t n,
                            const T* __restrict__ vol, const T* __restrict__ rho_scratch,
                            const uint32_t* __restrict__ oflow)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t pid = id[r];
    if (pid >= (uint64_t)E.idr) return;   // the push reported it (push_error)
    if (vol) E.vol_id[pid] = vol[r];
    if (rho_scratch) E.rho_scratch_id[pid] = rho_scratch[r];
    // flagged by this step's sweeps: 1 (as the plain push's value would have
    // been overwritten); else the pushed value
    if (oflow && E.oflow_id[pid] == 0u) E.oflow_id[pid] = oflow[r];
}

// registry-order copies of the fields in mask (bit k: field k of x, v, rho,
// p, m, Vol, drho, dvdt, rho_scratch, id, wall, nnb, oflow)
template <class T, int D>
__global__ void k_pull(Eng<T> E, int cur_v, int cur_rp, uint32_t mask, T* __restrict__ x,
                       T* __restrict__ v, T* __restrict__ rho, T* __restrict__ p,
                       T* __restrict__ m, T* __restrict__ vol, T* __restrict__ drho,
                       T* __restrict__ dvdt, T* __restrict__ rho_scratch,
                       uint32_t* __restrict__ id, uint32_t* __restrict__ wall,
                       uint32_t* __restrict__ nnb, uint32_t* __restrict__ oflow)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    const uint32_t r = E.refpos[i];
    const uint32_t pid = E.id[i];
    if (mask & (1u << 0)) {
        const vec4<T> P4 = E.pos[i];
        x[r * D] = P4.x; x[r * D + 1] = P4.y;
        if (D == 3) x[r * D + 2] = P4.z;
    }
    if (mask & (1u << 1)) {
        const vec4<T> V4 = E.vel[cur_v][i];
        v[r * D] = V4.x; v[r * D + 1] = V4.y;
        if (D == 3) v[r * D + 2] = V4.z;
    }
    if (mask & (3u << 2)) {
        const vec2<T> RP = E.rp[cur_rp][i];
        if (mask & (1u << 2)) rho[r] = RP.x;
        if (mask & (1u << 3)) p[r] = RP.y;
    }
    if (mask & (1u << 4)) m[r] = E.pos[i].w;
    if (mask & (1u << 5)) vol[r] = E.vol_id[pid];
    if (mask & (1u << 6)) drho[r] = E.drho[i];
    if (mask & (1u << 7)) {
        const vec4<T> A4 = E.dvdt[i];
        dvdt[r * D] = A4.x; dvdt[r * D + 1] = A4.y;
        if (D == 3) dvdt[r * D + 2] = A4.z;
    }
    if (mask & (1u << 8)) rho_scratch[r] = E.rho_scratch_id[pid];
    if (mask & (1u << 9)) id[r] = pid;
    if (mask & (1u << 10)) wall[r] = E.wall_id[pid];
    if (mask & (1u << 11)) nnb[r] = E.nnb[i];
    if (mask & (1u << 12)) oflow[r] = E.oflow_id[pid];
}

static void seg_offsets(const uint32_t* keys, int64_t n, int64_t ncells, uint32_t or_mask,
                        uint32_t* offsets, cudaStream_t s);

// offsets of a segment whose sorted keys carry or_mask in the high bit
__global__ void k_seg_offsets(const uint32_t* __restrict__ keys, int64_t n, int64_t ncells,
                              uint32_t or_mask, uint32_t* __restrict__ offsets)
{
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncells) return;
    uint32_t target = (uint32_t)c | or_mask;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    offsets[c] = (uint32_t)lo;
}


// fluid cell keys for the per-step re-sort (neighborhood.py:105-117 on pos)
template <class T, int D>
__global__ void k_fluid_keys(const vec4<T>* __restrict__ pos, int64_t nf, GridP<T> g,
                             uint32_t* __restrict__ keys, unsigned int* __restrict__ oob)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int cl = 0;
    if (i < nf) {
        vec4<T> P4 = pos[i];
        int c0 = cell_coord<T>(P4.x, g.o[0], g.cs, g.s[0], cl);
        int c1 = cell_coord<T>(P4.y, g.o[1], g.cs, g.s[1], cl);
        uint32_t lin = (uint32_t)c0 * g.s[1] + c1;
        if (D == 3) lin = lin * g.s[2] + cell_coord<T>(P4.z, g.o[2], g.cs, g.s[2], cl);
        keys[i] = lin;
    }
    unsigned b = __ballot_sync(0xffffffffu, cl);
    if (lane_id() == 0 && b) atomicAdd(oob, (unsigned)__popc(b));
}

// all-particle cell keys scattered to registry order (sort_particles_by_cell)
template <class T, int D>
__global__ void k_ref_keys(const vec4<T>* __restrict__ pos, const uint32_t* __restrict__ refpos,
                           int64_t n, GridP<T> g, uint32_t* __restrict__ keys_by_ref,
                           uint32_t* __restrict__ phys_by_ref)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int cl = 0;
    vec4<T> P4 = pos[i];
    int c0 = cell_coord<T>(P4.x, g.o[0], g.cs, g.s[0], cl);
    int c1 = cell_coord<T>(P4.y, g.o[1], g.cs, g.s[1], cl);
    uint32_t lin = (uint32_t)c0 * g.s[1] + c1;
    if (D == 3) lin = lin * g.s[2] + cell_coord<T>(P4.z, g.o[2], g.cs, g.s[2], cl);
    uint32_t r = refpos[i];
    keys_by_ref[r] = lin;
    phys_by_ref[r] = (uint32_t)i;
}

__global__ void k_ref_assign(const uint32_t* __restrict__ phys_sorted, int64_t n,
                             uint32_t* __restrict__ refpos)
{
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) refpos[phys_sorted[r]] = (uint32_t)r;
}

// fused gather of every per-particle field of the fluid segment by perm; for
// walls only the (rho, p) buffer becoming current is refreshed (velocity
// buffers always agree on the never-moving walls)
template <class T>
__global__ void k_fluid_gather(const uint32_t* __restrict__ perm, int64_t nf, int64_t n,
                               const vec4<T>* __restrict__ pos, vec4<T>* __restrict__ pos_o,
                               const vec4<T>* __restrict__ vel, vec4<T>* __restrict__ vel_o,
                               const vec2<T>* __restrict__ rp, vec2<T>* __restrict__ rp_o,
                               const vec4<T>* __restrict__ dvdt, vec4<T>* __restrict__ dvdt_o,
                               const T* __restrict__ drho, T* __restrict__ drho_o,
                               const uint32_t* __restrict__ id, uint32_t* __restrict__ id_o,
                               const uint32_t* __restrict__ refpos,
                               uint32_t* __restrict__ refpos_o,
                               const uint32_t* __restrict__ nnb, uint32_t* __restrict__ nnb_o)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) {
        if (i < n) rp_o[i] = rp[i];
        return;
    }
    uint32_t r = perm[i];
    pos_o[i] = pos[r];
    vel_o[i] = vel[r];
    rp_o[i] = rp[r];
    dvdt_o[i] = dvdt[r];
    drho_o[i] = drho[r];
    id_o[i] = id[r];
    refpos_o[i] = refpos[r];
    nnb_o[i] = nnb[r];
}

// persistent-list bookkeeping of a fluid re-sort (engine.cu maintain):
// key_prev[i] = the previous CLL's key of new particle i (key_sorted still
// holds the previous sorted keys, in the old order), inv = old -> new
__global__ void __launch_bounds__(256)
k_resort_keys(const uint32_t* __restrict__ perm, int64_t nf,
              const uint32_t* __restrict__ key_sorted, uint32_t* __restrict__ key_prev,
              uint32_t* __restrict__ inv)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const uint32_t o = perm[i];
    key_prev[i] = key_sorted[o];
    inv[o] = (uint32_t)i;
}

// the per-particle list state travels with its particle through the re-sort
template <class T>
__global__ void __launch_bounds__(256)
k_resort_list_state(const uint32_t* __restrict__ perm, int64_t nf,
                    const uint32_t* __restrict__ cell0, uint32_t* __restrict__ cell0_o,
                    const T* __restrict__ disp, T* __restrict__ disp_o,
                    const T* __restrict__ disp0, T* __restrict__ disp0_o)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const uint32_t o = perm[i];
    cell0_o[i] = cell0[o];
    disp_o[i] = disp[o];
    disp0_o[i] = disp0[o];
}

// the static cells of the walls (push: sorted keys carry a wall flag bit)
__global__ void __launch_bounds__(256)
k_strip_keys(const uint32_t* __restrict__ sk, int64_t n, uint32_t mask, uint32_t* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = sk[i] & mask;
}

// exact max |v|, |dvdt| (physics.py:296-310 / 390-391) and the stability
// inputs min rho, max run-precision |v|^2 (physics.py:554-564), all particles
template <class T, int D>
__global__ void k_stats(Eng<T> E, int cv, int crp)
{
    double vm = 0.0, am = 0.0;
    unsigned long long rmin = ~0ull, v2k = 0ull;
    unsigned nanf = 0u;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!is_owned(E, i)) continue;
        vec4<T> V4 = E.vel[cv][i], A4 = E.dvdt[i];
        T vv[3], aa[3];
        to3<T>(V4, vv);
        to3<T>(A4, aa);
        double sv = 0.0, sa = 0.0;
        T s2 = T(0);
#pragma unroll
        for (int k = 0; k < D; k++) {
            T pv = RN<T>::mul(vv[k], vv[k]);
            sv = dadd(sv, double(pv));
            sa = dadd(sa, double(RN<T>::mul(aa[k], aa[k])));
            s2 = RN<T>::add(s2, pv);
        }
        sv = __dsqrt_rn(sv);
        sa = __dsqrt_rn(sa);
        vm = sv > vm ? sv : vm;
        am = sa > am ? sa : am;
        const T rr = E.rp[crp][i].x;
        unsigned long long rk = dkey(double(rr));
        rmin = rk < rmin ? rk : rmin;
        unsigned long long vk = dkey(double(s2));
        v2k = vk > v2k ? vk : v2k;
        // numpy's min/max propagate NaN (physics.py:556, 561)
        nanf |= (rr != rr ? 1u : 0u) | (s2 != s2 ? 2u : 0u);
    }
    nanf = __reduce_or_sync(0xffffffffu, nanf);
    unsigned long long vb = warp_max_u64(dbits(vm));
    unsigned long long ab = warp_max_u64(dbits(am));
    v2k = warp_max_u64(v2k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, rmin, o);
        rmin = w < rmin ? w : rmin;
    }
    if (lane_id() == 0) {
        atomicMax(&E.stats->vmax_bits, vb);
        atomicMax(&E.stats->amax_bits, ab);
        atomicMin(&E.stats->rho_min_key, rmin);
        atomicMax(&E.stats->v2max_key, v2k);
        if (nanf) atomicOr(&E.stats->nan_flags, nanf);
    }
}

// physics.py:589-606 sample_pressure, device half: the fluid particles
// within reach of a probe (binary64 distance, conservatively widened; the
// host applies the reference's exact test), one record each:
// (registry position, x, y, z, m, rho, p) as binary64 (exact widening)
template <class T, int D>
__global__ void k_probe(Eng<T> E, int crp, double lx, double ly, double lz, double r2max,
                        double* __restrict__ out, int cap, unsigned int* __restrict__ count)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.nf) return;
    const vec4<T> P4 = E.pos[i];
    const double dx = dsub(double(P4.x), lx), dy = dsub(double(P4.y), ly);
    double r2 = dadd(dmul(dx, dx), dmul(dy, dy));
    if (D == 3) {
        const double dz = dsub(double(P4.z), lz);
        r2 = dadd(r2, dmul(dz, dz));
    }
    if (!(r2 < r2max)) return;
    const unsigned k = atomicAdd(count, 1u);
    if ((int)k >= cap) return;
    const vec2<T> RP = E.rp[crp][i];
    double* o = out + 7 * (size_t)k;
    o[0] = double(E.refpos[i]);
    o[1] = double(P4.x); o[2] = double(P4.y); o[3] = D == 3 ? double(P4.z) : 0.0;
    o[4] = double(P4.w); o[5] = double(RP.x); o[6] = double(RP.y);
}

// report.py:187-205 snapshot fields by original id: row id of out holds
// x[D], v[D], rho, p (run precision)
template <class T, int D>
__global__ void k_snapshot(Eng<T> E, int cv, int crp, T* __restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    const vec4<T> P4 = E.pos[i], V4 = E.vel[cv][i];
    const vec2<T> RP = E.rp[crp][i];
    T* o = out + (size_t)E.id[i] * (2 * D + 2);
    o[0] = P4.x; o[1] = P4.y;
    if (D == 3) o[2] = P4.z;
    o[D] = V4.x; o[D + 1] = V4.y;
    if (D == 3) o[D + 2] = V4.z;
    o[2 * D] = RP.x; o[2 * D + 1] = RP.y;
}

static void seg_offsets(const uint32_t* keys, int64_t n, int64_t ncells, uint32_t or_mask,
                        uint32_t* offsets, cudaStream_t s)
{
    note_launch(), k_seg_offsets<<<grid_for(ncells + 1, 256), 256, 0, s>>>(keys, n, ncells,
                                                                         or_mask, offsets);
}

}  // namespace sph

using namespace sph;

template <class T, int D>
static int snapshot_impl(const SphEngine* e, void* out, cudaStream_t s)
{
    if (e->n > 0)
        note_launch(), k_snapshot<T, D><<<grid_for(e->n, 256), 256, 0, s>>>(
            eng_of<T>(e), e->cur_v, e->cur_rp, (T*)out);
    return check_launch("engine_snapshot");
}

extern "C" int sph_engine_snapshot(const SphEngine* e, void* out, cudaStream_t s)
{
    int rc = engine_validate(e);
    if (rc) return rc;
    return SPH_DISPATCH(e, snapshot_impl, e, out, s);
}

template <class T, int D>
static int probe_impl(const SphEngine* e, const double* loc, double radius, double* out,
                      int32_t cap, unsigned int* count, cudaStream_t s)
{
    cudaMemsetAsync(count, 0, sizeof(unsigned int), s);
    if (e->nf > 0)
        note_launch(), k_probe<T, D><<<grid_for(e->nf, 256), 256, 0, s>>>(
            eng_of<T>(e), e->cur_rp, loc[0], loc[1], D == 3 ? loc[2] : 0.0, radius * radius,
            out, cap, count);
    return check_launch("engine_probe");
}

extern "C" int sph_engine_probe(const SphEngine* e, const double* loc, double radius, double* out,
                                int32_t cap, unsigned int* count, cudaStream_t s)
{
    int rc = engine_validate(e);
    if (rc) return rc;
    return SPH_DISPATCH(e, probe_impl, e, loc, radius, out, cap, count, s);
}

static size_t engine_sort_bytes(int64_t n)
{
    size_t m = (size_t)(n > 0 ? n : 1);
    return 4 * align_up(sizeof(uint32_t) * m) + radix_hist_bytes(n);
}

extern "C" size_t sph_engine_workspace_bytes_ids(int64_t n, int64_t ncells, int32_t f64,
                                                 int64_t id_range)
{
    // the skin build's phys_of_id map is indexed by id
    // (id_range itself, not id_range - n: the size must not shrink with n)
    const size_t base = sph_engine_workspace_bytes(n, ncells, f64);
    const int64_t extra = id_range > 0 ? id_range : 0;
    return base + align_up(sizeof(uint32_t) * (size_t)extra);
}

extern "C" size_t sph_engine_workspace_bytes(int64_t n, int64_t ncells, int32_t f64)
{
    size_t m = (size_t)(n > 0 ? n : 1);
    size_t es = f64 ? 8 : 4;
    // sort scratch + spare buffers for the fused fluid gather
    const size_t rebuild = engine_sort_bytes(n) + 2 * align_up(4 * es * m) + align_up(es * m) +
                           3 * align_up(sizeof(uint32_t) * m) + 4096;
    // list maintenance: three per-cell arrays, the movers, scan scratch
    const int64_t nc = ncells + 1;
    const size_t maintain = 3 * align_up(sizeof(uint32_t) * (size_t)nc) +
                            align_up(sizeof(uint32_t) * m) + scan_scratch_bytes(nc) + 4096;
    return rebuild > maintain ? rebuild : maintain;
}

struct SortBufs { uint32_t *k0, *k1, *v0, *v1; void* hist; };

static SortBufs sort_bufs(const SphEngine* e, Bump& bump)
{
    SortBufs b;
    b.k0 = bump.take<uint32_t>(e->n);
    b.k1 = bump.take<uint32_t>(e->n);
    b.v0 = bump.take<uint32_t>(e->n);
    b.v1 = bump.take<uint32_t>(e->n);
    b.hist = bump.take<char>(radix_hist_bytes(e->n));
    return b;
}

static int validate_ws(const SphEngine* e)
{
    int rc = engine_validate(e);
    if (rc) return rc;
    if (e->ws_bytes < sph_engine_workspace_bytes_ids(e->n, e->ncells, e->f64, e->id_range)) {
        set_error("engine: workspace too small");
        return SPH_ERR_WORKSPACE;
    }
    return SPH_OK;
}

template <class T, int D>
static int push_begin_impl(SphEngine* e, const void* x, const uint32_t* id,
                           const uint32_t* wall, cudaStream_t s)
{
    Bump bump(e->ws, e->ws_bytes);
    SortBufs sb = sort_bufs(e, bump);
    if (!sb.hist) return SPH_ERR_WORKSPACE;
    GridP<T> g = grid_of_engine<T>(e);
    Eng<T> E = eng_of<T>(e);
    const int64_t n = e->n;
    cudaMemsetAsync(e->stats, 0, sizeof(SphStepStats), s);
    if (n > 0) {
        note_launch(), k_push_keys<T, D><<<grid_for(n, 256), 256, 0, s>>>(
            (const T*)x, wall, n, g, e->key_bits, sb.k0, e->stats);
        int which = 0;
        int rc = radix_sort_u32(sb.k0, sb.k1, sb.v0, sb.v1, n, e->key_bits + 1, true, sb.hist,
                                &which, s);
        if (rc) return rc;
        const uint32_t* sk = which ? sb.k1 : sb.k0;
        const uint32_t* perm = which ? sb.v1 : sb.v0;
        note_launch(), k_push_place<T, D><<<grid_for(n, 256), 256, 0, s>>>(
            E, perm, (const T*)x, id, wall);
        // fluid offsets over sk[0, nf), wall offsets over sk[nf, n) (flag bit set)
        seg_offsets(sk, e->nf, e->ncells, 0u, e->offs_f, s);
        seg_offsets(sk + e->nf, n - e->nf, e->ncells, 1u << e->key_bits, e->offs_w, s);
        if (e->key_sorted)   // every particle's cell (walls keep theirs for good)
            note_launch(), k_strip_keys<<<grid_for(n, 256), 256, 0, s>>>(
                sk, n, (1u << e->key_bits) - 1u, e->key_sorted);
    } else {
        cudaMemsetAsync(e->offs_f, 0, sizeof(uint32_t) * (size_t)(e->ncells + 1), s);
        cudaMemsetAsync(e->offs_w, 0, sizeof(uint32_t) * (size_t)(e->ncells + 1), s);
    }
    e->cur_v = 0;
    e->cur_rp = 0;
    e->cur_pos = 0;
    e->drifted = 0;
    e->lists_ready = 0;
    e->lists_stale = 0;
    e->nww_ready = 0;
    e->cll_fresh = 1;
    return check_launch("engine_push_begin");
}

template <class T, int D>
static int push_end_impl(SphEngine* e, const void* v, const void* rho, const void* p,
                         const void* m, const void* vol, const void* drho, const void* dvdt,
                         const void* rho_scratch, const uint32_t* nnb, const uint32_t* oflow,
                         cudaStream_t s)
{
    const int64_t n = e->n;
    if (n > 0) {
        if (!oflow)   // deferred to sph_engine_push_tail, which ORs into these
            cudaMemsetAsync(e->oflow_id, 0, sizeof(uint32_t) * (size_t)eng_of<T>(e).idr, s);
        note_launch(), k_push_fields<T, D><<<grid_for(n, 256), 256, 0, s>>>(
            eng_of<T>(e), (const T*)v, (const T*)rho, (const T*)p, (const T*)m, (const T*)vol,
            (const T*)drho, (const T*)dvdt, (const T*)rho_scratch, nnb, oflow);
        if (e->id_range <= 0) {   // duplicates (id_range mode: distinct by contract)
            Bump bump(e->ws, e->ws_bytes);
            uint32_t* cnt = bump.take<uint32_t>(n);
            if (!cnt) return SPH_ERR_WORKSPACE;
            cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (size_t)n, s);
            note_launch(), k_id_count<<<grid_for(n, 256), 256, 0, s>>>(e->id, n, cnt);
            note_launch(), k_id_check<<<grid_for(n, 256), 256, 0, s>>>(cnt, n, e->stats);
        }
    }
    return check_launch("engine_push_end");
}

template <class T, int D>
static int push_tail_impl(SphEngine* e, const uint32_t* id, const void* vol,
                          const void* rho_scratch, const uint32_t* oflow, cudaStream_t s)
{
    if (e->n > 0)
        note_launch(), k_push_tail<T><<<grid_for(e->n, 256), 256, 0, s>>>(
            eng_of<T>(e), id, e->n, (const T*)vol, (const T*)rho_scratch, oflow);
    return check_launch("engine_push_tail");
}

extern "C" int sph_engine_push_tail(SphEngine* e, const uint32_t* id, const void* vol,
                                    const void* rho_scratch, const uint32_t* oflow,
                                    cudaStream_t s)
{
    int rc = engine_validate(e);
    if (rc) return rc;
    if (!id) return SPH_ERR_INVALID;
    return SPH_DISPATCH(e, push_tail_impl, e, id, vol, rho_scratch, oflow, s);
}

extern "C" int sph_engine_push_begin(SphEngine* e, const void* x, const uint32_t* id,
                                     const uint32_t* wall, cudaStream_t s)
{
    int rc = validate_ws(e);
    if (rc) return rc;
    return SPH_DISPATCH(e, push_begin_impl, e, x, id, wall, s);
}

extern "C" int sph_engine_push_end(SphEngine* e, const void* v, const void* rho, const void* p,
                                   const void* m, const void* vol, const void* drho, const void* dvdt,
                                   const void* rho_scratch, const uint32_t* nnb,
                                   const uint32_t* oflow, cudaStream_t s)
{
    int rc = validate_ws(e);
    if (rc) return rc;
    return SPH_DISPATCH(e, push_end_impl, e, v, rho, p, m, vol, drho, dvdt, rho_scratch, nnb,
                        oflow, s);
}

extern "C" int sph_engine_push(SphEngine* e, const void* x, const void* v, const void* rho,
                               const void* p, const void* m, const void* vol, const void* drho,
                               const void* dvdt, const void* rho_scratch, const uint32_t* id,
                               const uint32_t* wall, const uint32_t* nnb, const uint32_t* oflow,
                               cudaStream_t s)
{
    int rc = sph_engine_push_begin(e, x, id, wall, s);
    if (rc) return rc;
    return sph_engine_push_end(e, v, rho, p, m, vol, drho, dvdt, rho_scratch, nnb, oflow, s);
}

template <class T, int D>
static int pull_impl(const SphEngine* e, uint32_t mask, void* x, void* v, void* rho, void* p,
                     void* m, void* vol, void* drho, void* dvdt, void* rho_scratch, uint32_t* id,
                     uint32_t* wall, uint32_t* nnb, uint32_t* oflow, cudaStream_t s)
{
    if (e->n <= 0 || !mask) return SPH_OK;
    Eng<T> E = eng_of<T>(e);
    note_launch(), k_pull<T, D><<<grid_for(e->n, 256), 256, 0, s>>>(
        E, e->cur_v, e->cur_rp, mask, (T*)x, (T*)v, (T*)rho, (T*)p, (T*)m, (T*)vol, (T*)drho,
        (T*)dvdt, (T*)rho_scratch, id, wall, nnb, oflow);
    return check_launch("engine_pull");
}

extern "C" int sph_engine_pull(const SphEngine* e, void* x, void* v, void* rho, void* p, void* m,
                               void* vol, void* drho, void* dvdt, void* rho_scratch,
                               uint32_t* id, uint32_t* wall, uint32_t* nnb, uint32_t* oflow,
                               cudaStream_t s)
{
    return sph_engine_pull_fields(e, 0x1fffu, x, v, rho, p, m, vol, drho, dvdt, rho_scratch, id,
                                  wall, nnb, oflow, s);
}

extern "C" int sph_engine_pull_fields(const SphEngine* e, uint32_t mask, void* x, void* v,
                                      void* rho, void* p, void* m, void* vol, void* drho,
                                      void* dvdt, void* rho_scratch, uint32_t* id,
                                      uint32_t* wall, uint32_t* nnb, uint32_t* oflow,
                                      cudaStream_t s)
{
    int rc = engine_validate(e);
    if (rc) return rc;
    void* ptrs[13] = {x, v, rho, p, m, vol, drho, dvdt, rho_scratch, id, wall, nnb, oflow};
    for (int k = 0; k < 13; k++)
        if (((mask >> k) & 1u) && !ptrs[k]) return SPH_ERR_INVALID;
    if (mask >> 13) return SPH_ERR_INVALID;
    return SPH_DISPATCH(e, pull_impl, e, mask, x, v, rho, p, m, vol, drho, dvdt, rho_scratch, id,
                        wall, nnb, oflow, s);
}

template <class T, int D>
static int rebuild_impl(SphEngine* e, cudaStream_t s)
{
    const int64_t nf = e->nf;
    // lists valid until now can be carried across this rebuild (maintain)
    e->lists_stale = e->lists_ready && e->key_sorted ? 1 : 0;
    e->lists_ready = 0;
    e->cll_fresh = 1;   // walls never move: their order stays current
    if (nf <= 0) return SPH_OK;
    Bump bump(e->ws, e->ws_bytes);
    SortBufs sb = sort_bufs(e, bump);
    vec4<T>* pos_o = bump.take<vec4<T>>(e->n);
    vec4<T>* dvdt_o = bump.take<vec4<T>>(e->n);
    T* drho_o = bump.take<T>(e->n);
    uint32_t* id_o = bump.take<uint32_t>(e->n);
    uint32_t* ref_o = bump.take<uint32_t>(e->n);
    uint32_t* nnb_o = bump.take<uint32_t>(e->n);
    if (!nnb_o) return SPH_ERR_WORKSPACE;
    GridP<T> g = grid_of_engine<T>(e);
    Eng<T> E = eng_of<T>(e);
    note_launch(), k_fluid_keys<T, D><<<grid_for(nf, 256), 256, 0, s>>>(E.pos, nf, g, sb.k0,
                                                                        &e->stats->oob);
    int which = 0;
    int rc = radix_sort_u32(sb.k0, sb.k1, sb.v0, sb.v1, nf, e->key_bits, true, sb.hist, &which, s);
    if (rc) return rc;
    const uint32_t* sk = which ? sb.k1 : sb.k0;
    const uint32_t* perm = which ? sb.v1 : sb.v0;
    const int cv = e->cur_v, crp = e->cur_rp;
    note_launch(), k_fluid_gather<T><<<grid_for(e->n, 256), 256, 0, s>>>(
        perm, nf, e->n, E.pos, pos_o, E.vel[cv], E.vel[cv ^ 1], E.rp[crp], E.rp[crp ^ 1], E.dvdt,
        dvdt_o, E.drho, drho_o, E.id, id_o, E.refpos, ref_o, E.nnb, nnb_o);
    // the gathered fluid prefix goes back into the primary arrays; the wall
    // suffix there is untouched (walls never move)
    const size_t es = sizeof(T);
    cudaMemcpyAsync(e->pos[e->cur_pos], pos_o, 4 * es * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->dvdt, dvdt_o, 4 * es * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->drho, drho_o, es * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->id, id_o, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->refpos, ref_o, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->nnb, nnb_o, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    e->cur_v = cv ^ 1;
    e->cur_rp = crp ^ 1;
    seg_offsets(sk, nf, e->ncells, 0u, e->offs_f, s);
    if (e->key_sorted) {
        note_launch(), k_resort_keys<<<grid_for(nf, 256), 256, 0, s>>>(perm, nf, e->key_sorted,
                                                                       e->key_prev, e->inv);
        cudaMemcpyAsync(e->key_sorted, sk, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(e->perm, perm, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
        if (e->lists_stale) {   // list state by particle: reuse the gather's spare buffers
            uint32_t* c0 = id_o;
            T* d = reinterpret_cast<T*>(pos_o);
            T* d0 = drho_o;
            note_launch(), k_resort_list_state<T><<<grid_for(nf, 256), 256, 0, s>>>(
                perm, nf, e->cell0, c0, (const T*)e->disp, d, (const T*)e->disp0, d0);
            cudaMemcpyAsync(e->cell0, c0, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(e->disp, d, sizeof(T) * (size_t)nf, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(e->disp0, d0, sizeof(T) * (size_t)nf, cudaMemcpyDeviceToDevice, s);
        }
    }
    return check_launch("engine_rebuild_cll");
}

extern "C" int sph_engine_rebuild_cll(SphEngine* e, cudaStream_t s)
{
    int rc = validate_ws(e);
    if (rc) return rc;
    return SPH_DISPATCH(e, rebuild_impl, e, s);
}

template <class T, int D>
static int ref_sort_impl(SphEngine* e, cudaStream_t s)
{
    const int64_t n = e->n;
    if (n <= 0) return SPH_OK;
    Bump bump(e->ws, e->ws_bytes);
    SortBufs sb = sort_bufs(e, bump);
    GridP<T> g = grid_of_engine<T>(e);
    Eng<T> E = eng_of<T>(e);
    note_launch(), k_ref_keys<T, D><<<grid_for(n, 256), 256, 0, s>>>(E.pos, E.refpos, n, g, sb.k0,
                                                                     sb.v0);
    int which = 0;
    int rc = radix_sort_u32(sb.k0, sb.k1, sb.v0, sb.v1, n, e->key_bits, false, sb.hist, &which, s);
    if (rc) return rc;
    note_launch(), k_ref_assign<<<grid_for(n, 256), 256, 0, s>>>(which ? sb.v1 : sb.v0, n,
                                                                E.refpos);
    return check_launch("engine_ref_sort");
}

extern "C" int sph_engine_ref_sort(SphEngine* e, cudaStream_t s)
{
    int rc = validate_ws(e);
    if (rc) return rc;
    return SPH_DISPATCH(e, ref_sort_impl, e, s);
}

template <class T, int D>
static int stats_impl(SphEngine* e, int flags, cudaStream_t s)
{
    if (flags & 1) {   // counters: everything but the wall clamps recorded at push
        cudaMemsetAsync(&e->stats->interactions, 0, sizeof(unsigned long long), s);
        cudaMemsetAsync(&e->stats->overflow, 0, 2 * sizeof(unsigned int), s);
        cudaMemsetAsync(&e->stats->nfix, 0, sizeof(unsigned int), s);
        cudaMemsetAsync(&e->stats->ndisp, 0, sizeof(unsigned int), s);
    }
    if (flags & 2) {
        cudaMemsetAsync(e->stats, 0, 2 * sizeof(unsigned long long), s);   // vmax, amax
        cudaMemsetAsync(&e->stats->v2max_key, 0, sizeof(unsigned long long), s);
        cudaMemsetAsync(&e->stats->rho_min_key, 0xff, sizeof(unsigned long long), s);
        cudaMemsetAsync(&e->stats->nan_flags, 0, sizeof(unsigned int), s);
        if (e->n > 0) {
            Eng<T> E = eng_of<T>(e);
            note_launch(), k_stats<T, D><<<grid_for(e->n, 256, 4 * 148), 256, 0, s>>>(
                E, e->cur_v, e->cur_rp);
        }
    }
    return check_launch("engine_stats");
}

extern "C" int sph_engine_stats(SphEngine* e, int flags, cudaStream_t s)
{
    int rc = engine_validate(e);
    if (rc) return rc;
    return SPH_DISPATCH(e, stats_impl, e, flags, s);
}
