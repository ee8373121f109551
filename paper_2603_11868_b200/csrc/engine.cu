// engine.cu -- device-resident restatement of Simulation.advance
// (physics.py:416-564) on a B200-native layout.
//
// Layout in HBM (SphEngine): particles in two segments, fluid [0, nf) and
// walls [nf, n), each ordered by grid cell.  Structure of arrays with packed
// vectors so a neighbour costs three 16/8-byte loads:
//   pos  vec4 (x, y, z, m)          -- drift updates x in place
//   vel  vec4 x2 (double buffer)    -- kick2 writes the other buffer
//   rp   vec2 (rho, p) x2           -- continuity+density-update writes the
//                                      other buffer, walls follow
//   dvdt vec4, drho, id, nnb, refpos (registry position of each particle)
// Cold per-particle fields that no kernel reads per pair (rho_scratch,
// oflow, wall, Vol) are stored BY ORIGINAL ID so re-sorting never moves them.
// The fluid segment is re-sorted by cell at every CLL rebuild (the reference
// rebuilds its CLL at every advective step, physics.py:498); static walls are
// sorted once.  Neighbour sums run in ascending original id, so any physical
// order gives the reference's bits.
//
// One acoustic sub-step (physics.py:522-548) is five kernels:
//   kick+drift -> ordered lists -> continuity+density update -> wall
//   pressure -> momentum+kick
#include <cstddef>

#include "common.cuh"
#include "internal.cuh"
#include "nlist.cuh"
#include "physics.cuh"

namespace sph {

void launch_offsets_u32(const uint32_t* sorted_keys, int64_t n, int64_t ncells,
                        uint32_t* offsets, cudaStream_t s);

constexpr int kSweepThreads = 128;

template <class T>
struct Eng {
    int64_t n, nf, nw, nf_pad;
    vec4<T>* pos; vec4<T>* vel[2]; vec2<T>* rp[2]; vec4<T>* dvdt; T* drho;
    uint32_t* id; uint32_t* nnb; uint32_t* refpos;
    T* rho_scratch_id; uint32_t* oflow_id; uint32_t* wall_id; T* vol_id;
    uint32_t* offs_f; uint32_t* offs_w;
    int32_t* lists; int32_t* lcount;
    SphStepStats* stats;
};

template <class T>
static Eng<T> eng_of(const SphEngine* e)
{
    Eng<T> g;
    g.n = e->n; g.nf = e->nf; g.nw = e->n - e->nf; g.nf_pad = (e->nf + 31) / 32 * 32;
    g.pos = (vec4<T>*)e->pos;
    g.vel[0] = (vec4<T>*)e->vel[0]; g.vel[1] = (vec4<T>*)e->vel[1];
    g.rp[0] = (vec2<T>*)e->rp[0]; g.rp[1] = (vec2<T>*)e->rp[1];
    g.dvdt = (vec4<T>*)e->dvdt; g.drho = (T*)e->drho;
    g.id = e->id; g.nnb = e->nnb; g.refpos = e->refpos;
    g.rho_scratch_id = (T*)e->rho_scratch_id; g.oflow_id = e->oflow_id;
    g.wall_id = e->wall_id; g.vol_id = (T*)e->vol_id;
    g.offs_f = e->offs_f; g.offs_w = e->offs_w;
    g.lists = e->lists; g.lcount = e->lcount; g.stats = e->stats;
    return g;
}

static PhysP phys_of_engine(const SphEngine* e)
{
    PhysP P;
    P.cell_size = e->cell_size; P.cutoff = e->cutoff; P.h = e->h; P.alpha_d = e->alpha_d;
    P.c0 = e->c0; P.rho0 = e->rho0; P.alpha_visc = e->alpha_visc; P.eps_h2 = e->eps_h2;
    P.g[0] = e->g[0]; P.g[1] = e->g[1]; P.g[2] = e->dim == 3 ? e->g[2] : 0.0;
    return P;
}

template <class T>
static GridP<T> grid_of_engine(const SphEngine* e)
{
    GridP<T> g;
    for (int k = 0; k < 3; k++) {
        g.o[k] = k < e->dim ? T(e->origin[k]) : T(0);
        g.s[k] = k < e->dim ? (int)e->shape[k] : 1;
    }
    g.cs = T(e->cell_size);
    T c = T(e->cutoff);
    g.c2 = c * c;
    return g;
}

// list slot of particle i (walls start on a fresh 32-particle tile)
template <class T>
__device__ __forceinline__ int64_t slot_of(const Eng<T>& E, int64_t i)
{
    return i < E.nf ? i : E.nf_pad + (i - E.nf);
}

template <class T>
__device__ __forceinline__ void to3(const vec4<T>& v, T (&o)[3])
{
    o[0] = v.x; o[1] = v.y; o[2] = v.z;
}

__device__ __forceinline__ void add_interactions(SphStepStats* st, unsigned long long c)
{
    c = warp_sum(c);
    if (lane_id() == 0 && c) atomicAdd(&st->interactions, c);
}

// ---------------------------------------------------------------------------
// layout kernels
// ---------------------------------------------------------------------------
template <class T, int D>
__global__ void k_push_keys(const T* __restrict__ x, const uint32_t* __restrict__ wall, int64_t n,
                            GridP<T> g, int key_bits, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ oob_walls)
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
    if (lane_id() == 0 && b) atomicAdd(oob_walls, (uint32_t)__popc(b));
}

template <class T, int D>
__global__ void k_push_gather(Eng<T> E, const uint32_t* __restrict__ perm, const T* __restrict__ x,
                              const T* __restrict__ v, const T* __restrict__ rho,
                              const T* __restrict__ p, const T* __restrict__ m,
                              const T* __restrict__ vol, const T* __restrict__ drho,
                              const T* __restrict__ dvdt, const T* __restrict__ rho_scratch,
                              const uint32_t* __restrict__ id, const uint32_t* __restrict__ wall,
                              const uint32_t* __restrict__ nnb, const uint32_t* __restrict__ oflow)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    uint32_t r = perm[i];
    vec4<T> P4, V4, A4;
    P4.x = x[r * D]; P4.y = x[r * D + 1]; P4.z = D == 3 ? x[r * D + 2] : T(0); P4.w = m[r];
    V4.x = v[r * D]; V4.y = v[r * D + 1]; V4.z = D == 3 ? v[r * D + 2] : T(0); V4.w = T(0);
    A4.x = dvdt[r * D]; A4.y = dvdt[r * D + 1]; A4.z = D == 3 ? dvdt[r * D + 2] : T(0);
    A4.w = T(0);
    vec2<T> RP; RP.x = rho[r]; RP.y = p[r];
    E.pos[i] = P4;
    E.vel[0][i] = V4; E.vel[1][i] = V4;
    E.rp[0][i] = RP; E.rp[1][i] = RP;
    E.dvdt[i] = A4;
    E.drho[i] = drho[r];
    uint32_t pid = id[r];
    E.id[i] = pid;
    E.nnb[i] = nnb[r];
    E.refpos[i] = r;
    E.rho_scratch_id[pid] = rho_scratch[r];
    E.oflow_id[pid] = oflow[r];
    E.wall_id[pid] = wall[r];
    E.vol_id[pid] = vol[r];
}

template <class T, int D>
__global__ void k_pull(Eng<T> E, int cur_v, int cur_rp, T* __restrict__ x, T* __restrict__ v,
                       T* __restrict__ rho, T* __restrict__ p, T* __restrict__ m,
                       T* __restrict__ vol, T* __restrict__ drho, T* __restrict__ dvdt,
                       T* __restrict__ rho_scratch, uint32_t* __restrict__ id,
                       uint32_t* __restrict__ wall, uint32_t* __restrict__ nnb,
                       uint32_t* __restrict__ oflow)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    uint32_t r = E.refpos[i];
    uint32_t pid = E.id[i];
    vec4<T> P4 = E.pos[i], V4 = E.vel[cur_v][i], A4 = E.dvdt[i];
    vec2<T> RP = E.rp[cur_rp][i];
    x[r * D] = P4.x; x[r * D + 1] = P4.y;
    v[r * D] = V4.x; v[r * D + 1] = V4.y;
    dvdt[r * D] = A4.x; dvdt[r * D + 1] = A4.y;
    if (D == 3) { x[r * D + 2] = P4.z; v[r * D + 2] = V4.z; dvdt[r * D + 2] = A4.z; }
    m[r] = P4.w;
    rho[r] = RP.x; p[r] = RP.y;
    drho[r] = E.drho[i];
    id[r] = pid;
    nnb[r] = E.nnb[i];
    rho_scratch[r] = E.rho_scratch_id[pid];
    oflow[r] = E.oflow_id[pid];
    wall[r] = E.wall_id[pid];
    vol[r] = E.vol_id[pid];
}

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

// all-particle cell keys scattered to registry order (for sort_particles_by_cell)
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

// fused gather of every per-particle field of the fluid segment by perm
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
        // walls: the (rho, p) buffer becoming current must carry the walls'
        // latest wall-pressure values (velocity buffers agree on walls)
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

// ---------------------------------------------------------------------------
// step kernels
// ---------------------------------------------------------------------------
// physics.py:526-529 KICK(half) then DRIFT(full), fluid only
template <class T, int D>
__global__ void __launch_bounds__(256)
k_kick_drift(vec4<T>* __restrict__ pos, vec4<T>* __restrict__ vel,
             const vec4<T>* __restrict__ dvdt, int64_t nf, T half, T full)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    vec4<T> P4 = pos[i], V4 = vel[i], A4 = dvdt[i];
    V4.x = RN<T>::add(V4.x, RN<T>::mul(half, A4.x));
    V4.y = RN<T>::add(V4.y, RN<T>::mul(half, A4.y));
    P4.x = RN<T>::add(P4.x, RN<T>::mul(full, V4.x));
    P4.y = RN<T>::add(P4.y, RN<T>::mul(full, V4.y));
    if (D == 3) {
        V4.z = RN<T>::add(V4.z, RN<T>::mul(half, A4.z));
        P4.z = RN<T>::add(P4.z, RN<T>::mul(full, V4.z));
    }
    vel[i] = V4;
    pos[i] = P4;
}

// physics.py:94-119 CONTINUITY fused with :268-274 DENSITY_UPDATE(full),
// fluid only: reads rho of the current buffer, writes (rho, p) to the other.
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads)
k_cont_du(Eng<T> E, PhysP pp, int cv, int crp, T full)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.nf) return;
    int cnt = E.lcount[i];
    if (cnt < 0) {
        E.oflow_id[E.id[i]] = 1;
        atomicAdd(&E.stats->overflow, 1u);
        return;
    }
    PhysT<T> P; P.load(pp);
    const vec4<T>* __restrict__ pos = E.pos;
    const vec4<T>* __restrict__ vel = E.vel[cv];
    const vec2<T>* __restrict__ rp = E.rp[crp];
    T xi[3], vi[3];
    to3<T>(pos[i], xi);
    to3<T>(vel[i], vi);
    const T rho_i = rp[i].x;
    double acc = double(RN<T>::sub(rho_i, rho_i));
    const int32_t* lp = E.lists + ell_index(i, 0);
    for (int t = 0; t < cnt; t++) {
        const int j = lp[t * 32];
        const vec4<T> PJ = pos[j];
        T xj[3], vj[3], dx[3], r2, vx;
        to3<T>(PJ, xj);
        to3<T>(vel[j], vj);
        pair_geometry<T, D>(xi, xj, vi, vj, r2, vx, dx);
        acc = dadd(acc, continuity_term<T>(r2, vx, PJ.w, rp[j].x, P));
    }
    const T dr = RN<T>::from_d(dmul(double(rho_i), acc));
    E.drho[i] = dr;
    vec2<T> out;
    out.x = RN<T>::add(rho_i, RN<T>::mul(full, dr));
    out.y = RN<T>::mul(P.c0c0, RN<T>::sub(out.x, P.rho0));
    E.rp[crp ^ 1][i] = out;
}

// physics.py:161-194 WALL_PRESSURE over the wall segment: fluid p from
// buffer b, walls' (rho, p) written into the same buffer.  zero_drho mirrors
// the continuity body's drho = 0 for walls (physics.py:99-101) in a sub-step.
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads)
k_wall(Eng<T> E, PhysP pp, int b, int zero_drho, int count_factor)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long visits_sum = 0;
    if (t < E.nw) {
        const int64_t i = E.nf + t;
        const int64_t slot = E.nf_pad + t;
        int cnt = E.lcount[slot];
        if (cnt < 0) {
            E.oflow_id[E.id[i]] = 1;
            atomicAdd(&E.stats->overflow, 1u);
        } else {
            PhysT<T> P; P.load(pp);
            vec2<T>* __restrict__ rp = E.rp[b];
            T xi[3];
            to3<T>(E.pos[i], xi);
            const T rho_i = rp[i].x;
            double num = double(RN<T>::sub(rho_i, rho_i));
            double den = num;
            const int32_t* lp = E.lists + ell_index(slot, 0);
            for (int k = 0; k < cnt; k++) {
                const int j = lp[k * 32];
                T xj[3];
                to3<T>(E.pos[j], xj);
                double w = wall_weight<T>(pair_r2<T, D>(xi, xj), P);
                num = dadd(num, dmul(double(rp[j].y), w));
                den = dadd(den, w);
            }
            vec2<T> out;
            out.y = den > 0.0 ? RN<T>::from_d(ddiv(num, den)) : T(0);
            out.x = RN<T>::add(P.rho0, RN<T>::div(out.y, P.c0c0));
            rp[i] = out;
            E.nnb[i] = (uint32_t)cnt;
            if (zero_drho) E.drho[i] = T(0);
            visits_sum = (unsigned long long)cnt * (unsigned long long)count_factor;
        }
    }
    add_interactions(E.stats, visits_sum);
}

// physics.py:122-158 MOMENTUM (+ :546-547 KICK(half) into the other velocity
// buffer when kick != 0), fluid only; rho/p from buffer brp.
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads)
k_mom(Eng<T> E, PhysP pp, int cv, int brp, int kick, T half, int count_factor)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long csum = 0;
    if (i < E.nf) {
        int cnt = E.lcount[i];
        if (cnt < 0) {
            E.oflow_id[E.id[i]] = 1;
            atomicAdd(&E.stats->overflow, 1u);
        } else {
            PhysT<T> P; P.load(pp);
            const vec4<T>* __restrict__ pos = E.pos;
            const vec4<T>* __restrict__ vel = E.vel[cv];
            const vec2<T>* __restrict__ rp = E.rp[brp];
            T xi[3], vi[3];
            to3<T>(pos[i], xi);
            const vec4<T> VI = vel[i];
            to3<T>(VI, vi);
            const vec2<T> RPI = rp[i];
            const T rho_i = RPI.x;
            const T pi_rr = RN<T>::div(RPI.y, RN<T>::mul(rho_i, rho_i));
            T a[3] = {P.g[0], P.g[1], P.g[2]};
            const int32_t* lp = E.lists + ell_index(i, 0);
            for (int t = 0; t < cnt; t++) {
                const int j = lp[t * 32];
                const vec4<T> PJ = pos[j];
                const vec2<T> RPJ = rp[j];
                T xj[3], vj[3], dx[3], r2, vx;
                to3<T>(PJ, xj);
                to3<T>(vel[j], vj);
                pair_geometry<T, D>(xi, xj, vi, vj, r2, vx, dx);
                momentum_pair<T, D>(r2, vx, dx, rho_i, pi_rr, RPJ.x, RPJ.y, PJ.w, P, a);
            }
            vec4<T> A4;
            A4.x = a[0]; A4.y = a[1]; A4.z = D == 3 ? a[2] : T(0); A4.w = T(0);
            E.dvdt[i] = A4;
            E.nnb[i] = (uint32_t)cnt;
            if (kick) {
                vec4<T> V4 = VI;
                V4.x = RN<T>::add(V4.x, RN<T>::mul(half, A4.x));
                V4.y = RN<T>::add(V4.y, RN<T>::mul(half, A4.y));
                if (D == 3) V4.z = RN<T>::add(V4.z, RN<T>::mul(half, A4.z));
                E.vel[cv ^ 1][i] = V4;
            }
            csum = (unsigned long long)cnt * (unsigned long long)count_factor;
        }
    }
    add_interactions(E.stats, csum);
}

// physics.py:220-247 SHEPARD + :277-280 COPY_SCALAR + :268-274
// DENSITY_UPDATE(dt=0), all particles; reads buffer crp, writes crp^1.
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads)
k_shepard(Eng<T> E, PhysP pp, int crp)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    const vec2<T>* __restrict__ rp = E.rp[crp];
    const vec2<T> RPI = rp[i];
    const uint32_t pid = E.id[i];
    if (i >= E.nf) {   // walls: rho_new = rho; density update skips walls
        E.rho_scratch_id[pid] = RPI.x;
        E.rp[crp ^ 1][i] = RPI;
        return;
    }
    int cnt = E.lcount[i];
    PhysT<T> P; P.load(pp);
    T rho_new = RPI.x;
    if (cnt >= 0) {
        T xi[3];
        const vec4<T> PI = E.pos[i];
        to3<T>(PI, xi);
        const T m_i = PI.w;
        double num = double(RN<T>::mul(m_i, P.alpha_d));
        double den = double(RN<T>::mul(RN<T>::div(m_i, RPI.x), P.alpha_d));
        const int32_t* lp = E.lists + ell_index(i, 0);
        for (int t = 0; t < cnt; t++) {
            const int j = lp[t * 32];
            const vec4<T> PJ = E.pos[j];
            T xj[3];
            to3<T>(PJ, xj);
            double w = wall_weight<T>(pair_r2<T, D>(xi, xj), P);
            num = dadd(num, dmul(double(PJ.w), w));
            den = dadd(den, dmul(double(RN<T>::div(PJ.w, rp[j].x)), w));
        }
        rho_new = RN<T>::from_d(ddiv(num, den));
    }
    E.rho_scratch_id[pid] = rho_new;
    vec2<T> out;
    out.x = RN<T>::add(rho_new, RN<T>::mul(T(0), E.drho[i]));
    out.y = RN<T>::mul(P.c0c0, RN<T>::sub(out.x, P.rho0));
    E.rp[crp ^ 1][i] = out;
}

// exact max |v|, |dvdt| (physics.py:296-310 / 390-391) and the stability
// inputs min rho, max binary32 |v|^2 (physics.py:554-564), all particles
template <class T, int D>
__global__ void k_stats(Eng<T> E, int cv, int crp)
{
    double vm = 0.0, am = 0.0;
    unsigned long long rmin = ~0ull, v2k = 0ull;
    unsigned nanf = 0u;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E.n;
         i += (int64_t)gridDim.x * blockDim.x) {
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

}  // namespace sph

using namespace sph;

// ---------------------------------------------------------------------------
// ABI
// ---------------------------------------------------------------------------
static size_t engine_sort_bytes(int64_t n)
{
    size_t m = (size_t)(n > 0 ? n : 1);
    return 4 * align_up(sizeof(uint32_t) * m) + radix_hist_bytes(n);
}

extern "C" size_t sph_engine_workspace_bytes(int64_t n, int64_t ncells, int32_t f64)
{
    (void)ncells;
    size_t m = (size_t)(n > 0 ? n : 1);
    size_t es = f64 ? 8 : 4;
    // sort scratch + spare buffers for the fused fluid gather
    return engine_sort_bytes(n) + 2 * align_up(4 * es * m) + align_up(es * m) +
           3 * align_up(sizeof(uint32_t) * m) + 4096;
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

template <class T, int D>
static int push_impl(SphEngine* e, const void* x, const void* v, const void* rho, const void* p,
                     const void* m, const void* vol, const void* drho, const void* dvdt,
                     const void* rho_scratch, const uint32_t* id, const uint32_t* wall,
                     const uint32_t* nnb, const uint32_t* oflow, cudaStream_t s)
{
    Bump bump(e->ws, e->ws_bytes);
    SortBufs sb = sort_bufs(e, bump);
    if (!sb.hist) return SPH_ERR_WORKSPACE;
    GridP<T> g = grid_of_engine<T>(e);
    Eng<T> E = eng_of<T>(e);
    const int64_t n = e->n;
    cudaMemsetAsync(e->stats, 0, sizeof(SphStepStats), s);
    if (n > 0) {
        note_launch(), k_push_keys<T, D><<<grid_for(n, 256), 256, 0, s>>>((const T*)x, wall, n, g, e->key_bits,
                                                             sb.k0, &e->stats->oob_walls);
        int which = 0;
        int rc = radix_sort_u32(sb.k0, sb.k1, sb.v0, sb.v1, n, e->key_bits + 1, true, sb.hist,
                                &which, s);
        if (rc) return rc;
        const uint32_t* sk = which ? sb.k1 : sb.k0;
        const uint32_t* perm = which ? sb.v1 : sb.v0;
        note_launch(), k_push_gather<T, D><<<grid_for(n, 256), 256, 0, s>>>(
            E, perm, (const T*)x, (const T*)v, (const T*)rho, (const T*)p, (const T*)m,
            (const T*)vol, (const T*)drho, (const T*)dvdt, (const T*)rho_scratch, id, wall, nnb,
            oflow);
        // fluid offsets over sk[0, nf), wall offsets over sk[nf, n) (flag bit set)
        note_launch(), k_seg_offsets<<<grid_for(e->ncells + 1, 256), 256, 0, s>>>(sk, e->nf, e->ncells, 0u,
                                                                  e->offs_f);
        note_launch(), k_seg_offsets<<<grid_for(e->ncells + 1, 256), 256, 0, s>>>(
            sk + e->nf, n - e->nf, e->ncells, 1u << e->key_bits, e->offs_w);
    } else {
        cudaMemsetAsync(e->offs_f, 0, sizeof(uint32_t) * (size_t)(e->ncells + 1), s);
        cudaMemsetAsync(e->offs_w, 0, sizeof(uint32_t) * (size_t)(e->ncells + 1), s);
    }
    e->cur_v = 0;
    e->cur_rp = 0;
    return check_launch("engine_push");
}

#define DISPATCH(e, FN, ...)                                                                 \
    ((e)->f64 ? ((e)->dim == 3 ? FN<double, 3>(__VA_ARGS__) : FN<double, 2>(__VA_ARGS__))    \
              : ((e)->dim == 3 ? FN<float, 3>(__VA_ARGS__) : FN<float, 2>(__VA_ARGS__)))

static int validate(const SphEngine* e)
{
    if (!e || (e->dim != 2 && e->dim != 3) || e->n < 0 || e->nf < 0 || e->nf > e->n)
        return SPH_ERR_INVALID;
    if (e->ncells + 1 >= (int64_t)INT32_MAX || e->key_bits > 30 || e->n >= (int64_t)INT32_MAX) {
        set_error("engine: grid or particle count too large for 32-bit keys");
        return SPH_ERR_UNSUPPORTED;
    }
    if (e->ws_bytes < sph_engine_workspace_bytes(e->n, e->ncells, e->f64)) {
        set_error("engine: workspace too small");
        return SPH_ERR_WORKSPACE;
    }
    return SPH_OK;
}

extern "C" int sph_engine_push(SphEngine* e, const void* x, const void* v, const void* rho,
                               const void* p, const void* m, const void* vol, const void* drho,
                               const void* dvdt, const void* rho_scratch, const uint32_t* id,
                               const uint32_t* wall, const uint32_t* nnb, const uint32_t* oflow,
                               cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, push_impl, e, x, v, rho, p, m, vol, drho, dvdt, rho_scratch, id, wall,
                    nnb, oflow, s);
}

template <class T, int D>
static int pull_impl(const SphEngine* e, void* x, void* v, void* rho, void* p, void* m, void* vol,
                     void* drho, void* dvdt, void* rho_scratch, uint32_t* id, uint32_t* wall,
                     uint32_t* nnb, uint32_t* oflow, cudaStream_t s)
{
    if (e->n <= 0) return SPH_OK;
    Eng<T> E = eng_of<T>(e);
    note_launch(), k_pull<T, D><<<grid_for(e->n, 256), 256, 0, s>>>(
        E, e->cur_v, e->cur_rp, (T*)x, (T*)v, (T*)rho, (T*)p, (T*)m, (T*)vol, (T*)drho, (T*)dvdt,
        (T*)rho_scratch, id, wall, nnb, oflow);
    return check_launch("engine_pull");
}

extern "C" int sph_engine_pull(const SphEngine* e, void* x, void* v, void* rho, void* p, void* m,
                               void* vol, void* drho, void* dvdt, void* rho_scratch,
                               uint32_t* id, uint32_t* wall, uint32_t* nnb, uint32_t* oflow,
                               cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, pull_impl, e, x, v, rho, p, m, vol, drho, dvdt, rho_scratch, id, wall, nnb,
                    oflow, s);
}

template <class T, int D>
static int rebuild_impl(SphEngine* e, cudaStream_t s)
{
    const int64_t nf = e->nf;
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
    note_launch(), k_fluid_keys<T, D><<<grid_for(nf, 256), 256, 0, s>>>(E.pos, nf, g, sb.k0, &e->stats->oob);
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
    cudaMemcpyAsync(e->pos, pos_o, 4 * es * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->dvdt, dvdt_o, 4 * es * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->drho, drho_o, es * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->id, id_o, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->refpos, ref_o, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(e->nnb, nnb_o, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, s);
    // velocity buffers agree on the (never moving) walls
    e->cur_v = cv ^ 1;
    e->cur_rp = crp ^ 1;
    note_launch(), k_seg_offsets<<<grid_for(e->ncells + 1, 256), 256, 0, s>>>(sk, nf, e->ncells, 0u, e->offs_f);
    return check_launch("engine_rebuild_cll");
}

extern "C" int sph_engine_rebuild_cll(SphEngine* e, cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, rebuild_impl, e, s);
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
    note_launch(), k_ref_keys<T, D><<<grid_for(n, 256), 256, 0, s>>>(E.pos, E.refpos, n, g, sb.k0, sb.v0);
    int which = 0;
    int rc = radix_sort_u32(sb.k0, sb.k1, sb.v0, sb.v1, n, e->key_bits, false, sb.hist, &which, s);
    if (rc) return rc;
    note_launch(), k_ref_assign<<<grid_for(n, 256), 256, 0, s>>>(which ? sb.v1 : sb.v0, n, E.refpos);
    return check_launch("engine_ref_sort");
}

extern "C" int sph_engine_ref_sort(SphEngine* e, cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, ref_sort_impl, e, s);
}

template <class T, int D>
static int build_all_lists(const SphEngine* e, cudaStream_t s)
{
    GridP<T> g = grid_of_engine<T>(e);
    EngAcc<T> acc;
    acc.pos = (const vec4<T>*)e->pos;
    acc.id = e->id;
    acc.offs_f = e->offs_f;
    acc.offs_w = e->offs_w;
    acc.nf = e->nf;
    acc.store_walls = true;
    launch_build_lists<T, D>(acc, g, 0, e->nf, 0, e->lists, e->lcount, s);
    acc.store_walls = false;
    const int64_t nf_pad = (e->nf + 31) / 32 * 32;
    launch_build_lists<T, D>(acc, g, e->nf, e->n - e->nf, nf_pad, e->lists, e->lcount, s);
    return check_launch("engine_build_lists");
}

template <class T, int D>
static int initialize_impl(SphEngine* e, cudaStream_t s)
{
    int rc = build_all_lists<T, D>(e, s);
    if (rc) return rc;
    Eng<T> E = eng_of<T>(e);
    PhysP P = phys_of_engine(e);
    const int64_t nw = e->n - e->nf;
    if (nw > 0)
        note_launch(), k_wall<T, D><<<grid_for(nw, kSweepThreads), kSweepThreads, 0, s>>>(E, P, e->cur_rp, 0, 1);
    if (e->nf > 0)
        note_launch(), k_mom<T, D><<<grid_for(e->nf, kSweepThreads), kSweepThreads, 0, s>>>(
            E, P, e->cur_v, e->cur_rp, 0, T(0), 1);
    // momentum writes dvdt = 0 for walls (physics.py:128-131)
    if (nw > 0)
        cudaMemsetAsync((char*)e->dvdt + sizeof(vec4<T>) * (size_t)e->nf, 0,
                        sizeof(vec4<T>) * (size_t)nw, s);
    return check_launch("engine_initialize");
}

extern "C" int sph_engine_initialize(SphEngine* e, cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, initialize_impl, e, s);
}

template <class T, int D>
static int shepard_impl(SphEngine* e, cudaStream_t s)
{
    if (e->n <= 0) return SPH_OK;
    int rc = build_all_lists<T, D>(e, s);
    if (rc) return rc;
    Eng<T> E = eng_of<T>(e);
    PhysP P = phys_of_engine(e);
    note_launch(), k_shepard<T, D><<<grid_for(e->n, kSweepThreads), kSweepThreads, 0, s>>>(E, P, e->cur_rp);
    e->cur_rp ^= 1;
    return check_launch("engine_shepard");
}

extern "C" int sph_engine_shepard(SphEngine* e, cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, shepard_impl, e, s);
}

// ev (optional, 6 events): boundaries of kick+drift | lists | continuity+DU
// | wall pressure | momentum+kick, for bench.py's per-kernel timing
template <class T, int D>
static int substep_impl(SphEngine* e, double half_d, double full_d, cudaEvent_t* ev,
                        cudaStream_t s)
{
    const T half = T(half_d), full = T(full_d);
    Eng<T> E = eng_of<T>(e);
    PhysP P = phys_of_engine(e);
    const int cv = e->cur_v, crp = e->cur_rp;
    const int64_t nf = e->nf, nw = e->n - e->nf;
    if (ev) cudaEventRecord(ev[0], s);
    if (nf > 0)
        note_launch(), k_kick_drift<T, D><<<grid_for(nf, 256), 256, 0, s>>>(
            E.pos, E.vel[cv], E.dvdt, nf, half, full);
    if (ev) cudaEventRecord(ev[1], s);
    int rc = build_all_lists<T, D>(e, s);
    if (rc) return rc;
    if (ev) cudaEventRecord(ev[2], s);
    if (nf > 0)
        note_launch(), k_cont_du<T, D><<<grid_for(nf, kSweepThreads), kSweepThreads, 0, s>>>(
            E, P, cv, crp, full);
    else if (nw > 0)   // no fluid: the other rp buffer must still carry walls
        cudaMemcpyAsync(E.rp[crp ^ 1], E.rp[crp], sizeof(vec2<T>) * (size_t)e->n,
                        cudaMemcpyDeviceToDevice, s);
    if (ev) cudaEventRecord(ev[3], s);
    if (nw > 0)
        note_launch(), k_wall<T, D><<<grid_for(nw, kSweepThreads), kSweepThreads, 0, s>>>(
            E, P, crp ^ 1, 1, 1);
    if (ev) cudaEventRecord(ev[4], s);
    if (nf > 0)
        note_launch(), k_mom<T, D><<<grid_for(nf, kSweepThreads), kSweepThreads, 0, s>>>(
            E, P, cv, crp ^ 1, 1, half, 2);
    else
        cudaMemcpyAsync(E.vel[cv ^ 1], E.vel[cv], sizeof(vec4<T>) * (size_t)e->n,
                        cudaMemcpyDeviceToDevice, s);
    if (ev) cudaEventRecord(ev[5], s);
    e->cur_v = cv ^ 1;
    e->cur_rp = crp ^ 1;
    return check_launch("engine_substep");
}

extern "C" int sph_engine_substep(SphEngine* e, double half_dt, double full_dt, cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, substep_impl, e, half_dt, full_dt, (cudaEvent_t*)nullptr, s);
}

extern "C" int sph_engine_substep_timed(SphEngine* e, double half_dt, double full_dt,
                                        float* ms_out, cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    cudaEvent_t ev[6];
    for (int k = 0; k < 6; k++) cudaEventCreate(&ev[k]);
    rc = DISPATCH(e, substep_impl, e, half_dt, full_dt, ev, s);
    if (rc == SPH_OK) {
        cudaEventSynchronize(ev[5]);
        for (int k = 0; k < 5; k++) cudaEventElapsedTime(&ms_out[k], ev[k], ev[k + 1]);
    }
    for (int k = 0; k < 6; k++) cudaEventDestroy(ev[k]);
    return rc ? rc : check_launch("engine_substep_timed");
}

template <class T, int D>
static int stats_impl(SphEngine* e, int flags, cudaStream_t s)
{
    if (flags & 1) {   // counters: everything but the wall clamps recorded at push
        cudaMemsetAsync(&e->stats->interactions, 0, sizeof(unsigned long long), s);
        cudaMemsetAsync(&e->stats->overflow, 0, 2 * sizeof(unsigned int), s);
        cudaMemsetAsync(&e->stats->nfix, 0, sizeof(unsigned int), s);
    }
    if (flags & 2) {
        cudaMemsetAsync(e->stats, 0, 2 * sizeof(unsigned long long), s);   // vmax, amax
        cudaMemsetAsync(&e->stats->v2max_key, 0, sizeof(unsigned long long), s);
        cudaMemsetAsync(&e->stats->rho_min_key, 0xff, sizeof(unsigned long long), s);
        cudaMemsetAsync(&e->stats->nan_flags, 0, sizeof(unsigned int), s);
        if (e->n > 0) {
            Eng<T> E = eng_of<T>(e);
            note_launch(), k_stats<T, D><<<grid_for(e->n, 256, 4 * 148), 256, 0, s>>>(E, e->cur_v, e->cur_rp);
        }
    }
    return check_launch("engine_stats");
}

extern "C" int sph_engine_stats(SphEngine* e, int flags, cudaStream_t s)
{
    int rc = validate(e);
    if (rc) return rc;
    return DISPATCH(e, stats_impl, e, flags, s);
}
