// engine.cuh -- shared view of the device-resident engine state (SphEngine).
//
// Layout in HBM: particles in two segments, fluid [0, nf) and walls [nf, n),
// each ordered by grid cell.  Structure of arrays with packed vectors so a
// neighbour costs three 16/8-byte loads:
//   pos  vec4 (x, y, z, m)          -- drift updates x in place
//   vel  vec4 x2 (double buffer)    -- kick2 writes the other buffer
//   rp   vec2 (rho, p) x2           -- continuity+density update writes the
//                                      other buffer, walls follow
//   rq   vec2 (rho, p/rho^2)        -- per-neighbour momentum operands, written
//                                      with rp by the density update / walls
//   vel.w = m/rho                   -- per-neighbour continuity operand, set by
//                                      kick+drift before every continuity sweep
//   dvdt vec4, drho, id, nnb, refpos (registry position of each particle)
// Cold per-particle fields no kernel reads per pair (rho_scratch, oflow,
// wall, Vol) are stored BY ORIGINAL ID, so re-sorting never moves them.
#pragma once

#include "common.cuh"
#include "internal.cuh"
#include "nlist.cuh"
#include "physics.cuh"

namespace sph {

#ifndef SPH_SWEEP_THREADS
#define SPH_SWEEP_THREADS 128
#endif
constexpr int kSweepThreads = SPH_SWEEP_THREADS;
constexpr uint32_t kInvalidCell = 0xffffffffu;   // list is not a valid skin list

template <class T>
struct Eng {
    int64_t n, nf, nw, nf_pad;
    int64_t idr;         // ids are below idr (the by-id arrays' length)
    vec4<T>* pos;        // the current position buffer
    vec4<T>* pos_next;   // the other one (fused kick+drift writes it)
    vec4<T>* vel[2]; vec2<T>* rp[2]; vec2<T>* rq; vec4<T>* dvdt; T* drho;
    uint32_t* id; uint32_t* nnb; uint32_t* refpos;
    T* rho_scratch_id; uint32_t* oflow_id; uint32_t* wall_id; T* vol_id;
    const uint8_t* owned_id;
    uint32_t* offs_f; uint32_t* offs_w;
    int32_t* lists; int32_t* lcount; int32_t* acount; int32_t* nww; int32_t* elist;
    uint32_t* cellmax; const uint32_t* blockmax; const uint32_t* key_sorted;
    uint32_t* cell0; T* disp; T* disp0; uint32_t* queue; uint32_t* qcount;
    SphStepStats* stats;
};

template <class T>
inline Eng<T> eng_of(const SphEngine* e)
{
    Eng<T> g;
    g.n = e->n; g.nf = e->nf; g.nw = e->n - e->nf; g.nf_pad = (e->nf + 31) / 32 * 32;
    g.idr = e->id_range > 0 ? e->id_range : e->n;
    g.pos = (vec4<T>*)e->pos[e->cur_pos];
    g.pos_next = (vec4<T>*)e->pos[e->cur_pos ^ 1];
    g.vel[0] = (vec4<T>*)e->vel[0]; g.vel[1] = (vec4<T>*)e->vel[1];
    g.rp[0] = (vec2<T>*)e->rp[0]; g.rp[1] = (vec2<T>*)e->rp[1];
    g.rq = (vec2<T>*)e->rq;
    g.dvdt = (vec4<T>*)e->dvdt; g.drho = (T*)e->drho;
    g.id = e->id; g.nnb = e->nnb; g.refpos = e->refpos;
    g.rho_scratch_id = (T*)e->rho_scratch_id; g.oflow_id = e->oflow_id;
    g.wall_id = e->wall_id; g.vol_id = (T*)e->vol_id;
    g.owned_id = e->owned_id;
    g.offs_f = e->offs_f; g.offs_w = e->offs_w;
    g.lists = e->lists; g.lcount = e->lcount; g.acount = e->acount; g.nww = e->nww;
    g.elist = e->elist;
    const bool local = sizeof(T) == 4 && e->cellmax && e->blockmax && e->key_sorted;
    g.cellmax = local ? e->cellmax : nullptr;
    g.blockmax = local ? e->blockmax : nullptr;
    g.key_sorted = e->key_sorted;
    g.cell0 = e->cell0; g.disp = (T*)e->disp; g.disp0 = (T*)e->disp0;
    g.queue = e->queue;
    g.qcount = e->qcount; g.stats = e->stats;
    return g;
}

inline PhysP phys_of_engine(const SphEngine* e)
{
    PhysP P;
    P.cell_size = e->cell_size; P.cutoff = e->cutoff; P.h = e->h; P.alpha_d = e->alpha_d;
    P.c0 = e->c0; P.rho0 = e->rho0; P.alpha_visc = e->alpha_visc; P.eps_h2 = e->eps_h2;
    P.g[0] = e->g[0]; P.g[1] = e->g[1]; P.g[2] = e->dim == 3 ? e->g[2] : 0.0;
    return P;
}

template <class T>
inline GridP<T> grid_of_engine(const SphEngine* e)
{
    GridP<T> g;
    for (int k = 0; k < 3; k++) {
        g.o[k] = k < e->dim ? T(e->origin[k]) : T(0);
        g.s[k] = k < e->dim ? (int)e->shape[k] : 1;
    }
    g.cs = T(e->cell_size);
    const T c = T(e->cutoff);
    g.c2 = c * c;   // binary32 product in the f32 run (neighborhood.py:185)
    return g;
}

template <class T>
inline EngAcc<T> acc_of_engine(const SphEngine* e)
{
    EngAcc<T> acc;
    acc.pos = (const vec4<T>*)e->pos[e->cur_pos];
    acc.id = e->id;
    acc.offs_f = e->offs_f;
    acc.offs_w = e->offs_w;
    acc.nf = e->nf;
#if SPH_PERIODIC
    acc.segs = e->n > e->nf ? 2 : 1;
#endif
    return acc;
}

// the displacement bound a list's validity test uses: the largest path
// length in the list cell's 3^d block (local mode) or over all particles
template <class T>
__device__ __forceinline__ T dmax_for(const Eng<T>& E, uint32_t cell, T global)
{
    if (sizeof(T) == 4 && E.blockmax && cell != 0xffffffffu)
        return T(__uint_as_float(E.blockmax[cell]));
    return global;
}

// record a fluid particle's path length in its CLL cell's maximum
template <class T>
__device__ __forceinline__ void note_disp(const Eng<T>& E, int64_t i, T d)
{
    if (sizeof(T) == 4 && E.cellmax && i < E.nf)
        atomicMax(&E.cellmax[E.key_sorted[i]], __float_as_uint(float(d)));
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

// multi-rank slabs: halo ghosts are neither integrated nor counted
template <class T>
__device__ __forceinline__ bool is_owned(const Eng<T>& E, int64_t i)
{
    return !E.owned_id || E.owned_id[E.id[i]];
}

__device__ __forceinline__ void add_interactions(SphStepStats* st, unsigned long long c)
{
    c = warp_sum(c);
    if (lane_id() == 0 && c) atomicAdd(&st->interactions, c);
}

inline int engine_validate(const SphEngine* e)
{
    if (!e || (e->dim != 2 && e->dim != 3) || e->n < 0 || e->nf < 0 || e->nf > e->n)
        return SPH_ERR_INVALID;
    if (e->ncells + 1 >= (int64_t)INT32_MAX || e->key_bits > 30 || e->n >= (int64_t)INT32_MAX) {
        set_error("engine: grid or particle count too large for 32-bit keys");
        return SPH_ERR_UNSUPPORTED;
    }
    bool periodic = false, last_periodic = false;
    for (int k = 0; k < e->dim; k++) {
        if (!(e->period[k] >= 0.0)) return SPH_ERR_INVALID;
        if (e->period[k] > 0.0) {
            periodic = true;
            last_periodic = k == e->dim - 1;
            // the cells must tile the period: the last one reaches the period
            // end and is at least a cutoff wide (wrap-around blocks are exact)
            const double L = e->period[k], s = (double)e->shape[k];
            if (e->shape[k] < 3 || L > s * e->cell_size * (1.0 + 1e-12) ||
                L < (s - 1.0) * e->cell_size + e->cutoff) {
                set_error("engine: a periodic axis needs >= 3 cells tiling the period");
                return SPH_ERR_INVALID;
            }
        }
    }
#if SPH_PERIODIC
    // wall-free periodic boxes only (the tested configuration; a warp also
    // enumerates at most 18 key runs per block, engine.cu k_skin_tile)
    (void)last_periodic;
    if (periodic && e->n > e->nf) {
        set_error("engine: periodic boxes are supported for wall-free cases");
        return SPH_ERR_UNSUPPORTED;
    }
#else
    (void)last_periodic;
    if (periodic) {
        set_error("engine: periodic boxes need libsphb200_periodic.so");
        return SPH_ERR_UNSUPPORTED;
    }
#endif
    return SPH_OK;
}

// validation + the periodic box of this translation unit's kernels, set on
// the caller's stream (engine.cu entry points)
inline int engine_begin(const SphEngine* e, cudaStream_t s)
{
    int rc = engine_validate(e);
    if (rc) return rc;
#if SPH_PERIODIC
    PerBox b;
    for (int k = 0; k < 3; k++) {
        const bool p = k < e->dim && e->period[k] > 0.0;
        // run-precision values: lo = origin, hi = RN(lo + L), L/2 exact
        const float lf = p ? (float)e->period[k] : 0.f, of = p ? (float)e->origin[k] : 0.f;
        const double ld = p ? e->period[k] : 0.0, od = p ? e->origin[k] : 0.0;
        volatile float hf = of + lf;
        volatile double hd = od + ld;
        b.Lf[k] = lf; b.hLf[k] = lf * 0.5f; b.lof[k] = of; b.hif[k] = hf;
        b.Ld[k] = ld; b.hLd[k] = ld * 0.5; b.lod[k] = od; b.hid[k] = hd;
    }
    if (cudaMemcpyToSymbolAsync(c_box, &b, sizeof(b), 0, cudaMemcpyHostToDevice, s) !=
        cudaSuccess)
        return check_launch("engine periodic box");
#else
    (void)s;
#endif
    return SPH_OK;
}

#define SPH_DISPATCH(e, FN, ...)                                                              \
    ((e)->f64 ? ((e)->dim == 3 ? FN<double, 3>(__VA_ARGS__) : FN<double, 2>(__VA_ARGS__))     \
              : ((e)->dim == 3 ? FN<float, 3>(__VA_ARGS__) : FN<float, 2>(__VA_ARGS__)))

}  // namespace sph
