// engine.cu -- device-resident restatement of Simulation.advance
// (physics.py:489-552) on the B200 layout of engine.cuh.
//
// Neighbour lists are Verlet skin lists built once per advective step
// (after the CLL rebuild): for each particle, the ascending-id list of the
// CLL-block candidates within cutoff + skin of its position.  Within the
// step the reference recomputes neighbours at every sweep from CURRENT
// positions with the stale CLL (neighborhood.py:188-213); the engine gets the
// identical ordered set by filtering the skin list exactly (0 < r2 < c^2 in
// binary32, the reference's test) into an exact list per sub-step, which is
// exact as long as (a) the particle is still in the cell its list was built
// for and (b) its displacement bound plus the largest displacement bound of
// any particle stays below the skin (triangle inequality; bounds are
// accumulated with upward rounding).  Particles failing (a) or (b) get an
// exact list rebuilt for that sub-step (k_fix_build), so the result never
// depends on the skin choice -- only the speed does.
//
// Per advective step: k_skin_warp (2D: a warp per cell) / k_skin_tile (a
// block per cell) / k_skin_big (oversized blocks) build the skin lists.
// One acoustic sub-step (physics.py:522-548):
//   k_kick_drift  KICK + DRIFT, displacement bounds, cell-change marks
//                 (first sub-step only; later ones come fused in k_mom)
//   k_mark        queue particles whose skin list is no longer valid
//   k_fix_build   exact ordered lists for the queued particles
//   k_cont_du     skin-list filter + CONTINUITY + DENSITY_UPDATE (fluid);
//                 writes the exact lists the momentum sweep reads
//   k_wall        skin-list filter + WALL_PRESSURE (walls)
//   k_mom         MOMENTUM + KICK (fluid), + the next sub-step's KICK + DRIFT
//
// Tuning knobs below were chosen by measurement.
#include <type_traits>
#include "engine.cuh"

#ifndef SPH_SWEEP_MINB
#define SPH_SWEEP_MINB 12    // min resident blocks of the sweeps (register cap)
#endif
#ifndef SPH_CONT_MINB         // fused skin filter (3D: 8 measured -14% vs 10)
#define SPH_CONT_MINB (D == 3 ? 8 : 12)
#endif
#ifndef SPH_CONT_EXACT_MINB   // exact-list walk (split filtering)
#if SPH_PERIODIC
#define SPH_CONT_EXACT_MINB (D == 3 ? 8 : 12)
#else
#define SPH_CONT_EXACT_MINB (D == 3 ? 10 : 12)
#endif
#endif
#ifndef SPH_MARK_FUSED        // sub-step list check + refresh in one queue-free kernel
#define SPH_MARK_FUSED 1
#endif
#ifndef SPH_MOM_MINB          // the momentum sweep holds more live state
#define SPH_MOM_MINB (D == 2 ? 9 : 8)   // (2D 9: -1%; 3D 9/10: no gain, spills)
#endif
#ifndef SPH_MASK_MINB
#define SPH_MASK_MINB 12     // k_mask (split filtering): quad prefetch + staged stores
#endif
#ifndef SPH_FIX_MINB
#define SPH_FIX_MINB 4          // k_fix_build blocks per SM (register cap)
#endif
#ifndef SPH_SKIN_SORT_CT
#define SPH_SKIN_SORT_CT 1     // block bitonic: straight-line chunk merge stages
#endif
#ifndef SPH_SKIN_FLUID_PASS
#define SPH_SKIN_FLUID_PASS 1   // k_skin_tile: fluid-pair passes without wall tests
#endif
#ifndef SPH_SKIN_PRUNE          // drop block candidates beyond the cell's skin reach (against
#define SPH_SKIN_PRUNE 1        // the cell box: 3D 4M -4%, Taylor-Green +2%; against the
#endif                          // particles' box, SPH_SKIN_BBOX: -14% / -8%)
#ifndef SPH_SKIN_FMA
#define SPH_SKIN_FMA 1          // skin test r2 with FMAs (not rounded like the reference)
#endif
#ifndef SPH_SKIN_SORT_ASC
#define SPH_SKIN_SORT_ASC 1     // skin tile: all-ascending bitonic that never touches the padding
#endif
#ifndef SPH_SKIN_SORT_K4
#define SPH_SKIN_SORT_K4 1      // ... with 4 keys per lane (128-key register chunks)
#endif
#ifndef SPH_LIST_FRESH
#define SPH_LIST_FRESH 1        // list builds on a fresh CLL take each particle's cell from it
#endif
#ifndef SPH_SKIN_BLOCKED
#define SPH_SKIN_BLOCKED 1      // skin tile: each thread loads a contiguous candidate range
#endif
#ifndef SPH_SKIN_DYN
#define SPH_SKIN_DYN 1          // skin tile: cells handed out by an atomic counter
#endif
#ifndef SPH_SKIN_BBOX
#define SPH_SKIN_BBOX 1         // skin tile: prune against the cell's particles' bounding box
#endif
#ifndef SPH_SKIN_STAGE
#define SPH_SKIN_STAGE 1        // k_skin_tile: survivors staged in shared memory, int4 stores
#endif
#ifndef SPH_SKIN_WALL_SKIP
#define SPH_SKIN_WALL_SKIP 1    // skip wall-only blocks once the wall-wall counts are known
#endif
#ifndef SPH_SKIN_THREADS_PER_SM
#define SPH_SKIN_THREADS_PER_SM 1024   // skin-list build occupancy (register cap)
#endif
#ifndef SPH_SKINW_MINB
#define SPH_SKINW_MINB 4     // warp-per-cell skin build: blocks per SM (register cap)
#endif
#ifndef SPH_CONT_FILTER_QUADS      // continuity: visit accepted entries per list quad
#define SPH_CONT_FILTER_QUADS (D == 3)   // (measured: 3D -4.5%, 2D +23%)
#endif
#ifndef SPH_ELIST_SCALAR     // continuity's exact-list stores: 4-byte stores per entry
#define SPH_ELIST_SCALAR (D == 3)   // (1) or int4 quads assembled in registers (0); 3D -4% cont, 2D -3% PU/s
#endif
#ifndef SPH_LIST_CS          // list streams (skin / exact lists, ~1 GB each per
#define SPH_LIST_CS 0        // 3D 4M sub-step) with evict-first hints (measured: 3D -1%, 2D +11%: off)
#endif
#ifndef SPH_MOM_ILP
#define SPH_MOM_ILP 1        // momentum: two pairs per basic block (1: in 2D, 2: always)
#endif

namespace sph {

// neighbour-list quads: streamed once per sweep and larger than L2, so they
// are loaded / stored evict-first (the gathered particle data keeps L2)
__device__ __forceinline__ int4 ld_list(const int4* p)
{
#if SPH_LIST_CS
    return __ldcs(p);
#else
    return *p;
#endif
}
__device__ __forceinline__ void st_list(int4* p, int4 v)
{
#if SPH_LIST_CS
    __stcs(p, v);
#else
    *p = v;
#endif
}

// Software-pipelined walk over the exact list of slot (ascending original
// id): the list entry two pairs ahead and the neighbour data one pair ahead
// are in flight while the current pair is computed.
template <class T, class Load, class Body>
__device__ __forceinline__ void sweep_list(const Eng<T>& E, int64_t slot, int cnt, Load load,
                                           Body body)
{
    if (cnt <= 0) return;
    // quad-ELL: 4 entries per int4; the next quad is requested before the
    // current one is processed, so the list stream never stalls a pair
    const int4* __restrict__ q4 = reinterpret_cast<const int4*>(E.elist + ell_base(slot));
    int4 qn = ld_list(q4);
    for (int t0 = 0; t0 < cnt; t0 += 4) {
        const int4 q = qn;
        if (t0 + 4 < cnt) qn = ld_list(q4 + ((t0 >> 2) + 1) * 32);
        body(t0, load(q.x));
        if (t0 + 1 < cnt) body(t0 + 1, load(q.y));
        if (t0 + 2 < cnt) body(t0 + 2, load(q.z));
        if (t0 + 3 < cnt) body(t0 + 3, load(q.w));
    }
}

template <class T> struct NbrPVR { vec4<T> p; vec4<T> v; vec2<T> rp; };
template <class T> struct NbrPV { vec4<T> p; vec4<T> v; };

// momentum operands of a particle: (rho, p / rho^2) (physics.py:147-148)
template <class T>
__device__ __forceinline__ vec2<T> rq_of(const vec2<T>& rp)
{
    vec2<T> q;
    q.x = rp.x;
    q.y = RN<T>::div(rp.y, RN<T>::mul(rp.x, rp.x));
    return q;
}

template <class T>
__global__ void __launch_bounds__(256) k_rq_fill(Eng<T> E, int crp, int64_t count)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) E.rq[i] = rq_of<T>(E.rp[crp][i]);
}
template <class T> struct NbrPR { vec4<T> p; vec2<T> rp; };

// Exact filter of slot's skin list fused into a sweep: per chunk of CH (32,
// 64 or 128) entries, the reference's acceptance test (0 < r2 < c^2,
// binary32) runs first with the list quads + positions in flight (phase 1,
// bits in registers), then the accepted neighbours are visited in list (=
// ascending id) order (phase 2).  A warp runs phase 2 for the largest
// accepted count among its lanes, so longer chunks waste fewer bodies on
// uneven lanes (per-chunk maxima average out).
#ifndef SPH_WALK_CHUNK
#define SPH_WALK_CHUNK 32
#endif
template <class T, int D, class Load, class Body>
__device__ __forceinline__ void filter_walk(const Eng<T>& E, int64_t slot, const T (&xi)[3],
                                            T c2, int nl, Load load, Body body)
{
    constexpr int CH = SPH_WALK_CHUNK, NM = CH / 32;
    const int32_t* __restrict__ lp = E.lists + ell_base(slot);
    const int4* __restrict__ q4 = reinterpret_cast<const int4*>(lp);
    for (int w0 = 0; w0 < nl; w0 += CH) {
        const int ne = min(CH, nl - w0);
        uint32_t m[NM];
#pragma unroll
        for (int h = 0; h < NM; h++) m[h] = 0;
        for (int u0 = 0; u0 < ne; u0 += 4) {
            const int4 q = ld_list(q4 + ((w0 + u0) >> 2) * 32);
            int jj[4] = {q.x, u0 + 1 < ne ? q.y : -1, u0 + 2 < ne ? q.z : -1,
                         u0 + 3 < ne ? q.w : -1};
            vec4<T> pj[4];
#pragma unroll
            for (int k = 0; k < 4; k++) pj[k] = E.pos[jj[k] >= 0 ? jj[k] : 0];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                T xj[3];
                to3<T>(pj[k], xj);
                const T r2 = accept_r2<T, D>(xi, xj);
                const int u = u0 + k;
                if (jj[k] >= 0 && (r2 < c2) && (r2 > T(0))) {
                    if (NM == 1) m[0] |= 1u << u;
                    else
#pragma unroll
                        for (int h = 0; h < NM; h++)
                            if ((u >> 5) == h) m[h] |= 1u << (u & 31);
                }
            }
        }
#pragma unroll
        for (int h = 0; h < NM; h++) {
            uint32_t mh = m[h];
            while (mh) {
                const int u = __ffs(mh) - 1;
                mh &= mh - 1;
                const int j = lp[ell_off(w0 + 32 * h + u)];
                body(j, load(j));
            }
        }
    }
}

// Exact filter of slot's skin list quad by quad: the 4 entries' positions
// are gathered together, tested (0 < r2 < c^2, binary32), and each accepted
// neighbour is visited right away with the position already in registers
// (body(j, pos_j)); visits stay in list (= ascending id) order.
template <class T, int D, class Body>
__device__ __forceinline__ void filter_quads(const Eng<T>& E, int64_t slot, const T (&xi)[3], T c2,
                                             int nl, Body body)
{
    if (nl <= 0) return;
    const int4* __restrict__ q4 = reinterpret_cast<const int4*>(E.lists + ell_base(slot));
    int4 qn = ld_list(q4);
    for (int u0 = 0; u0 < nl; u0 += 4) {
        const int4 q = qn;
        if (u0 + 4 < nl) qn = ld_list(q4 + ((u0 >> 2) + 1) * 32);
        const int jj[4] = {q.x, u0 + 1 < nl ? q.y : -1, u0 + 2 < nl ? q.z : -1,
                           u0 + 3 < nl ? q.w : -1};
        vec4<T> pj[4];
#pragma unroll
        for (int k = 0; k < 4; k++) pj[k] = E.pos[jj[k] >= 0 ? jj[k] : 0];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            T xj[3];
            to3<T>(pj[k], xj);
            const T r2 = accept_r2<T, D>(xi, xj);
            if (jj[k] >= 0 && (r2 < c2) && (r2 > T(0))) body(jj[k], pj[k]);
        }
    }
}

__device__ __forceinline__ void enqueue(uint32_t* queue, uint32_t* qcount, bool need,
                                        uint32_t value)
{
    const unsigned b = __ballot_sync(0xffffffffu, need);
    if (!b) return;
    const unsigned lane = lane_id();
    const int leader = __ffs(b) - 1;
    uint32_t base = 0;
    if ((int)lane == leader) base = atomicAdd(qcount, (uint32_t)__popc(b));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (need) queue[base + __popc(b & lanemask_lt())] = value;
}

// ---------------------------------------------------------------------------
// skin lists (one per advective step)
// ---------------------------------------------------------------------------
// Every particle of a cell shares the cell's 3^d candidate block, so the
// lists are built per CELL: one block loads the block's candidates once,
// sorts them by original id in shared memory, and then each warp streams
// the sorted candidates past one particle of the cell -- the ballot-compacted
// survivors are already in ascending id, so no per-particle sort is needed.
// Blocks larger than the tile fall back to the per-particle collector.
// Periodic builds: the cell tile stores every candidate at its image
// nearest the cell's centre, so the skin test is a plain difference (no
// minimum image per test).  The shifted coordinate RN(x_j +- L) differs from
// the exact minimum-image difference by a rounding of L-scale values; the
// periodic skin radius carries a 1e-4 relative margin for it (skin_cs2),
// far above that error, and the lists are filtered exactly afterwards.
template <class T, int D>
__device__ __forceinline__ void tile_image(vec4<T>& p, const int (&cc)[3], const GridP<T>& g)
{
#if SPH_PERIODIC
    T* x = reinterpret_cast<T*>(&p);
#pragma unroll
    for (int k = 0; k < D; k++) {
        const T L = BoxOf<T>::L(k);
        if (L > T(0)) {
            const T c = g.o[k] + (T(cc[k]) + T(0.5)) * g.cs;
            const T d = x[k] - c;
            if (d > BoxOf<T>::hL(k)) x[k] = x[k] - L;
            else if (d < -BoxOf<T>::hL(k)) x[k] = x[k] + L;
        }
    }
#else
    (void)p; (void)cc; (void)g;
#endif
}

// the skin test's r2 against a tile candidate (already imaged)
template <class T, int D>
__device__ __forceinline__ T tile_r2(const T (&xi)[3], const T (&xj)[3])
{
    T r2 = RN<T>::mul(RN<T>::sub(xi[0], xj[0]), RN<T>::sub(xi[0], xj[0]));
    r2 = RN<T>::add(r2, RN<T>::mul(RN<T>::sub(xi[1], xj[1]), RN<T>::sub(xi[1], xj[1])));
    if (D == 3) r2 = RN<T>::add(r2, RN<T>::mul(RN<T>::sub(xi[2], xj[2]), RN<T>::sub(xi[2], xj[2])));
    return r2;
}

// The skin test's r2 with fused multiply-adds: the skin lists only need to
// be a superset of the pairs within cutoff + skin - margin (skin_eff keeps a
// margin of 1e-4 relative, far above the ulp-level difference from the
// exact r2), so this test need not round like the reference's
template <class T, int D>
__device__ __forceinline__ T skin_r2(const T (&xi)[3], const T (&xj)[3])
{
    const T dx = xi[0] - xj[0], dy = xi[1] - xj[1];
    T r2 = fma_rn(dy, dy, dx * dx);
    if (D == 3) {
        const T dz = xi[2] - xj[2];
        r2 = fma_rn(dz, dz, r2);
    }
    return r2;
}

// Box of cell cc widened for rounding and opened at bounded grid faces
// (clamped particles live beyond them): a candidate farther than the skin
// reach from it is in no skin list of the cell's particles (SPH_SKIN_PRUNE)
template <class T, int D>
struct CellReach {
    T lo[3], hi[3], r2;
    __device__ __forceinline__ CellReach(const int (&cc)[3], const GridP<T>& g, T cs2)
    {
        const T w = T(1e-4) * g.cs, inf = T(INFINITY);
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const T a = g.o[k] + T(cc[k]) * g.cs;
#if SPH_PERIODIC
            lo[k] = a - w;
            hi[k] = a + g.cs + w;
#else
            lo[k] = cc[k] > 0 ? a - w : -inf;
            hi[k] = cc[k] < g.s[k] - 1 ? a + g.cs + w : inf;
#endif
        }
        r2 = cs2 * T(1.0002);
    }
    // the box spanned by the cell's own particles (bounded grids): every
    // candidate within reach of a particle is within reach of this box
    __device__ __forceinline__ CellReach(const T (&bl)[3], const T (&bh)[3], const GridP<T>& g,
                                         T cs2)
    {
        const T w = T(1e-4) * g.cs;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            lo[k] = bl[k] - w;
            hi[k] = bh[k] + w;
        }
        r2 = cs2 * T(1.0002);
    }
    __device__ __forceinline__ bool reaches(const vec4<T>& p) const
    {
        const T x[3] = {p.x, p.y, p.z};
        T d2 = T(0);
#pragma unroll
        for (int k = 0; k < D; k++) {
            const T d = fmax(fmax(lo[k] - x[k], x[k] - hi[k]), T(0));
            d2 = fma_rn(d, d, d2);
        }
        return d2 <= r2;
    }
};

template <class T, int D> struct SkinTile;
#ifndef SPH_SKIN2_THREADS
#define SPH_SKIN2_THREADS 128
#endif
#ifndef SPH_SKIN2_CANDS
#define SPH_SKIN2_CANDS 256
#endif
template <> struct SkinTile<float, 2> {
    static constexpr int kThreads = SPH_SKIN2_THREADS, kCands = SPH_SKIN2_CANDS;
};
#ifndef SPH_SKIN3_THREADS
#define SPH_SKIN3_THREADS 128
#endif
#ifndef SPH_SKIN3_CANDS
#define SPH_SKIN3_CANDS 768
#endif
template <> struct SkinTile<float, 3> {
    static constexpr int kThreads = SPH_SKIN3_THREADS, kCands = SPH_SKIN3_CANDS;
};
template <> struct SkinTile<double, 2> { static constexpr int kThreads = 128, kCands = 256; };
template <> struct SkinTile<double, 3> { static constexpr int kThreads = 256, kCands = 512; };

// Ascending bitonic sort of the P (power of two, >= 64) keys in shared
// memory: stages whose partner distance is < 64 run in registers on 64-key
// chunks (2 per lane, shuffles), the wider ones as shared-memory passes.
template <class K>
__device__ __forceinline__ void chunk_bitonic(K (&v)[2], int base, int k, int jtop, unsigned lane)
{
    for (int j = jtop; j > 0; j >>= 1) {
        if (j >= 2) {
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const K o = __shfl_xor_sync(0xffffffffu, v[r], j >> 1);
                const int e = base + 2 * (int)lane + r;
                const bool up = (e & k) == 0, lower = (e & j) == 0;
                // keep the smaller iff lower == up
                v[r] = ((o < v[r]) == (lower == up)) ? o : v[r];
            }
        } else {
            const int e = base + 2 * (int)lane;
            const bool up = (e & k) == 0;
            const K x0 = v[0], x1 = v[1];
            const bool sw = (x0 > x1) == up;
            v[0] = sw ? x1 : x0;
            v[1] = sw ? x0 : x1;
        }
    }
}

// chunk_bitonic with a compile-time top partner distance (straight-line
// stages; the runtime-k merge stages otherwise dispatch through a jump table)
template <int J, class K>
__device__ __forceinline__ void chunk_bitonic_ct(K (&v)[2], int base, int k, unsigned lane)
{
    if constexpr (J >= 2) {
#pragma unroll
        for (int r = 0; r < 2; r++) {
            const K o = __shfl_xor_sync(0xffffffffu, v[r], J >> 1);
            const int e = base + 2 * (int)lane + r;
            const bool up = (e & k) == 0, lower = (e & J) == 0;
            v[r] = ((o < v[r]) == (lower == up)) ? o : v[r];
        }
        chunk_bitonic_ct<J / 2>(v, base, k, lane);
    } else {
        const int e = base + 2 * (int)lane;
        const bool up = (e & k) == 0;
        const K x0 = v[0], x1 = v[1];
        const bool sw = (x0 > x1) == up;
        v[0] = sw ? x1 : x0;
        v[1] = sw ? x0 : x1;
    }
}

template <int NT, class K>
__device__ __forceinline__ void block_bitonic(K* key, int P)
{
    constexpr int NW = NT / 32;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    for (int c = warp; c < (P >> 6); c += NW) {   // chunks of 64: k = 2 .. 64
        const int base = c << 6;
        K v[2] = {key[base + 2 * lane], key[base + 2 * lane + 1]};
        for (int k = 2; k <= 64; k <<= 1) chunk_bitonic(v, base, k, k >> 1, lane);
        key[base + 2 * lane] = v[0];
        key[base + 2 * lane + 1] = v[1];
    }
    __syncthreads();
    for (int k = 128; k <= P; k <<= 1) {
        for (int j = k >> 1; j >= 64; j >>= 1) {
            for (int q = threadIdx.x; q < (P >> 1); q += NT) {
                const int lo = ((q & ~(j - 1)) << 1) | (q & (j - 1)), hi = lo + j;
                const K x0 = key[lo], x1 = key[hi];
                if ((x0 > x1) == ((lo & k) == 0)) { key[lo] = x1; key[hi] = x0; }
            }
            __syncthreads();
        }
        for (int c = warp; c < (P >> 6); c += NW) {
            const int base = c << 6;
            K v[2] = {key[base + 2 * lane], key[base + 2 * lane + 1]};
#if SPH_SKIN_SORT_CT
            chunk_bitonic_ct<32>(v, base, k, lane);
#else
            chunk_bitonic(v, base, k, 32, lane);
#endif
            key[base + 2 * lane] = v[0];
            key[base + 2 * lane + 1] = v[1];
        }
        __syncthreads();
    }
}

// All-ascending bitonic network (each merge level starts with a "flip"
// stage, partner i ^ (k - 1), then half-cleaners i ^ j; every comparator
// puts the smaller key at the lower index).  With the M real keys first and
// +inf (0xffffffff) padding after them, a comparator whose upper index is
// >= M would compare with +inf and leave both keys in place, so it is
// skipped: padding is never read or written and 64-key chunks wholly past
// M are never loaded -- the work follows M, not the power of two P.
// In registers: 2 keys per lane (positions base + 2 lane + r) of a 64-key
// chunk; keys are unsigned, so each comparator is one min or max.
template <class K>
__device__ __forceinline__ K cmp_keep(K v, K o, bool keep_min)
{
    return keep_min ? (o < v ? o : v) : (o < v ? v : o);
}

// flip stage of block size KB (4..64) within a chunk: element 2 l + r pairs
// with element 2 l' + 1 - r of lane l' = l ^ (KB / 2 - 1)
template <int KB, class K>
__device__ __forceinline__ void chunk_flip(K (&v)[2], unsigned lane)
{
    if constexpr (KB == 2) {
        const K a = v[0], b = v[1];
        v[0] = a < b ? a : b;
        v[1] = a < b ? b : a;
    } else {
        const K o0 = __shfl_xor_sync(0xffffffffu, v[0], KB / 2 - 1);
        const K o1 = __shfl_xor_sync(0xffffffffu, v[1], KB / 2 - 1);
        const bool lower = (lane & (KB / 4)) == 0;
        v[0] = cmp_keep(v[0], o1, lower);
        v[1] = cmp_keep(v[1], o0, lower);
    }
}

// half-cleaner stages J, J/2, .., 1 within a chunk (partner i ^ j)
template <int J, class K>
__device__ __forceinline__ void chunk_clean(K (&v)[2], unsigned lane)
{
    if constexpr (J >= 2) {
        const bool lower = (lane & (J / 2)) == 0;
        const K o0 = __shfl_xor_sync(0xffffffffu, v[0], J / 2);
        const K o1 = __shfl_xor_sync(0xffffffffu, v[1], J / 2);
        v[0] = cmp_keep(v[0], o0, lower);
        v[1] = cmp_keep(v[1], o1, lower);
        chunk_clean<J / 2>(v, lane);
    } else if constexpr (J == 1) {
        const K a = v[0], b = v[1];
        v[0] = a < b ? a : b;
        v[1] = a < b ? b : a;
    }
}

template <int KB, class K>
__device__ __forceinline__ void chunk_sort_levels(K (&v)[2], unsigned lane)
{
    chunk_flip<KB>(v, lane);
    chunk_clean<KB / 4>(v, lane);
    if constexpr (KB < 64) chunk_sort_levels<KB * 2>(v, lane);
}

template <int NT, class K>
__device__ __forceinline__ void block_sort_asc(K* key, int P, int M)
{
    constexpr int NW = NT / 32;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const int nchunks = (M + 63) >> 6;   // chunks holding a real key
    for (int c = warp; c < nchunks; c += NW) {   // levels k = 2 .. 64
        const int base = c << 6;
        K v[2] = {key[base + 2 * lane], key[base + 2 * lane + 1]};
        chunk_sort_levels<2>(v, lane);
        key[base + 2 * lane] = v[0];
        key[base + 2 * lane + 1] = v[1];
    }
    __syncthreads();
    for (int k = 128; k <= P; k <<= 1) {
        for (int q = threadIdx.x; q < (P >> 1); q += NT) {   // flip stage
            const int h = k >> 1, t = q & (h - 1), blk = (q & ~(h - 1)) << 1;
            const int lo = blk + t, hi = blk + k - 1 - t;
            if (hi < M) {
                const K x0 = key[lo], x1 = key[hi];
                if (x1 < x0) { key[lo] = x1; key[hi] = x0; }
            }
        }
        __syncthreads();
        for (int j = k >> 2; j >= 64; j >>= 1) {
            for (int q = threadIdx.x; q < (P >> 1); q += NT) {
                const int lo = ((q & ~(j - 1)) << 1) | (q & (j - 1)), hi = lo + j;
                if (hi < M) {
                    const K x0 = key[lo], x1 = key[hi];
                    if (x1 < x0) { key[lo] = x1; key[hi] = x0; }
                }
            }
            __syncthreads();
        }
        for (int c = warp; c < nchunks; c += NW) {   // j = 32 .. 1 in registers
            const int base = c << 6;
            K v[2] = {key[base + 2 * lane], key[base + 2 * lane + 1]};
            chunk_clean<32>(v, lane);
            key[base + 2 * lane] = v[0];
            key[base + 2 * lane + 1] = v[1];
        }
        __syncthreads();
    }
}

// The same network with 4 keys per lane (positions base + 4 lane + r of a
// 128-key chunk): partner distances 1 and 2 stay inside a thread.
template <class K>
__device__ __forceinline__ void cas_pair(K& a, K& b)
{
    const K lo = a < b ? a : b, hi = a < b ? b : a;
    a = lo;
    b = hi;
}

template <int KB, class K>
__device__ __forceinline__ void chunk4_flip(K (&v)[4], unsigned lane)
{
    if constexpr (KB == 2) {
        cas_pair(v[0], v[1]);
        cas_pair(v[2], v[3]);
    } else if constexpr (KB == 4) {
        cas_pair(v[0], v[3]);
        cas_pair(v[1], v[2]);
    } else {   // element 4 l + r pairs with 4 l' + 3 - r, l' = l ^ (KB / 4 - 1)
        K o[4];
#pragma unroll
        for (int r = 0; r < 4; r++) o[r] = __shfl_xor_sync(0xffffffffu, v[r], KB / 4 - 1);
        const bool lower = (lane & (KB / 8)) == 0;
#pragma unroll
        for (int r = 0; r < 4; r++) v[r] = cmp_keep(v[r], o[3 - r], lower);
    }
}

template <int J, class K>
__device__ __forceinline__ void chunk4_clean(K (&v)[4], unsigned lane)
{
    if constexpr (J >= 4) {
        const bool lower = (lane & (J / 4)) == 0;
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const K o = __shfl_xor_sync(0xffffffffu, v[r], J / 4);
            v[r] = cmp_keep(v[r], o, lower);
        }
        chunk4_clean<J / 2>(v, lane);
    } else if constexpr (J == 2) {
        cas_pair(v[0], v[2]);
        cas_pair(v[1], v[3]);
        chunk4_clean<1>(v, lane);
    } else if constexpr (J == 1) {
        cas_pair(v[0], v[1]);
        cas_pair(v[2], v[3]);
    }
}

template <int KB, class K>
__device__ __forceinline__ void chunk4_sort_levels(K (&v)[4], unsigned lane)
{
    chunk4_flip<KB>(v, lane);
    chunk4_clean<KB / 4>(v, lane);
    if constexpr (KB < 128) chunk4_sort_levels<KB * 2>(v, lane);
}

// P >= 128; keys [M, roundup(M, 128)) hold +inf
template <int NT, class K>
__device__ __forceinline__ void block_sort_asc4(K* key, int P, int M)
{
    constexpr int NW = NT / 32;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const int nchunks = (M + 127) >> 7;
    auto ld4 = [&](int base, K (&v)[4]) {
        const uint4 q = *reinterpret_cast<const uint4*>(key + base + 4 * lane);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    };
    auto st4 = [&](int base, const K (&v)[4]) {
        *reinterpret_cast<uint4*>(key + base + 4 * lane) = make_uint4(v[0], v[1], v[2], v[3]);
    };
    for (int c = warp; c < nchunks; c += NW) {   // levels k = 2 .. 128
        K v[4];
        ld4(c << 7, v);
        chunk4_sort_levels<2>(v, lane);
        st4(c << 7, v);
    }
    __syncthreads();
    for (int k = 256; k <= P; k <<= 1) {
        const int h = k >> 1;
        const int qf = ((M + k - 1) & ~(k - 1)) >> 1;   // flip pairs of blocks holding a real key
        for (int q = threadIdx.x; q < qf; q += NT) {
            const int t = q & (h - 1), blk = (q & ~(h - 1)) << 1;
            const int lo = blk + t, hi = blk + k - 1 - t;
            if (hi < M) {
                const K x0 = key[lo], x1 = key[hi];
                if (x1 < x0) { key[lo] = x1; key[hi] = x0; }
            }
        }
        __syncthreads();
        for (int j = k >> 2; j >= 128; j >>= 1) {
            for (int q = threadIdx.x; q < (P >> 1); q += NT) {
                const int lo = ((q & ~(j - 1)) << 1) | (q & (j - 1)), hi = lo + j;
                if (hi >= M) break;   // hi grows with q: no later pair is real
                const K x0 = key[lo], x1 = key[hi];
                if (x1 < x0) { key[lo] = x1; key[hi] = x0; }
            }
            __syncthreads();
        }
        for (int c = warp; c < nchunks; c += NW) {   // j = 64 .. 1 in registers
            K v[4];
            ld4(c << 7, v);
            chunk4_clean<64>(v, lane);
            st4(c << 7, v);
        }
        __syncthreads();
    }
}

template <class T, int D>
__global__ void __launch_bounds__(SkinTile<T, D>::kThreads, SPH_SKIN_THREADS_PER_SM / SkinTile<T, D>::kThreads)
k_skin_tile(const EngAcc<T> acc, const GridP<T> g, T cs2, Eng<T> E,
            const uint32_t* __restrict__ cells, const uint32_t* __restrict__ ncells_p,
            const uint32_t* __restrict__ phys_of_id, int wall_pairs, int fresh,
            uint32_t* __restrict__ work)
{
    constexpr int NT = SkinTile<T, D>::kThreads, NW = NT / 32, kC = SkinTile<T, D>::kCands;
    constexpr int kP = kC <= 64 ? 64 : (kC <= 128 ? 128 : (kC <= 256 ? 256 : (kC <= 512 ? 512
                                     : (kC <= 1024 ? 1024 : 2048))));
    static_assert(kP >= 128, "the 4-key sort works on 128-key chunks");
    __shared__ __align__(16) uint32_t sj[kP];   // candidate ids, sorted; then their indices j
    __shared__ vec4<T> spos[kC];       // positions in sorted order
    __shared__ uint32_t run_start[2 * 9], run_pre[2 * 9 + 1];
    __shared__ int s_kept;
    // per warp: the two particles' survivors, flushed as int4 quads (f32
    // only: the f64 tile would drop the 3D build below 8 CTAs per SM)
    constexpr bool kStage = SPH_SKIN_STAGE && sizeof(T) == 4;
    __shared__ __align__(16) int32_t stage[kStage ? NW : 1][2][kStage ? kCap : 4];
    const unsigned tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const unsigned lt = lanemask_lt();
    const int64_t nf = E.nf;
    const T inf = T(INFINITY);
    const uint32_t ncells = *(volatile const uint32_t*)ncells_p;
    // SPH_SKIN_DYN: after its first cell a CTA takes the next unclaimed one
    // (*work counts the cells claimed beyond the first gridDim.x), so cells of
    // uneven cost spread over the CTAs; else a static grid stride
    __shared__ uint32_t s_next;
    __shared__ T s_bb[NW][6];   // per-warp bounding boxes of the cell's particles
    auto next_cell = [&](uint32_t cur) -> uint32_t {
        if (!SPH_SKIN_DYN) return cur + gridDim.x;
        if (tid == 0) s_next = gridDim.x + atomicAdd(work, 1u);
        __syncthreads();
        return s_next;
    };
    for (uint32_t ci = blockIdx.x; ci < ncells; ci = next_cell(ci)) {
        const uint32_t c = cells[ci];   // cell keys are 32-bit: 32-bit divisions
        const uint32_t f0 = E.offs_f[c], f1 = E.offs_f[c + 1];
        const uint32_t w0 = E.offs_w[c], w1 = E.offs_w[c + 1];
        const int ntf = (int)(f1 - f0), nt = ntf + (int)(w1 - w0);
        int cc[3];
        if (D == 3) {
            const uint32_t s2 = (uint32_t)g.s[2], s1 = (uint32_t)g.s[1];
            const uint32_t col = c / s2;
            cc[2] = (int)(c - col * s2);
            cc[0] = (int)(col / s1);
            cc[1] = (int)(col - (uint32_t)cc[0] * s1);
        } else {
            const uint32_t s1 = (uint32_t)g.s[1];
            cc[0] = (int)(c / s1);
            cc[1] = (int)(c - (uint32_t)cc[0] * s1);
            cc[2] = 0;
        }
#if SPH_PERIODIC
        const PerBlock pb = per_block<T, D>(g, cc);
        const int rps = per_runs(pb);
        const int nruns = acc.nsegs() * rps;
#else
        const int xlo = max(cc[0] - 1, 0), xhi = min(cc[0] + 1, g.s[0] - 1);
        const int ylo = max(cc[1] - 1, 0), yhi = min(cc[1] + 1, g.s[1] - 1);
        const int zlo = D == 3 ? max(cc[2] - 1, 0) : 0;
        const int zhi = D == 3 ? min(cc[2] + 1, g.s[2] - 1) : 0;
        const int nyr = D == 3 ? (yhi - ylo + 1) : 1;
        const int rps = (xhi - xlo + 1) * nyr;
        const int nruns = 2 * rps;
#endif
        if (warp == 0) {   // run bounds of both segments + exclusive prefix
            if (SPH_SKIN_SORT_ASC && lane == 0) s_kept = 0;
            int64_t s0 = 0, s1 = 0;
            if ((int)lane < nruns) {
                const int seg = (int)lane / rps, rr = (int)lane - seg * rps;
                uint32_t klo, khi;
#if SPH_PERIODIC
                per_run<T, D>(g, pb, rr, klo, khi);
#else
                const int ax = xlo + rr / nyr, ay = ylo + rr % nyr;
                if (D == 3) {
                    const uint32_t rowk = ((uint32_t)ax * g.s[1] + ay) * g.s[2];
                    klo = rowk + zlo;
                    khi = rowk + zhi;
                } else {
                    klo = (uint32_t)ax * g.s[1] + ylo;
                    khi = (uint32_t)ax * g.s[1] + yhi;
                }
#endif
                acc.run(seg, klo, khi, s0, s1);
            }
            const uint32_t len = (uint32_t)(s1 - s0);
            uint32_t incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (unsigned)o) incl += t;
            }
            if ((int)lane < nruns) {
                run_start[lane] = (uint32_t)s0;
                run_pre[lane] = incl - len;
            }
            if ((int)lane == nruns - 1) run_pre[nruns] = incl;
        }
        __syncthreads();
        const int M = (int)run_pre[nruns];
        if (!wall_pairs && run_pre[rps] == 0) {
            // wall-only block (no fluid candidate, so no fluid particle in the
            // cell): walls' lists hold fluid neighbours only -- all empty; the
            // static wall-wall counts (nww) were set by the first build
            for (int t = (int)tid; t < nt; t += NT) {
                const int64_t i = nf + w0 + t;
                T xi[3];
                to3<T>(E.pos[i], xi);
                int cxyz[3];
                E.cell0[i] = fresh || cell_key_of<T, D>(xi, g, cxyz) == (uint32_t)c
                                 ? (uint32_t)c : kInvalidCell;
                E.lcount[E.nf_pad + (i - nf)] = 0;
                E.disp[i] = T(0);
                E.disp0[i] = T(0);
            }
            __syncthreads();
            continue;
        }
        if (M > kC) {   // oversized block: per-particle path (k_skin_big)
            if (tid == 0) E.queue[atomicAdd(E.qcount, 1u)] = (uint32_t)c;
            __syncthreads();
            continue;
        }
#if SPH_SKIN_SORT_ASC
        // kept candidates' ids appended in any order (warp-aggregated), then
        // sorted by a network that never touches the slots past them
        int r = 0;   // k only grows: each thread's run search resumes where it stopped
        uint32_t nb = nruns > 1 ? run_pre[1] : 0xffffffffu;   // run r ends at nb
#if SPH_SKIN_BBOX && SPH_SKIN_PRUNE
        // the cell's particles' bounding box (block min / max reduction)
        T bl[3] = {inf, inf, inf}, bh[3] = {-inf, -inf, -inf};
        for (int t = (int)tid; t < nt; t += NT) {
            const int64_t i = t < ntf ? (int64_t)f0 + t : nf + w0 + (t - ntf);
            T x[3];
            to3<T>(E.pos[i], x);
#pragma unroll
            for (int k = 0; k < D; k++) {
                bl[k] = fmin(bl[k], x[k]);
                bh[k] = fmax(bh[k], x[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < D; k++) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                bl[k] = fmin(bl[k], __shfl_xor_sync(0xffffffffu, bl[k], o));
                bh[k] = fmax(bh[k], __shfl_xor_sync(0xffffffffu, bh[k], o));
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < D; k++) {
                s_bb[warp][k] = bl[k];
                s_bb[warp][3 + k] = bh[k];
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < D; k++) {
            bl[k] = s_bb[0][k];
            bh[k] = s_bb[0][3 + k];
#pragma unroll
            for (int w = 1; w < NW; w++) {
                bl[k] = fmin(bl[k], s_bb[w][k]);
                bh[k] = fmax(bh[k], s_bb[w][3 + k]);
            }
        }
        if (D == 2) { bl[2] = T(0); bh[2] = T(0); }
        const CellReach<T, D> reach(bl, bh, g, cs2);
#else
        const CellReach<T, D> reach(cc, g, cs2);
#endif
        // SPH_SKIN_BLOCKED: thread t takes candidates [t per, t per + per), so
        // its run search moves past few run boundaries; else k = t + NT i
        const int per = SPH_SKIN_BLOCKED ? (M + NT - 1) / NT : 1;
        for (int kb = 0; kb < (SPH_SKIN_BLOCKED ? per : M); kb += (SPH_SKIN_BLOCKED ? 1 : NT)) {
            const int k = SPH_SKIN_BLOCKED ? (int)tid * per + kb : kb + (int)tid;
            bool keep = false;
            uint32_t key = 0;
            if (k < M) {
                while ((uint32_t)k >= nb) {
                    r++;
                    nb = r + 1 < nruns ? run_pre[r + 1] : 0xffffffffu;
                }
                const uint32_t ph = run_start[r] + ((uint32_t)k - run_pre[r]);
                keep = true;
                if (SPH_SKIN_PRUNE) {
                    vec4<T> p = E.pos[ph];
                    tile_image<T, D>(p, cc, g);
                    keep = reach.reaches(p);
                }
                if (keep) key = E.id[ph];
            }
            const unsigned b = __ballot_sync(0xffffffffu, keep);
            if (b) {
                const int leader = __ffs(b) - 1;
                int base = 0;
                if ((int)lane == leader) base = atomicAdd(&s_kept, __popc(b));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (keep) sj[base + __popc(b & lt)] = key;
            }
        }
        __syncthreads();
        const int Mk = s_kept;   // candidates kept
        constexpr int kChunk = SPH_SKIN_SORT_K4 ? 128 : 64;
        int P = kChunk;
        while (P < Mk) P <<= 1;
        for (int k = Mk + (int)tid; k < ((Mk + kChunk - 1) & ~(kChunk - 1)); k += NT)
            sj[k] = 0xffffffffu;
        __syncthreads();
        // ids are unique: a total order
        if (SPH_SKIN_SORT_K4) block_sort_asc4<NT>(sj, P, Mk);
        else block_sort_asc<NT>(sj, P, Mk);
#else
        int P = 64;
        while (P < M) P <<= 1;
        int r = 0;   // k only grows: each thread's run search resumes where it stopped
        int kept = 0;
        const CellReach<T, D> reach(cc, g, cs2);
        for (int k = tid; k < P; k += NT) {
            uint32_t key = 0xffffffffu;   // pruned / padding: sorts to the end
            if (k < M) {
                while (r + 1 < nruns && run_pre[r + 1] <= (uint32_t)k) r++;
                const uint32_t ph = run_start[r] + ((uint32_t)k - run_pre[r]);
                bool keep = true;
                if (SPH_SKIN_PRUNE) {
                    vec4<T> p = E.pos[ph];
                    tile_image<T, D>(p, cc, g);
                    keep = reach.reaches(p);
                }
                if (keep) {
                    key = E.id[ph];
                    kept++;
                }
            }
            sj[k] = key;
        }
        if (tid == 0) s_kept = 0;
        __syncthreads();
        kept = warp_sum(kept);
        if (lane == 0 && kept) atomicAdd(&s_kept, kept);
        __syncthreads();
        const int Mk = s_kept;   // candidates kept, first after the sort
        block_bitonic<NT>(sj, P);   // ids are unique: a total order
#endif
        const int Mp = (Mk + 31) & ~31;
        for (int k = tid; k < Mp; k += NT) {
            vec4<T> p;
            if (k < Mk) {
                const uint32_t j = phys_of_id[sj[k]];
                sj[k] = j;
                p = E.pos[j];
                tile_image<T, D>(p, cc, g);
            } else {   // padding: never within reach
                p.x = inf; p.y = inf; p.z = inf; p.w = T(0);
                sj[k] = 0;
            }
            spos[k] = p;
        }
        __syncthreads();
        // two particles of the cell per warp pass: each candidate's shared
        // data is read once for both
        for (int t = 2 * warp; t < nt; t += 2 * NW) {
            const bool hasB = t + 1 < nt;
            const bool flA = t < ntf, flB = t + 1 < ntf;
            const int64_t iA = flA ? (int64_t)f0 + t : nf + w0 + (t - ntf);
            const int64_t iB = hasB ? (flB ? (int64_t)f0 + t + 1 : nf + w0 + (t + 1 - ntf)) : iA;
            const int64_t slA = flA ? iA : E.nf_pad + (iA - nf);
            const int64_t slB = flB ? iB : E.nf_pad + (iB - nf);
            T xa[3], xb[3];
            to3<T>(E.pos[iA], xa);
            to3<T>(E.pos[iB], xb);
            int32_t* __restrict__ lpA = E.lists + ell_base(slA);
            int32_t* __restrict__ lpB = E.lists + ell_base(slB);
            int cntA = 0, cntB = 0, naA = 0, naB = 0;
            // FO: both particles fluid (warp-uniform; most passes) -- every
            // candidate is eligible and no wall-wall count is kept
            auto scan = [&](auto fo) {
                constexpr bool FO = decltype(fo)::value;
                for (int base = 0; base < Mp; base += 32) {
                    const int k = base + (int)lane;
                    const uint32_t j = sj[k];
                    T xj[3];
                    to3<T>(spos[k], xj);
#if SPH_PERIODIC
                    const T r2a = tile_r2<T, D>(xa, xj);
                    const T r2b = tile_r2<T, D>(xb, xj);
#else
                    const T r2a = SPH_SKIN_FMA ? skin_r2<T, D>(xa, xj) : accept_r2<T, D>(xa, xj);
                    const T r2b = SPH_SKIN_FMA ? skin_r2<T, D>(xb, xj) : accept_r2<T, D>(xb, xj);
#endif
                    const bool jf = FO || (int64_t)j < nf;
                    const bool stA = (FO || flA || jf) && r2a < cs2 && j != (uint32_t)iA;
                    const bool stB = (FO || hasB) && (FO || flB || jf) && r2b < cs2 &&
                                     j != (uint32_t)iB;
                    const unsigned bA = __ballot_sync(0xffffffffu, stA);
                    const unsigned bB = __ballot_sync(0xffffffffu, stB);
                    if (stA) {
                        const int p = cntA + __popc(bA & lt);
                        if (p < kCap) {
                            if (kStage) stage[kStage ? warp : 0][0][p] = (int32_t)j;
                            else lpA[ell_off(p)] = (int32_t)j;
                        }
                    }
                    if (stB) {
                        const int p = cntB + __popc(bB & lt);
                        if (p < kCap) {
                            if (kStage) stage[kStage ? warp : 0][1][p] = (int32_t)j;
                            else lpB[ell_off(p)] = (int32_t)j;
                        }
                    }
                    cntA += __popc(bA);
                    cntB += __popc(bB);
                    if (!FO && wall_pairs && (!flA || !flB)) {   // walls: static wall-wall count
                        // (the reference's exact acceptance test)
                        const T e2a = accept_r2<T, D>(xa, xj), e2b = accept_r2<T, D>(xb, xj);
                        const bool ctA = !flA && !jf && e2a < g.c2 && e2a > T(0) &&
                                         j != (uint32_t)iA;
                        const bool ctB = hasB && !flB && !jf && e2b < g.c2 && e2b > T(0) &&
                                         j != (uint32_t)iB;
                        naA += __popc(__ballot_sync(0xffffffffu, ctA));
                        naB += __popc(__ballot_sync(0xffffffffu, ctB));
                    }
                }
            };
#if SPH_SKIN_FLUID_PASS
            if (flB) scan(std::true_type{});   // flB implies flA and hasB
            else scan(std::false_type{});
#else
            scan(std::false_type{});
#endif
            if (kStage) {   // the staged lists out as whole quads (tile-ELL)
                __syncwarp();
                const int qa = (min(cntA, kCap) + 3) >> 2;
                const int qb = hasB ? (min(cntB, kCap) + 3) >> 2 : 0;
                const int4* sa = reinterpret_cast<const int4*>(stage[kStage ? warp : 0][0]);
                const int4* sb = reinterpret_cast<const int4*>(stage[kStage ? warp : 0][1]);
                for (int q = (int)lane; q < qa + qb; q += 32) {
                    if (q < qa) reinterpret_cast<int4*>(lpA)[q * 32] = sa[q];
                    else reinterpret_cast<int4*>(lpB)[(q - qa) * 32] = sb[q - qa];
                }
                __syncwarp();
            }
            if (lane < 2 && (lane == 0 || hasB)) {
                const int64_t i = lane ? iB : iA;
                const int64_t slot = lane ? slB : slA;
                const int cnt = lane ? cntB : cntA;
                T xi[3];
                xi[0] = lane ? xb[0] : xa[0];
                xi[1] = lane ? xb[1] : xa[1];
                xi[2] = lane ? xb[2] : xa[2];
                int cxyz[3];
                // fresh CLL: the particle's cell is c by construction
                const bool ok = (fresh || cell_key_of<T, D>(xi, g, cxyz) == (uint32_t)c) &&
                                cnt <= kCap;
                E.cell0[i] = ok ? (uint32_t)c : kInvalidCell;
                E.lcount[slot] = ok ? cnt : 0;
                if (wall_pairs) E.nww[slot] = lane ? naB : naA;
                E.disp[i] = T(0);
                E.disp0[i] = T(0);
            }
        }
        __syncthreads();   // shared tile reused by the next cell
    }
}

// the cells holding at least one particle (order irrelevant)
__global__ void __launch_bounds__(256)
k_nonempty_cells(const uint32_t* __restrict__ offs_f, const uint32_t* __restrict__ offs_w,
                 int64_t ncells, uint32_t* __restrict__ out, uint32_t* __restrict__ count)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ne = c < ncells && (offs_f[c] != offs_f[c + 1] || offs_w[c] != offs_w[c + 1]);
    const unsigned b = __ballot_sync(0xffffffffu, ne);
    if (!b) return;
    const unsigned lane = lane_id();
    const int leader = __ffs(b) - 1;
    uint32_t base = 0;
    if ((int)lane == leader) base = atomicAdd(count, (uint32_t)__popc(b));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (ne) out[base + __popc(b & lanemask_lt())] = (uint32_t)c;
}

__global__ void __launch_bounds__(256)
k_phys_of_id(const uint32_t* __restrict__ id, int64_t n, uint32_t* __restrict__ phys_of_id)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) phys_of_id[id[i]] = (uint32_t)i;
}

// Ascending bitonic sort of 32*PER keys held blocked in a warp (lane owns
// elements lane*PER .. lane*PER+PER-1).
template <int PER, class K>
__device__ __forceinline__ void warp_sort_blocked(K (&v)[PER], unsigned lane)
{
    constexpr int N = 32 * PER;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= PER) {
#pragma unroll
                for (int r = 0; r < PER; r++) {
                    const K o = __shfl_xor_sync(0xffffffffu, v[r], j / PER);
                    const int e = (int)lane * PER + r;
                    const bool up = (e & k) == 0, lower = (e & j) == 0;
                    v[r] = ((o < v[r]) == (lower == up)) ? o : v[r];
                }
            } else {
#pragma unroll
                for (int r = 0; r < PER; r++) {
                    if (r & j) continue;
                    const int e = (int)lane * PER + r;
                    const bool up = (e & k) == 0;
                    const K a = v[r], b = v[r ^ j];
                    const bool sw = (a > b) == up;
                    v[r] = sw ? b : a;
                    v[r ^ j] = sw ? a : b;
                }
            }
        }
    }
}

// Skin lists of small candidate blocks (<= 128, the 2D case): a warp per
// cell with the sort in registers and the candidates in a per-warp shared
// tile, no block barriers; larger blocks are passed on to k_skin_tile.
template <class T, int D, int PER>
__device__ __forceinline__ void skin_warp_load_sort(const Eng<T>& E, int M, int nruns,
                                                    uint32_t s0, uint32_t pre, unsigned lane,
                                                    uint32_t* sj)
{
    uint32_t v[PER];
    int base[PER];
#pragma unroll
    for (int q = 0; q < PER; q++) base[q] = -1;
    for (int r = 0; r < nruns; r++) {   // the last run starting at or before e holds e
        const uint32_t rp = __shfl_sync(0xffffffffu, pre, r);
        const uint32_t rs = __shfl_sync(0xffffffffu, s0, r);
#pragma unroll
        for (int q = 0; q < PER; q++) {
            const uint32_t e = lane * PER + q;
            if (rp <= e) base[q] = (int)(rs + (e - rp));
        }
    }
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const int e = (int)lane * PER + q;
        v[q] = (e < M) ? E.id[base[q]] : 0xffffffffu;
    }
    warp_sort_blocked<PER>(v, lane);
#pragma unroll
    for (int q = 0; q < PER; q++) sj[lane * PER + q] = v[q];
    __syncwarp();
}

template <class T, int D>
__global__ void __launch_bounds__(256, SPH_SKINW_MINB)
k_skin_warp(const GridP<T> g, T cs2, Eng<T> E, const uint32_t* __restrict__ cells,
            const uint32_t* __restrict__ ncells_p, const uint32_t* __restrict__ phys_of_id,
            uint32_t* __restrict__ big, uint32_t* __restrict__ nbig, int fresh,
            uint32_t* __restrict__ work)
{
    constexpr int NW = 8, kW = 128;
    __shared__ uint32_t wsj[NW][kW];
    __shared__ vec4<T> wpos[NW][kW];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    uint32_t* sj = wsj[warp];
    vec4<T>* spos = wpos[warp];
    const int64_t nf = E.nf;
    const T inf = T(INFINITY);
    const uint32_t ncells = *(volatile const uint32_t*)ncells_p;
    auto next_cell = [&](uint32_t cur) -> uint32_t {   // as k_skin_tile, per warp
        if (!SPH_SKIN_DYN) return cur + gridDim.x * NW;
        uint32_t v = 0;
        if (lane == 0) v = gridDim.x * NW + atomicAdd(work, 1u);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    for (uint32_t ci = blockIdx.x * NW + warp; ci < ncells; ci = next_cell(ci)) {
        const uint32_t c = cells[ci];   // cell keys are 32-bit: 32-bit divisions
        const uint32_t f0 = E.offs_f[c], f1 = E.offs_f[c + 1];
        const uint32_t w0 = E.offs_w[c], w1 = E.offs_w[c + 1];
        const int ntf = (int)(f1 - f0), nt = ntf + (int)(w1 - w0);
        int cc[3];
        if (D == 3) {
            const uint32_t s2 = (uint32_t)g.s[2], s1 = (uint32_t)g.s[1];
            const uint32_t col = c / s2;
            cc[2] = (int)(c - col * s2);
            cc[0] = (int)(col / s1);
            cc[1] = (int)(col - (uint32_t)cc[0] * s1);
        } else {
            const uint32_t s1 = (uint32_t)g.s[1];
            cc[0] = (int)(c / s1);
            cc[1] = (int)(c - (uint32_t)cc[0] * s1);
            cc[2] = 0;
        }
#if SPH_PERIODIC
        const PerBlock pb = per_block<T, D>(g, cc);
        const int rps = per_runs(pb);
        const int nruns = (E.nw > 0 ? 2 : 1) * rps;
#else
        const int xlo = max(cc[0] - 1, 0), xhi = min(cc[0] + 1, g.s[0] - 1);
        const int ylo = max(cc[1] - 1, 0), yhi = min(cc[1] + 1, g.s[1] - 1);
        const int zlo = D == 3 ? max(cc[2] - 1, 0) : 0;
        const int zhi = D == 3 ? min(cc[2] + 1, g.s[2] - 1) : 0;
        const int nyr = D == 3 ? (yhi - ylo + 1) : 1;
        const int rps = (xhi - xlo + 1) * nyr;
        const int nruns = 2 * rps;
#endif
        int64_t s0 = 0, s1 = 0;
        if ((int)lane < nruns) {
            const int seg = (int)lane / rps, rr = (int)lane - seg * rps;
            uint32_t klo, khi;
#if SPH_PERIODIC
            per_run<T, D>(g, pb, rr, klo, khi);
#else
            const int ax = xlo + rr / nyr, ay = ylo + rr % nyr;
            if (D == 3) {
                const uint32_t rowk = ((uint32_t)ax * g.s[1] + ay) * g.s[2];
                klo = rowk + zlo;
                khi = rowk + zhi;
            } else {
                klo = (uint32_t)ax * g.s[1] + ylo;
                khi = (uint32_t)ax * g.s[1] + yhi;
            }
#endif
            if (seg == 0) { s0 = E.offs_f[klo]; s1 = E.offs_f[khi + 1]; }
            else { s0 = nf + E.offs_w[klo]; s1 = nf + E.offs_w[khi + 1]; }
        }
        const uint32_t len = (uint32_t)(s1 - s0);
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += t;
        }
        const int M = (int)__shfl_sync(0xffffffffu, incl, 31);
        if (M > kW) {
            if (lane == 0) big[atomicAdd(nbig, 1u)] = (uint32_t)c;
            continue;
        }
        if (M <= 64)
            skin_warp_load_sort<T, D, 2>(E, M, nruns, (uint32_t)s0, incl - len, lane, sj);
        else
            skin_warp_load_sort<T, D, 4>(E, M, nruns, (uint32_t)s0, incl - len, lane, sj);
        const int Mp = (M + 31) & ~31;
        for (int k = (int)lane; k < Mp; k += 32) {
            vec4<T> p;
            if (k < M) {
                const uint32_t j = phys_of_id[sj[k]];
                sj[k] = j;
                p = E.pos[j];
                tile_image<T, D>(p, cc, g);
            } else {
                p.x = inf; p.y = inf; p.z = inf; p.w = T(0);
                sj[k] = 0;
            }
            spos[k] = p;
        }
        __syncwarp();
        for (int t = 0; t < nt; t += 2) {
            const bool hasB = t + 1 < nt;
            const bool flA = t < ntf, flB = t + 1 < ntf;
            const int64_t iA = flA ? (int64_t)f0 + t : nf + w0 + (t - ntf);
            const int64_t iB = hasB ? (flB ? (int64_t)f0 + t + 1 : nf + w0 + (t + 1 - ntf)) : iA;
            const int64_t slA = flA ? iA : E.nf_pad + (iA - nf);
            const int64_t slB = flB ? iB : E.nf_pad + (iB - nf);
            T xa[3], xb[3];
            to3<T>(E.pos[iA], xa);
            to3<T>(E.pos[iB], xb);
            int32_t* __restrict__ lpA = E.lists + ell_base(slA);
            int32_t* __restrict__ lpB = E.lists + ell_base(slB);
            int cntA = 0, cntB = 0, naA = 0, naB = 0;
            auto scan = [&](auto fo) {   // FO: both fluid (as in k_skin_tile)
                constexpr bool FO = decltype(fo)::value;
                for (int base = 0; base < Mp; base += 32) {
                    const int k = base + (int)lane;
                    const uint32_t j = sj[k];
                    T xj[3];
                    to3<T>(spos[k], xj);
#if SPH_PERIODIC
                    const T r2a = tile_r2<T, D>(xa, xj);
                    const T r2b = tile_r2<T, D>(xb, xj);
#else
                    const T r2a = accept_r2<T, D>(xa, xj);
                    const T r2b = accept_r2<T, D>(xb, xj);
#endif
                    const bool jf = FO || (int64_t)j < nf;
                    const bool stA = (FO || flA || jf) && r2a < cs2 && j != (uint32_t)iA;
                    const bool stB = (FO || hasB) && (FO || flB || jf) && r2b < cs2 &&
                                     j != (uint32_t)iB;
                    const unsigned bA = __ballot_sync(0xffffffffu, stA);
                    const unsigned bB = __ballot_sync(0xffffffffu, stB);
                    if (stA) lpA[ell_off(cntA + __popc(bA & lt))] = (int32_t)j;   // M <= 128 < kCap
                    if (stB) lpB[ell_off(cntB + __popc(bB & lt))] = (int32_t)j;
                    cntA += __popc(bA);
                    cntB += __popc(bB);
                    if (!FO && (!flA || !flB)) {
                        const bool ctA = !flA && !jf && r2a < g.c2 && r2a > T(0) &&
                                         j != (uint32_t)iA;
                        const bool ctB = hasB && !flB && !jf && r2b < g.c2 && r2b > T(0) &&
                                         j != (uint32_t)iB;
                        naA += __popc(__ballot_sync(0xffffffffu, ctA));
                        naB += __popc(__ballot_sync(0xffffffffu, ctB));
                    }
                }
            };
#if SPH_SKIN_FLUID_PASS
            if (flB) scan(std::true_type{});
            else scan(std::false_type{});
#else
            scan(std::false_type{});
#endif
            if (lane < 2 && (lane == 0 || hasB)) {
                const int64_t i = lane ? iB : iA;
                const int64_t slot = lane ? slB : slA;
                T xi[3];
                xi[0] = lane ? xb[0] : xa[0];
                xi[1] = lane ? xb[1] : xa[1];
                xi[2] = lane ? xb[2] : xa[2];
                int cxyz[3];
                const bool ok = fresh || cell_key_of<T, D>(xi, g, cxyz) == (uint32_t)c;
                E.cell0[i] = ok ? (uint32_t)c : kInvalidCell;
                E.lcount[slot] = ok ? (lane ? cntB : cntA) : 0;
                E.nww[slot] = lane ? naB : naA;
                E.disp[i] = T(0);
                E.disp0[i] = T(0);
            }
        }
        __syncwarp();
    }
}

// skin lists of the cells k_skin_tile queued (candidate block above the
// tile): one warp per particle of the cell, per-particle collect + sort
template <class T, int D>
__global__ void __launch_bounds__(kNlThreads, 4)
k_skin_big(const EngAcc<T> acc, const GridP<T> g, T cs2, Eng<T> E)
{
    __shared__ WarpBuf bufs[kNlWarps];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    WarpBuf& sb = bufs[warp];
    const uint32_t nq = *(volatile uint32_t*)E.qcount;
    const int64_t nf = E.nf;
    for (uint32_t q = blockIdx.x; q < nq; q += gridDim.x) {
        const uint32_t c = E.queue[q];
        const uint32_t f0 = E.offs_f[c], ntf = E.offs_f[c + 1] - f0;
        const uint32_t w0 = E.offs_w[c], nt = ntf + (E.offs_w[c + 1] - w0);
        for (uint32_t t = warp; t < nt; t += kNlWarps) {
            const bool fluid = t < ntf;
            const int64_t i = fluid ? (int64_t)f0 + t : nf + w0 + (t - ntf);
            const int64_t slot = fluid ? i : E.nf_pad + (i - nf);
            T xi[3];
            acc.position(i, xi);
            CollectCounts cnts = warp_collect<T, D, true>(acc, g, i, xi, cs2, fluid ? 3u : 1u, sb);
            int cxyz[3];
            const uint32_t key0 = cell_key_of<T, D>(xi, g, cxyz);
            int stored = cnts.stored;
            if (stored > kCap) {
                stored = 0;
            } else {
                warp_emit_sorted(sb, stored, lane, [&](int pos, uint32_t j) {
                    E.lists[ell_index(slot, pos)] = (int32_t)j;
                });
            }
            if (lane == 0) {
                E.cell0[i] = cnts.stored > kCap ? kInvalidCell : key0;
                E.lcount[slot] = stored;
                E.nww[slot] = cnts.accepted;
                E.disp[i] = T(0);
                E.disp0[i] = T(0);
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
// skin lists carried across a CLL rebuild (sph_engine_maintain_lists)
// ---------------------------------------------------------------------------
// The reference's candidate set of i within step s is every j whose step-s
// CLL cell lies in the 3^d block of i's current cell (neighborhood.py:
// 188-213).  A list valid before the rebuild (i still in its list cell, the
// displacement test passing) holds, in ascending id, the block members of
// the previous CLL within cutoff + skin at build time; membership changes
// only through particles whose CLL cell changed (movers).  So the list of
// step s = the old entries renumbered through the re-sort, minus those
// whose new cell left the block, plus the movers that entered the block
// within cutoff + skin now (enough: any later pair within the cutoff, with
// the validity test holding, is within cutoff + skin now).
template <class T>
__device__ __forceinline__ bool axis_periodic(int k)
{
#if SPH_PERIODIC
    return BoxOf<T>::L(k) > T(0);
#else
    (void)k;
    return false;
#endif
}

template <class T, int D>
__device__ __forceinline__ void key_coords(uint32_t key, const GridP<T>& g, int (&c)[3])
{
    if (D == 3) {
        c[2] = (int)(key % (uint32_t)g.s[2]);
        key /= (uint32_t)g.s[2];
    } else {
        c[2] = 0;
    }
    c[1] = (int)(key % (uint32_t)g.s[1]);
    c[0] = (int)(key / (uint32_t)g.s[1]);
}

// is the cell of key within the 3^d block of cell cc (clamped or wrapped)
template <class T, int D>
__device__ __forceinline__ bool in_block(uint32_t key, const int (&cc)[3], const GridP<T>& g)
{
    int c[3];
    key_coords<T, D>(key, g, c);
#pragma unroll
    for (int k = 0; k < D; k++) {
        int d = c[k] - cc[k];
        d = d < 0 ? -d : d;
        if (axis_periodic<T>(k) && g.s[k] - d < d) d = g.s[k] - d;
        if (d > 1) return false;
    }
    return true;
}

// movers: fluid particles whose CLL cell changed in this rebuild, counted per
// (new) cell for a CSR of arrivals
__global__ void __launch_bounds__(256)
k_mover_count(const uint32_t* __restrict__ key_sorted, const uint32_t* __restrict__ key_prev,
              int64_t nf, uint32_t* __restrict__ ccount)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nf && key_sorted[i] != key_prev[i]) atomicAdd(&ccount[key_sorted[i]], 1u);
}

__global__ void __launch_bounds__(256)
k_mover_fill(const uint32_t* __restrict__ key_sorted, const uint32_t* __restrict__ key_prev,
             int64_t nf, uint32_t* __restrict__ cursor, uint32_t* __restrict__ movers)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nf && key_sorted[i] != key_prev[i])
        movers[atomicAdd(&cursor[key_sorted[i]], 1u)] = (uint32_t)i;
}

// local displacement bound: the largest cellmax over each cell's 3^d block
template <class T, int D>
__global__ void __launch_bounds__(256)
k_blockmax(GridP<T> g, int64_t ncells, const uint32_t* __restrict__ cellmax,
           uint32_t* __restrict__ blockmax)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    int cc[3];
    key_coords<T, D>((uint32_t)c, g, cc);
    int lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        if (k >= D) { lo[k] = hi[k] = 0; continue; }
        if (axis_periodic<T>(k)) { lo[k] = cc[k] - 1; hi[k] = cc[k] + 1; }
        else { lo[k] = max(cc[k] - 1, 0); hi[k] = min(cc[k] + 1, g.s[k] - 1); }
    }
    uint32_t m = 0;
    for (int a = lo[0]; a <= hi[0]; a++)
        for (int b = lo[1]; b <= hi[1]; b++)
            for (int z = lo[2]; z <= hi[2]; z++) {
                const int ax = (a + g.s[0]) % g.s[0], by = (b + g.s[1]) % g.s[1];
                uint32_t key = (uint32_t)ax * g.s[1] + by;
                if (D == 3) key = key * g.s[2] + (z + g.s[2]) % g.s[2];
                m = max(m, cellmax[key]);
            }
    blockmax[c] = m;
}

// a carried epoch's path lengths into the (reset) per-cell maxima
__global__ void __launch_bounds__(256)
k_cellmax_seed(const uint32_t* __restrict__ key_sorted, const float* __restrict__ disp,
               int64_t nf, uint32_t* __restrict__ cellmax)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nf && disp[i] > 0.0f) atomicMax(&cellmax[key_sorted[i]], __float_as_uint(disp[i]));
}

template <class T, int D>
static void launch_blockmax(const SphEngine* e, cudaStream_t s)
{
    if (sizeof(T) != 4 || !e->cellmax || !e->blockmax || !e->key_sorted) return;
    note_launch(), k_blockmax<T, D><<<grid_for(e->ncells, 256), 256, 0, s>>>(
        grid_of_engine<T>(e), e->ncells, e->cellmax, e->blockmax);
}

#ifndef SPH_MAINTAIN_ARRIVALS
#define SPH_MAINTAIN_ARRIVALS 8   // arrivals merged per list (more: the list is rebuilt)
#endif

template <class T, int D>
__global__ void __launch_bounds__(128)
k_maintain(Eng<T> E, GridP<T> g, T cs2, T s_eff, const uint32_t* __restrict__ key_sorted,
           const uint32_t* __restrict__ key_prev, const uint32_t* __restrict__ perm,
           const uint32_t* __restrict__ inv, const int32_t* __restrict__ lists_old,
           const int32_t* __restrict__ lcount_old, int32_t* __restrict__ lists_new,
           int32_t* __restrict__ lcount_new, const uint32_t* __restrict__ moff,
           const uint32_t* __restrict__ movers)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool need = false;
    if (i < E.n) {
        const int64_t nf = E.nf;
        const bool fluid = i < nf;
        const int64_t slot = slot_of(E, i);
        const int64_t so = fluid ? (int64_t)perm[i] : slot;   // walls never move
        const uint32_t c0 = E.cell0[i];
        const T dmax = T(__longlong_as_double((long long)E.stats->dmax_bits));
        if (c0 == kInvalidCell || c0 != key_sorted[i] ||
            RN<T>::add_ru(RN<T>::sub_ru(E.disp[i], E.disp0[i]), dmax_for(E, c0, dmax)) > s_eff) {
            need = true;
        } else {
            int cc[3];
            key_coords<T, D>(c0, g, cc);
            T xi[3];
            to3<T>(E.pos[i], xi);
            // movers that entered the block, within cutoff + skin
            uint32_t arr[SPH_MAINTAIN_ARRIVALS];
            int na = 0;
            bool ovf = false;
            int lo[3], hi[3];
#pragma unroll
            for (int k = 0; k < 3; k++) {
                if (k >= D) { lo[k] = hi[k] = 0; continue; }
                if (axis_periodic<T>(k)) { lo[k] = cc[k] - 1; hi[k] = cc[k] + 1; }
                else { lo[k] = max(cc[k] - 1, 0); hi[k] = min(cc[k] + 1, g.s[k] - 1); }
            }
            for (int a = lo[0]; a <= hi[0]; a++)
                for (int b = lo[1]; b <= hi[1]; b++)
                    for (int z = lo[2]; z <= hi[2]; z++) {
                        const int ax = (a + g.s[0]) % g.s[0], by = (b + g.s[1]) % g.s[1];
                        const int cz = D == 3 ? (z + g.s[2]) % g.s[2] : 0;
                        uint32_t key = (uint32_t)ax * g.s[1] + by;
                        if (D == 3) key = key * g.s[2] + cz;
                        for (uint32_t m = moff[key]; m < moff[key + 1]; m++) {
                            const uint32_t j = movers[m];
                            if ((int64_t)j == i || in_block<T, D>(key_prev[j], cc, g)) continue;
                            T xj[3];
                            to3<T>(E.pos[j], xj);
#if SPH_PERIODIC
                            if (!(accept_r2<T, D>(xi, xj) < cs2)) continue;   // minimum image
#else
                            if (!(skin_r2<T, D>(xi, xj) < cs2)) continue;
#endif
                            if (na < SPH_MAINTAIN_ARRIVALS) arr[na++] = j;
                            else ovf = true;
                        }
                    }
            // arrivals in ascending id (insertion sort, a handful)
            for (int u = 1; u < na; u++) {
                const uint32_t v = arr[u], iv = E.id[v];
                int w = u - 1;
                while (w >= 0 && E.id[arr[w]] > iv) { arr[w + 1] = arr[w]; w--; }
                arr[w + 1] = v;
            }
            const int nl = lcount_old[so];
            int cnt = 0, a = 0;
            int32_t* __restrict__ lp = lists_new + ell_base(slot);
            const int32_t* __restrict__ op = lists_old + ell_base(so);
            for (int t = 0; t < nl && !ovf; t++) {
                const int jo = op[ell_off(t)];
                const uint32_t j = jo < nf ? inv[jo] : (uint32_t)jo;
                if (!in_block<T, D>(key_sorted[j], cc, g)) continue;   // left the block
                const uint32_t idj = E.id[j];
                while (a < na && E.id[arr[a]] < idj) {
                    if (cnt < kCap) lp[ell_off(cnt)] = (int32_t)arr[a];
                    cnt++;
                    a++;
                }
                if (cnt < kCap) lp[ell_off(cnt)] = (int32_t)j;
                cnt++;
            }
            for (; a < na; a++) {
                if (cnt < kCap) lp[ell_off(cnt)] = (int32_t)arr[a];
                cnt++;
            }
            if (ovf || cnt > kCap) need = true;
            else lcount_new[slot] = cnt;
        }
        if (need) {
            E.cell0[i] = kInvalidCell;
            lcount_new[slot] = 0;
        }
    }
    enqueue(E.queue, E.qcount, need, (uint32_t)i);
}

// ---------------------------------------------------------------------------
// per-sub-step list maintenance
// ---------------------------------------------------------------------------
// physics.py:526-529 KICK(half) then DRIFT(full) of one fluid particle
// (in registers); returns the new position
template <class T, int D>
__device__ __forceinline__ void kick_drift_one(vec4<T>& P4, vec4<T>& V4, const vec4<T>& A4,
                                               T half, T full)
{
    V4.x = RN<T>::add(V4.x, RN<T>::mul(half, A4.x));
    V4.y = RN<T>::add(V4.y, RN<T>::mul(half, A4.y));
    if (D == 3) V4.z = RN<T>::add(V4.z, RN<T>::mul(half, A4.z));
    P4.x = RN<T>::add(P4.x, RN<T>::mul(full, V4.x));
    P4.y = RN<T>::add(P4.y, RN<T>::mul(full, V4.y));
    if (D == 3) P4.z = RN<T>::add(P4.z, RN<T>::mul(full, V4.z));
}

// a drifted position back into the periodic box (no-op when bounded)
template <class T, int D>
__device__ __forceinline__ void wrap_position(vec4<T>& P4)
{
#if SPH_PERIODIC
    P4.x = wrap_coord<T>(P4.x, 0);
    P4.y = wrap_coord<T>(P4.y, 1);
    if (D == 3) P4.z = wrap_coord<T>(P4.z, 2);
#else
    (void)P4;
#endif
}

// skin-list bookkeeping of a drift xo -> xn: the path length bound (upward
// rounded |xn - xo| added to disp; xn unwrapped) and the list-cell check of
// the position xc (xn, wrapped into a periodic box); returns the bound
template <class T, int D>
__device__ __forceinline__ T drift_bookkeeping(const Eng<T>& E, const GridP<T>& g, int64_t i,
                                               const T (&xo)[3], const T (&xn)[3],
                                               const T (&xc)[3])
{
    T s2 = T(0);
#pragma unroll
    for (int k = 0; k < D; k++) {
        const T dk = RN<T>::mul_ru(fabs(RN<T>::sub(xn[k], xo[k])), RN<T>::kOnePlus2Eps);
        s2 = RN<T>::add_ru(s2, RN<T>::mul_ru(dk, dk));
    }
    const T dnew = RN<T>::add_ru(E.disp[i], RN<T>::sqrt_ru(s2));
    E.disp[i] = dnew;
    int c[3];
    if (cell_key_of<T, D>(xc, g, c) != E.cell0[i]) E.cell0[i] = kInvalidCell;
    return dnew;
}

// physics.py:526-529 KICK(half) then DRIFT(full), fluid only, plus the
// upward-rounded displacement bound and the list-cell check
template <class T, int D>
__global__ void __launch_bounds__(256)
k_kick_drift(Eng<T> E, int cv, int crp, GridP<T> g, T half, T full)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    T dnew = T(0);
    if (i >= E.n) {
    } else if (i >= E.nf || !is_owned(E, i)) {
        // walls and halo ghosts: only the continuity operand m/rho (physics.py:113)
        reinterpret_cast<T*>(&E.vel[cv][i])[3] = RN<T>::div(E.pos[i].w, E.rp[crp][i].x);
    } else {
        vec4<T> P4 = E.pos[i], V4 = E.vel[cv][i];
        const vec4<T> A4 = E.dvdt[i];
        // the continuity operand m_j/rho_j of this sub-step (physics.py:113):
        // a per-particle quotient, evaluated once here instead of per pair
        V4.w = RN<T>::div(P4.w, E.rp[crp][i].x);
        const T xo[3] = {P4.x, P4.y, P4.z};
        kick_drift_one<T, D>(P4, V4, A4, half, full);
        const T xn[3] = {P4.x, P4.y, P4.z};
        wrap_position<T, D>(P4);
        E.vel[cv][i] = V4;
        E.pos[i] = P4;
        const T xc[3] = {P4.x, P4.y, P4.z};
        dnew = drift_bookkeeping<T, D>(E, g, i, xo, xn, xc);
        note_disp(E, i, dnew);
    }
    const unsigned long long b = warp_max_u64(dbits(double(dnew)));
    if (lane_id() == 0 && b) atomicMax(&E.stats->dmax_bits, b);
}

// exact filter of every valid skin list on current positions -> exact lists and
// accepted counts; particles whose list is not valid go to the fix queue
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads, SPH_MASK_MINB)
k_mask(Eng<T> E, GridP<T> g, T s_eff)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool need = false;
    if (i < E.n) {
        const int64_t slot = slot_of(E, i);
        const T dmax = T(__longlong_as_double((long long)E.stats->dmax_bits));
        const uint32_t c0 = E.cell0[i];
        if (c0 == kInvalidCell) {
            need = true;
        } else if (RN<T>::add_ru(RN<T>::sub_ru(E.disp[i], E.disp0[i]), dmax_for(E, c0, dmax)) >
                   s_eff) {
            E.cell0[i] = kInvalidCell;
            need = true;
            atomicAdd(&E.stats->ndisp, 1u);
        } else {
            T xi[3];
            to3<T>(E.pos[i], xi);
            const int nl = E.lcount[slot];
            int acc = 0;
            const int4* q4 = reinterpret_cast<const int4*>(E.lists + ell_base(slot));
            int32_t* ep = E.elist + ell_base(slot);
            // one quad of list entries + 4 positions in flight per trip
            for (int u0 = 0; u0 < nl; u0 += 4) {
                const int4 q = ld_list(q4 + (u0 >> 2) * 32);
                const int jj[4] = {q.x, u0 + 1 < nl ? q.y : -1, u0 + 2 < nl ? q.z : -1,
                                   u0 + 3 < nl ? q.w : -1};
                vec4<T> pj[4];
#pragma unroll
                for (int k = 0; k < 4; k++) pj[k] = E.pos[jj[k] >= 0 ? jj[k] : 0];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    T xj[3];
                    to3<T>(pj[k], xj);
                    const T r2 = accept_r2<T, D>(xi, xj);
                    if (jj[k] >= 0 && (r2 < g.c2) && (r2 > T(0))) ep[ell_off(acc++)] = jj[k];
                }
            }
            const int total = acc + (i >= E.nf ? E.nww[slot] : 0);
            E.acount[slot] = total > kCap ? -1 : acc;
        }
    }
    enqueue(E.queue, E.qcount, need, (uint32_t)i);
}

// list validity after a drift: particles whose skin list is no longer valid
// (cell changed, or disp_i + max disp > skin) are queued for exact rebuilds
template <class T>
__global__ void __launch_bounds__(256)
k_mark(Eng<T> E, T s_eff)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    // 4 consecutive particles per thread (vector loads)
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    const T dmax = T(__longlong_as_double((long long)E.stats->dmax_bits));
    uint32_t c4[4] = {0, 0, 0, 0};
    T d4[4] = {0, 0, 0, 0}, e4[4] = {0, 0, 0, 0};
    if (sizeof(T) == 4 && i0 + 3 < E.n) {
        const uint4 c = *reinterpret_cast<const uint4*>(E.cell0 + i0);
        const float4 d = *reinterpret_cast<const float4*>(E.disp + i0);
        const float4 z = *reinterpret_cast<const float4*>(E.disp0 + i0);
        c4[0] = c.x; c4[1] = c.y; c4[2] = c.z; c4[3] = c.w;
        d4[0] = d.x; d4[1] = d.y; d4[2] = d.z; d4[3] = d.w;
        e4[0] = z.x; e4[1] = z.y; e4[2] = z.z; e4[3] = z.w;
    } else {
#pragma unroll
        for (int r = 0; r < 4; r++)
            if (i0 + r < E.n) {
                c4[r] = E.cell0[i0 + r];
                d4[r] = E.disp[i0 + r];
                e4[r] = E.disp0[i0 + r];
            }
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int64_t i = i0 + r;
        bool need = false;
        if (i < E.n) {
            if (c4[r] == kInvalidCell) {
                need = true;
            } else if (RN<T>::add_ru(RN<T>::sub_ru(d4[r], e4[r]), dmax_for(E, c4[r], dmax)) >
                       s_eff) {
                E.cell0[i] = kInvalidCell;
                need = true;
                atomicAdd(&E.stats->ndisp, 1u);
            }
        }
        enqueue(E.queue, E.qcount, need, (uint32_t)i);
    }
}

// List refresh of the queued particles (cell changed, or own displacement
// + the largest displacement past the skin), one warp each: the skin list
// of the CURRENT cell's block within cutoff + skin (neighborhood.py:176-227
// with the skin radius, ascending id), re-based at the current displacement
// so it stays valid for the rest of the step, plus this sub-step's exact list
// (its 0 < r2 < c^2 subset, same order).  A particle whose skin candidates
// exceed the capacity gets the exact list only and stays queued.
template <class T, int D>
__device__ __forceinline__ void refresh_one(const EngAcc<T>& acc, const GridP<T>& g,
                                            const Eng<T>& E, T cs2, int64_t i, WarpBuf& sb,
                                            uint32_t* srt, unsigned lane, unsigned lt)
{
    const int64_t slot = slot_of(E, i);
    const bool fluid = i < E.nf;
    T xi[3];
    acc.position(i, xi);
    CollectCounts cc = warp_collect<T, D, true>(acc, g, i, xi, cs2, fluid ? 3u : 1u, sb);
    if (cc.stored <= kCap) {
        warp_emit_sorted(sb, cc.stored, lane, [&](int pos, uint32_t j) {
            E.lists[ell_index(slot, pos)] = (int32_t)j;
            srt[pos] = j;
        });
        // the exact subset in list order
        int ex = 0;
        for (int b = 0; b < cc.stored; b += 32) {
            const int k = b + (int)lane;
            bool ok = false;
            uint32_t j = 0;
            if (k < cc.stored) {
                j = srt[k];
                T xj[3];
                acc.position(j, xj);
                const T r2 = accept_r2<T, D>(xi, xj);
                ok = (r2 < g.c2) && (r2 > T(0));
            }
            const unsigned bl = __ballot_sync(0xffffffffu, ok);
            if (ok) E.elist[ell_index(slot, ex + __popc(bl & lt))] = (int32_t)j;
            ex += __popc(bl);
        }
        // walls: wall-wall neighbours count toward the capacity (nww)
        const int total = ex + (fluid ? 0 : cc.accepted);
        if (lane == 0) {
            int cxyz[3];
            E.acount[slot] = total > kCap ? -1 : ex;
            E.cell0[i] = cell_key_of<T, D>(xi, g, cxyz);
            E.lcount[slot] = cc.stored;
            E.nww[slot] = cc.accepted;
            E.disp0[i] = E.disp[i];
        }
    } else {   // skin list over capacity: this sub-step's exact list only
        __syncwarp();
        CollectCounts ce = warp_collect<T, D, false>(acc, g, i, xi, T(0), fluid ? 3u : 1u,
                                                     sb);
        if (ce.accepted > kCap) {
            if (lane == 0) E.acount[slot] = -1;
        } else {
            warp_emit_sorted(sb, ce.stored, lane, [&](int pos, uint32_t j) {
                E.elist[ell_index(slot, pos)] = (int32_t)j;
            });
            if (lane == 0) E.acount[slot] = ce.stored;
        }
        if (lane == 0) E.cell0[i] = kInvalidCell;
    }
    if (lane == 0) atomicAdd(&E.stats->nfix, 1u);
    __syncwarp();
}

template <class T, int D>
__global__ void __launch_bounds__(kNlThreads, SPH_FIX_MINB)
k_fix_build(const EngAcc<T> acc, const GridP<T> g, Eng<T> E, T cs2)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    __shared__ WarpBuf bufs[kNlWarps];
    __shared__ uint32_t sorted[kNlWarps][kCap];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const uint32_t qn = *(volatile uint32_t*)E.qcount;
    for (uint32_t q = blockIdx.x * kNlWarps + warp; q < qn; q += gridDim.x * kNlWarps)
        refresh_one<T, D>(acc, g, E, cs2, (int64_t)E.queue[q], bufs[warp], sorted[warp], lane,
                          lt);
}

// The sub-step's list check and refresh in one pass (no queue): each warp
// tests 32 consecutive particles (k_mark's criterion) and refreshes the
// ones it finds invalid itself, so scattered refreshes spread over all warps.
template <class T, int D>
__global__ void __launch_bounds__(kNlThreads, 4)
k_mark_refresh(const EngAcc<T> acc, const GridP<T> g, Eng<T> E, T cs2, T s_eff)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    __shared__ WarpBuf bufs[kNlWarps];
    __shared__ uint32_t sorted[kNlWarps][kCap];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const T dmax = T(__longlong_as_double((long long)E.stats->dmax_bits));
    // 4 consecutive particles per lane (vector loads), 128 per warp trip
    for (int64_t base = ((int64_t)blockIdx.x * kNlWarps + warp) * 128; base < E.n;
         base += (int64_t)gridDim.x * kNlWarps * 128) {
        const int64_t i0 = base + 4 * lane;
        uint32_t c4[4] = {0, 0, 0, 0};
        T d4[4] = {0, 0, 0, 0}, e4[4] = {0, 0, 0, 0};
        if (sizeof(T) == 4 && i0 + 3 < E.n) {
            const uint4 c = *reinterpret_cast<const uint4*>(E.cell0 + i0);
            const float4 d = *reinterpret_cast<const float4*>(E.disp + i0);
            const float4 z = *reinterpret_cast<const float4*>(E.disp0 + i0);
            c4[0] = c.x; c4[1] = c.y; c4[2] = c.z; c4[3] = c.w;
            d4[0] = d.x; d4[1] = d.y; d4[2] = d.z; d4[3] = d.w;
            e4[0] = z.x; e4[1] = z.y; e4[2] = z.z; e4[3] = z.w;
        } else {
#pragma unroll
            for (int r = 0; r < 4; r++)
                if (i0 + r < E.n) {
                    c4[r] = E.cell0[i0 + r];
                    d4[r] = E.disp[i0 + r];
                    e4[r] = E.disp0[i0 + r];
                }
        }
        unsigned bits = 0;
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int64_t i = i0 + r;
            if (i >= E.n) continue;
            if (c4[r] == kInvalidCell) {
                bits |= 1u << r;
            } else if (RN<T>::add_ru(RN<T>::sub_ru(d4[r], e4[r]), dmax_for(E, c4[r], dmax)) >
                       s_eff) {
                E.cell0[i] = kInvalidCell;
                bits |= 1u << r;
                atomicAdd(&E.stats->ndisp, 1u);
            }
        }
        unsigned m = __ballot_sync(0xffffffffu, bits != 0);
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const unsigned bl = __shfl_sync(0xffffffffu, bits, l);
#pragma unroll
            for (int r = 0; r < 4; r++)
                if ((bl >> r) & 1u)
                    refresh_one<T, D>(acc, g, E, cs2, base + 4 * l + r, bufs[warp],
                                      sorted[warp], lane, lt);
        }
    }
}

// ---------------------------------------------------------------------------
// sweeps (thread per particle, ascending-id accumulation)
// ---------------------------------------------------------------------------
// neighborhood.py:200-202 / physics.py:357-360 (owned particles only)
template <class T>
__device__ __forceinline__ void flag_overflow(const Eng<T>& E, int64_t i)
{
    if (!is_owned(E, i)) return;
    E.oflow_id[E.id[i]] = 1;
    atomicAdd(&E.stats->overflow, 1u);
}

// physics.py:94-119 CONTINUITY fused with :268-274 DENSITY_UPDATE(full),
// fluid only: reads rho of the current buffer, writes (rho, p) to the other.
// A particle with a valid skin list filters it here (writing the exact list
// the momentum sweep reuses); others read the exact list k_fix_build made.
template <class T, int D, bool EXACT>
__global__ void __launch_bounds__(kSweepThreads, EXACT ? SPH_CONT_EXACT_MINB : SPH_CONT_MINB)
k_cont_du(Eng<T> E, PhysT<T> P, GridP<T> g, int cv, int crp, T full)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.nf) return;
    const vec4<T>* __restrict__ pos = E.pos;
    const vec4<T>* __restrict__ vel = E.vel[cv];
    const vec2<T>* __restrict__ rp = E.rp[crp];
    T xi[3], vi[3];
    to3<T>(pos[i], xi);
    to3<T>(vel[i], vi);
    const T rho_i = rp[i].x;
    double acc = double(RN<T>::sub(rho_i, rho_i));
    auto loadf = [&](int j) { return NbrPV<T>{pos[j], vel[j]}; };
    auto pair = [&](int, const NbrPV<T>& nb) {
        T xj[3], vj[3], dx[3], r2, vx;
        to3<T>(nb.p, xj);
        to3<T>(nb.v, vj);
        pair_geometry<T, D>(xi, xj, vi, vj, r2, vx, dx);
        acc = dadd(acc, continuity_term<T>(r2, vx, nb.v.w, P));   // v.w = m_j/rho_j
    };
    int cnt;
    if (EXACT || E.cell0[i] == kInvalidCell) {   // exact list from k_mask / k_fix_build
        cnt = E.acount[i];
        if (cnt < 0) { flag_overflow(E, i); return; }
        sweep_list<T>(E, i, cnt, loadf, pair);
    } else {
        // the exact list, also stored a full int4 quad at a time
        int4* __restrict__ eq = reinterpret_cast<int4*>(E.elist + ell_base(i));
        int e0 = 0, e1 = 0, e2 = 0;
        cnt = 0;
        int32_t* __restrict__ ep = E.elist + ell_base(i);
        auto store = [&](int j) {
            if (SPH_ELIST_SCALAR) {   // one 4-byte store per entry
                if (cnt < kCap) ep[ell_off(cnt)] = j;
            } else {
                const int r = cnt & 3;
                if (r == 0) e0 = j;
                else if (r == 1) e1 = j;
                else if (r == 2) e2 = j;
                else if (cnt < kCap) st_list(eq + (cnt >> 2) * 32, make_int4(e0, e1, e2, j));
            }
            cnt++;
        };
        if (SPH_CONT_FILTER_QUADS) {
            filter_quads<T, D>(E, i, xi, g.c2, E.lcount[i], [&](int j, const vec4<T>& pj) {
                store(j);
                pair(cnt, NbrPV<T>{pj, vel[j]});
            });
        } else {
            filter_walk<T, D>(E, i, xi, g.c2, E.lcount[i], loadf,
                              [&](int j, const NbrPV<T>& nb) {
                store(j);
                pair(cnt, nb);
            });
        }
        if (!SPH_ELIST_SCALAR && (cnt & 3) && cnt < kCap) st_list(eq + (cnt >> 2) * 32, make_int4(e0, e1, e2, 0));
        if (cnt > kCap) {
            E.acount[i] = -1;
            flag_overflow(E, i);
            return;
        }
        E.acount[i] = cnt;
    }
    const T dr = RN<T>::from_d(dmul(double(rho_i), acc));
    E.drho[i] = dr;
    vec2<T> out;
    out.x = RN<T>::add(rho_i, RN<T>::mul(full, dr));
    out.y = RN<T>::mul(P.c0c0, RN<T>::sub(out.x, P.rho0));
    E.rp[crp ^ 1][i] = out;
    E.rq[i] = rq_of<T>(out);
}

// physics.py:161-194 WALL_PRESSURE over the wall segment: fluid p from
// buffer b, walls' (rho, p) written into the same buffer.  zero_drho mirrors
// the continuity body's drho = 0 for walls (physics.py:99-101) in a sub-step.
// filter != 0: valid skin lists are filtered here (walls' exact lists are
// used by no other sweep, so they are not stored).
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads, SPH_SWEEP_MINB)
k_wall(Eng<T> E, PhysT<T> P, GridP<T> g, int b, int zero_drho, int count_factor, int filter,
       int cvn)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long visits_sum = 0;
    if (t < E.nw) {
        const int64_t i = E.nf + t;
        const int64_t slot = E.nf_pad + t;
            vec2<T>* __restrict__ rp = E.rp[b];
        T xi[3];
        to3<T>(E.pos[i], xi);
        const T rho_i = rp[i].x;
        double num = double(RN<T>::sub(rho_i, rho_i));
        double den = num;
        auto loadf = [&](int j) { return NbrPR<T>{E.pos[j], rp[j]}; };
        auto pair = [&](int, const NbrPR<T>& nb) {
            T xj[3];
            to3<T>(nb.p, xj);
            const double w = wall_weight<T>(pair_r2<T, D>(xi, xj), P);
            num = dadd(num, dmul(double(nb.rp.y), w));
            den = dadd(den, w);
        };
        int acnt;
        if (!filter || E.cell0[i] == kInvalidCell) {
            acnt = E.acount[slot];
            if (acnt >= 0) sweep_list<T>(E, slot, acnt, loadf, pair);
        } else {
            acnt = 0;
            filter_walk<T, D>(E, slot, xi, g.c2, E.lcount[slot], loadf,
                              [&](int, const NbrPR<T>& nb) { pair(acnt++, nb); });
            if (acnt + E.nww[slot] > kCap) acnt = -1;
            E.acount[slot] = acnt;
        }
        if (acnt < 0) {
            flag_overflow(E, i);
        } else {
            vec2<T> out;
            out.y = den > 0.0 ? RN<T>::from_d(ddiv(num, den)) : T(0);
            out.x = RN<T>::add(P.rho0, RN<T>::div(out.y, P.c0c0));
            rp[i] = out;
            E.rq[i] = rq_of<T>(out);
            // the next sub-step's continuity operand m/rho, in the velocity
            // buffer current then (walls never move: both buffers agree)
            if (cvn >= 0) reinterpret_cast<T*>(&E.vel[cvn][i])[3] = RN<T>::div(E.pos[i].w, out.x);
            E.nnb[i] = (uint32_t)acnt;
            if (zero_drho) E.drho[i] = T(0);
            if (is_owned(E, i))
                visits_sum = (unsigned long long)acnt * (unsigned long long)count_factor;
        }
    }
    add_interactions(E.stats, visits_sum);
}

// WALL_PRESSURE with G lanes per wall: lane q evaluates list entries
// q, q + G, ... (gather, exact test, Shepard weight and p_j * w -- the
// expensive part), then every lane of the group adds the G terms in list
// order (shuffles), so the binary64 sums follow the reference's order bit
// for bit.  A thread per wall leaves most SMs idle (a few tens of thousands
// of walls, each a serial chain of dependent gathers).
#ifndef SPH_WALL_LANES   // 2D: 8 (wall pressure 14 -> 12 us per sub-step); 3D: most
#define SPH_WALL_LANES (D == 2 ? 8 : 1)   // walls have no fluid neighbour (G=8: 3x slower)
#endif
template <class T, int D, int G>
__global__ void __launch_bounds__(kSweepThreads)
k_wall_g(Eng<T> E, PhysT<T> P, GridP<T> g, int b, int zero_drho, int count_factor, int filter,
         int cvn)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const unsigned lane = lane_id(), q = lane & (G - 1);
    const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane & ~(G - 1));
    unsigned long long visits_sum = 0;
    if (gid < E.nw) {   // uniform across the group
        const int64_t i = E.nf + gid;
        const int64_t slot = E.nf_pad + gid;
        vec2<T>* __restrict__ rp = E.rp[b];
        T xi[3];
        to3<T>(E.pos[i], xi);
        const T rho_i = rp[i].x;
        double num = double(RN<T>::sub(rho_i, rho_i));
        double den = num;
        const bool exact = !filter || E.cell0[i] == kInvalidCell;
        const int nl = exact ? E.acount[slot] : E.lcount[slot];
        const int32_t* __restrict__ lp = (exact ? E.elist : E.lists) + ell_base(slot);
        int acnt = exact ? nl : 0;
        for (int base = 0; base < nl; base += G) {
            const int e = base + (int)q;
            bool ok = false;
            double tn = 0.0, tw = 0.0;
            if (e < nl) {
                const int j = lp[ell_off(e)];
                const vec4<T> pj = E.pos[j];
                T xj[3];
                to3<T>(pj, xj);
                const T r2 = pair_r2<T, D>(xi, xj);
                ok = exact || ((r2 < g.c2) && (r2 > T(0)));
                if (ok) {
                    tw = wall_weight<T>(r2, P);
                    tn = dmul(double(rp[j].y), tw);
                }
            }
            const unsigned okm = __ballot_sync(gmask, ok) >> (lane & ~(G - 1));
#pragma unroll
            for (int k = 0; k < G; k++) {
                const double an = __shfl_sync(gmask, tn, k, G);
                const double aw = __shfl_sync(gmask, tw, k, G);
                if ((okm >> k) & 1u) {
                    num = dadd(num, an);
                    den = dadd(den, aw);
                }
            }
            if (!exact) acnt += __popc(okm);
        }
        if (!exact && acnt + E.nww[slot] > kCap) acnt = -1;
        if (q == 0) {
            if (!exact) E.acount[slot] = acnt;
            if (acnt < 0) {
                flag_overflow(E, i);
            } else {
                vec2<T> out;
                out.y = den > 0.0 ? RN<T>::from_d(ddiv(num, den)) : T(0);
                out.x = RN<T>::add(P.rho0, RN<T>::div(out.y, P.c0c0));
                rp[i] = out;
                E.rq[i] = rq_of<T>(out);
                if (cvn >= 0)
                    reinterpret_cast<T*>(&E.vel[cvn][i])[3] = RN<T>::div(E.pos[i].w, out.x);
                E.nnb[i] = (uint32_t)acnt;
                if (zero_drho) E.drho[i] = T(0);
                if (is_owned(E, i))
                    visits_sum = (unsigned long long)acnt * (unsigned long long)count_factor;
            }
        }
    }
    add_interactions(E.stats, visits_sum);
}

// physics.py:122-158 MOMENTUM (+ :546-547 KICK(half) into the other velocity
// buffer when kick != 0), fluid only; rho/p from buffer brp.
//
// fuse != 0 (every sub-step of a step but the last): the next sub-step's
// KICK(half) + DRIFT(full) with the same dvdt follow here -- positions into
// the other buffer, m/rho for its continuity sweep, the skin-list
// bookkeeping -- so that sub-step starts at its list maintenance.
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads, SPH_MOM_MINB)
k_mom(Eng<T> E, PhysT<T> P, int cv, int brp, int kick, T half, int count_factor, GridP<T> g,
      int fuse, T full)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long csum = 0;
    T dnew = T(0);
    if (i < E.nf) {
        const int acnt = E.acount[i];
        if (acnt < 0) {
            flag_overflow(E, i);
        } else {
                    const vec4<T>* __restrict__ pos = E.pos;
            const vec4<T>* __restrict__ vel = E.vel[cv];
            const vec2<T>* __restrict__ rq = E.rq;   // (rho, p/rho^2) of buffer brp
            T xi[3], vi[3];
            to3<T>(pos[i], xi);
            const vec4<T> VI = vel[i];
            to3<T>(VI, vi);
            const vec2<T> RQI = rq[i];
            const T rho_i = RQI.x;
            const T pi_rr = RQI.y;
            DvAcc<T> a;
            a.init(P.g);
            auto loadf = [&](int j) { return NbrPVR<T>{pos[j], vel[j], rq[j]}; };
            constexpr bool kIlp = SPH_MOM_ILP && (SPH_MOM_ILP > 1 || D == 2);
            if (kIlp) {
            // two pairs per basic block: their terms are independent chains the
            // scheduler interleaves; accumulation stays in list order
            auto terms = [&](const NbrPVR<T>& nb, double (&t)[3]) {
                T xj[3], vj[3], dx[3], r2, vx;
                to3<T>(nb.p, xj);
                to3<T>(nb.v, vj);
                pair_geometry<T, D>(xi, xj, vi, vj, r2, vx, dx);
                momentum_terms<T, D>(r2, vx, dx, rho_i, pi_rr, nb.rp.x, nb.rp.y, nb.p.w, P, t);
            };
            if (acnt > 0) {
                const int4* __restrict__ q4 = reinterpret_cast<const int4*>(E.elist + ell_base(i));
                int4 qn = ld_list(q4);
                for (int t0 = 0; t0 < acnt; t0 += 4) {
                    const int4 q = qn;
                    if (t0 + 4 < acnt) qn = ld_list(q4 + ((t0 >> 2) + 1) * 32);
                    {
                        const bool hb = t0 + 1 < acnt;
                        const NbrPVR<T> na = loadf(q.x), nb = loadf(hb ? q.y : q.x);
                        double ta[3], tb[3];
                        terms(na, ta);
                        terms(nb, tb);
                        momentum_accumulate<T, D>(ta, a);
                        if (hb) momentum_accumulate<T, D>(tb, a);
                    }
                    if (t0 + 2 < acnt) {
                        const bool hb = t0 + 3 < acnt;
                        const NbrPVR<T> na = loadf(q.z), nb = loadf(hb ? q.w : q.z);
                        double ta[3], tb[3];
                        terms(na, ta);
                        terms(nb, tb);
                        momentum_accumulate<T, D>(ta, a);
                        if (hb) momentum_accumulate<T, D>(tb, a);
                    }
                }
            }
            } else {
            sweep_list<T>(E, i, acnt, loadf, [&](int, const NbrPVR<T>& nb) {
                T xj[3], vj[3], dx[3], r2, vx;
                to3<T>(nb.p, xj);
                to3<T>(nb.v, vj);
                pair_geometry<T, D>(xi, xj, vi, vj, r2, vx, dx);
                momentum_pair<T, D>(r2, vx, dx, rho_i, pi_rr, nb.rp.x, nb.rp.y, nb.p.w, P, a);
            });
            }
            vec4<T> A4;
            A4.x = a.out(0); A4.y = a.out(1); A4.z = D == 3 ? a.out(2) : T(0); A4.w = T(0);
            E.dvdt[i] = A4;
            E.nnb[i] = (uint32_t)acnt;
            if (kick) {
                vec4<T> V4 = VI;
                V4.x = RN<T>::add(V4.x, RN<T>::mul(half, A4.x));
                V4.y = RN<T>::add(V4.y, RN<T>::mul(half, A4.y));
                if (D == 3) V4.z = RN<T>::add(V4.z, RN<T>::mul(half, A4.z));
                if (fuse && is_owned(E, i)) {   // ghosts: the XV refresh brings them
                    vec4<T> P4 = pos[i];
                    const T xo[3] = {P4.x, P4.y, P4.z};
                    kick_drift_one<T, D>(P4, V4, A4, half, full);
                    V4.w = RN<T>::div(P4.w, rho_i);   // rho after this sub-step's DU
                    const T xn[3] = {P4.x, P4.y, P4.z};
                    wrap_position<T, D>(P4);
                    E.pos_next[i] = P4;
                    const T xc[3] = {P4.x, P4.y, P4.z};
                    dnew = drift_bookkeeping<T, D>(E, g, i, xo, xn, xc);
                    note_disp(E, i, dnew);
                }
                E.vel[cv ^ 1][i] = V4;
            }
            if (is_owned(E, i)) csum = (unsigned long long)acnt * (unsigned long long)count_factor;
        }
    }
    add_interactions(E.stats, csum);
    if (fuse) {
        const unsigned long long b = warp_max_u64(dbits(double(dnew)));
        if (lane_id() == 0 && b) atomicMax(&E.stats->dmax_bits, b);
    }
}

// physics.py:220-247 SHEPARD + :277-280 COPY_SCALAR + :268-274
// DENSITY_UPDATE(dt=0), all particles; reads buffer crp, writes crp^1.
template <class T, int D>
__global__ void __launch_bounds__(kSweepThreads, SPH_SWEEP_MINB)
k_shepard(Eng<T> E, PhysT<T> P, int crp)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= E.n) return;
    const vec2<T>* __restrict__ rp = E.rp[crp];
    const vec2<T> RPI = rp[i];
    const uint32_t pid = E.id[i];
    if (i >= E.nf) {   // walls: rho_new = rho; density update skips walls
        E.rho_scratch_id[pid] = RPI.x;
        E.rp[crp ^ 1][i] = RPI;
        return;
    }
    T rho_new = RPI.x;
    if (E.acount[i] >= 0) {
        T xi[3];
        const vec4<T> PI = E.pos[i];
        to3<T>(PI, xi);
        const T m_i = PI.w;
        double num = double(RN<T>::mul(m_i, P.alpha_d));
        double den = double(RN<T>::mul(RN<T>::div(m_i, RPI.x), P.alpha_d));
        sweep_list<T>(E, i, E.acount[i],
            [&](int j) { return NbrPR<T>{E.pos[j], rp[j]}; },
            [&](int, const NbrPR<T>& nb) {
                T xj[3];
                to3<T>(nb.p, xj);
                const double w = wall_weight<T>(pair_r2<T, D>(xi, xj), P);
                num = dadd(num, dmul(double(nb.p.w), w));
                den = dadd(den, dmul(double(RN<T>::div(nb.p.w, nb.rp.x)), w));
            });
        rho_new = RN<T>::from_d(ddiv(num, den));
    }
    E.rho_scratch_id[pid] = rho_new;
    vec2<T> out;
    out.x = RN<T>::add(rho_new, RN<T>::mul(T(0), E.drho[i]));
    out.y = RN<T>::mul(P.c0c0, RN<T>::sub(out.x, P.rho0));
    E.rp[crp ^ 1][i] = out;
}

}  // namespace sph

using namespace sph;

// ---------------------------------------------------------------------------
// orchestration
// ---------------------------------------------------------------------------
template <class T>
static T skin_cs2(const SphEngine* e)
{
#if SPH_PERIODIC
    const T cs = T((e->cutoff + e->skin) * (1.0 + 1e-4));   // tile_image margin
#else
    const T cs = T(e->cutoff + e->skin);
#endif
    return cs * cs;
}

// validity threshold of a skin list: disp_i + max_j disp_j <= s_eff, with a
// margin far above the binary32 rounding of r2 (~1e-7 relative)
template <class T>
static T skin_eff(const SphEngine* e)
{
    const double s = e->skin * (1.0 - 1e-4) - 1e-5 * (e->cutoff + e->skin);
    return s > 0.0 ? T(s) : T(0);
}

template <class T, int D>
static int build_lists_impl(SphEngine* e, double skin, cudaStream_t s)
{
    e->skin = skin > 0.0 ? skin : 0.0;
    cudaMemsetAsync(&e->stats->dmax_bits, 0, sizeof(unsigned long long), s);
    if (e->cellmax && e->blockmax) {   // fresh lists: every path length is 0
        cudaMemsetAsync(e->cellmax, 0, sizeof(uint32_t) * (size_t)e->ncells, s);
        cudaMemsetAsync(e->blockmax, 0, sizeof(uint32_t) * (size_t)e->ncells, s);
    }
    GridP<T> g = grid_of_engine<T>(e);
    EngAcc<T> acc = acc_of_engine<T>(e);
    Eng<T> E = eng_of<T>(e);
    const T cs2 = skin_cs2<T>(e);
    // walls' static wall-wall counts: computed by the first build after a push
    const int wall_pairs = (SPH_SKIN_WALL_SKIP && e->nww_ready) ? 0 : 1;
    if (e->n > 0) {
        constexpr int NT = SkinTile<T, D>::kThreads;
        const int64_t want = e->ncells < e->n ? e->ncells : e->n;
        const unsigned blocks = (unsigned)(want < 148 * 16 ? want : 148 * 16);
        cudaMemsetAsync(e->qcount, 0, sizeof(uint32_t), s);
        // physical index of every id (workspace scratch, free between rebuilds)
        Bump bump(e->ws, e->ws_bytes);
        uint32_t* phys_of_id = bump.take<uint32_t>(e->id_range > e->n ? e->id_range : e->n);
        uint32_t* cells = bump.take<uint32_t>(e->n);   // nonempty cells <= n
        uint32_t* big = bump.take<uint32_t>(e->n);     // cells with > 128 candidates
        uint32_t* counts = bump.take<uint32_t>(4);   // nonempty, big, tile / warp work counters
        if (!counts) return SPH_ERR_WORKSPACE;
        note_launch(), k_phys_of_id<<<grid_for(e->n, 256), 256, 0, s>>>(e->id, e->n, phys_of_id);
        cudaMemsetAsync(counts, 0, 4 * sizeof(uint32_t), s);
        note_launch(), k_nonempty_cells<<<grid_for(e->ncells, 256), 256, 0, s>>>(
            e->offs_f, e->offs_w, e->ncells, cells, counts);
        if (D == 2) {   // 2D blocks hold ~60 candidates: a warp per cell
            const int64_t wb = (want + 7) / 8;
            note_launch(), k_skin_warp<T, D><<<(unsigned)(wb < 148 * 8 ? wb : 148 * 8), 256, 0,
                                               s>>>(g, cs2, E, cells, counts, phys_of_id, big,
                                                    counts + 1, SPH_LIST_FRESH ? e->cll_fresh : 0,
                                                    counts + 3);
            note_launch(), k_skin_tile<T, D><<<blocks, NT, 0, s>>>(acc, g, cs2, E, big,
                                                                  counts + 1, phys_of_id, 1,
                                                                  SPH_LIST_FRESH ? e->cll_fresh : 0,
                                                                  counts + 2);
        } else {        // 3D blocks hold ~450: a thread block per cell
            note_launch(), k_skin_tile<T, D><<<blocks, NT, 0, s>>>(acc, g, cs2, E, cells, counts,
                                                                  phys_of_id, wall_pairs,
                                                                  SPH_LIST_FRESH ? e->cll_fresh : 0,
                                                                  counts + 2);
        }
        note_launch(), k_skin_big<T, D><<<148 * 2, kNlThreads, 0, s>>>(acc, g, cs2, E);
    }
    e->lists_ready = 1;
    e->nww_ready = 1;
    return check_launch("engine_build_lists");
}

extern "C" int sph_engine_build_lists(SphEngine* e, double skin, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc) return rc;
    return SPH_DISPATCH(e, build_lists_impl, e, skin, s);
}

template <class T, int D> static void launch_fix(const SphEngine* e, cudaStream_t s);

template <class T, int D>
static int maintain_impl(SphEngine* e, cudaStream_t s)
{
    if (!e->key_sorted || !e->key_prev || !e->perm || !e->inv || !e->lists_alt ||
        !e->lcount_alt) {
        set_error("engine_maintain_lists: the persistent-list arrays are not set");
        return SPH_ERR_INVALID;
    }
    if (!e->lists_stale) {
        set_error("engine_maintain_lists: no valid lists before the CLL rebuild");
        return SPH_ERR_INVALID;
    }
    const int64_t nc = e->ncells + 1, nf = e->nf;
    Bump bump(e->ws, e->ws_bytes);
    uint32_t* ccount = bump.take<uint32_t>(nc);
    uint32_t* moff = bump.take<uint32_t>(nc);
    uint32_t* cursor = bump.take<uint32_t>(nc);
    uint32_t* movers = bump.take<uint32_t>(nf > 0 ? nf : 1);
    void* scr = bump.take<char>(scan_scratch_bytes(nc));
    if (!scr) return SPH_ERR_WORKSPACE;
    // arrivals by cell (CSR over the movers' new cells)
    cudaMemsetAsync(ccount, 0, sizeof(uint32_t) * (size_t)nc, s);
    if (nf > 0)
        note_launch(), k_mover_count<<<grid_for(nf, 256), 256, 0, s>>>(e->key_sorted,
                                                                       e->key_prev, nf, ccount);
    int rc = exclusive_scan_u32(ccount, moff, nc, scr, s);
    if (rc) return rc;
    cudaMemcpyAsync(cursor, moff, sizeof(uint32_t) * (size_t)nc, cudaMemcpyDeviceToDevice, s);
    if (nf > 0)
        note_launch(), k_mover_fill<<<grid_for(nf, 256), 256, 0, s>>>(e->key_sorted,
                                                                      e->key_prev, nf, cursor,
                                                                      movers);
    if (sizeof(T) == 4 && e->cellmax && e->blockmax) {   // local bounds of the carried lists
        cudaMemsetAsync(e->cellmax, 0, sizeof(uint32_t) * (size_t)e->ncells, s);
        if (nf > 0)
            note_launch(), k_cellmax_seed<<<grid_for(nf, 256), 256, 0, s>>>(
                e->key_sorted, (const float*)e->disp, nf, e->cellmax);
        launch_blockmax<T, D>(e, s);
    }
    cudaMemsetAsync(e->qcount, 0, sizeof(uint32_t), s);
    if (e->n > 0)
        note_launch(), k_maintain<T, D><<<grid_for(e->n, 128), 128, 0, s>>>(
            eng_of<T>(e), grid_of_engine<T>(e), skin_cs2<T>(e), skin_eff<T>(e), e->key_sorted,
            e->key_prev, e->perm, e->inv, e->lists, e->lcount, e->lists_alt, e->lcount_alt,
            moff, movers);
    int32_t* t = e->lists; e->lists = e->lists_alt; e->lists_alt = t;
    t = e->lcount; e->lcount = e->lcount_alt; e->lcount_alt = t;
    if (e->n > 0) launch_fix<T, D>(e, s);   // fresh lists for the queued particles
    e->lists_ready = 1;
    e->lists_stale = 0;
    return check_launch("engine_maintain_lists");
}

extern "C" int sph_engine_maintain_lists(SphEngine* e, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc) return rc;
    return SPH_DISPATCH(e, maintain_impl, e, s);
}

// programmatic dependent launch for the sub-step kernels (common.cuh): 2D
// only, and not on slab ranks, whose sub-steps interleave NCCL kernels
static inline bool pdl_for(const SphEngine* e) { return e->dim == 2 && !e->owned_id; }

template <class T, int D>
static void launch_fix(const SphEngine* e, cudaStream_t s)
{
    GridP<T> g = grid_of_engine<T>(e);
    Eng<T> E = eng_of<T>(e);
    EngAcc<T> acc = acc_of_engine<T>(e);
    const int64_t want = (e->n + kNlWarps - 1) / kNlWarps;
    const int blocks = (int)(want < 148 * 8 ? want : 148 * 8);
    launch_pdl(pdl_for(e), k_fix_build<T, D>, blocks, kNlThreads, s, acc, g, E, skin_cs2<T>(e));
}

// exact lists for every particle: filtered skin lists (k_mask), exact
// rebuilds for the rest (initialize / Shepard paths)
template <class T, int D>
static void prepare_lists(const SphEngine* e, cudaStream_t s)
{
    GridP<T> g = grid_of_engine<T>(e);
    Eng<T> E = eng_of<T>(e);
    cudaMemsetAsync(e->qcount, 0, sizeof(uint32_t), s);
    if (e->n <= 0) return;
    launch_pdl(pdl_for(e), k_mask<T, D>, grid_for(e->n, kSweepThreads), kSweepThreads, s, E, g,
               skin_eff<T>(e));
    launch_fix<T, D>(e, s);
}

// Split filtering: with a wide skin (fast flows; e.g. the periodic
// Taylor-Green case keeps ~1.6x more skin entries than neighbours in 3D) a
// fused filter makes every warp run the continuity pair body for the union
// of its lanes' accepted entries, i.e. nearly every skin entry.  Past this
// skin/cutoff ratio the sub-step filters all skin lists up front (k_mask,
// exact lists for every particle) and the sweeps walk exact lists only.
// In 2D (~25 skin entries) the fused walk stays ahead at every skin
// (measured: +4% at rest, +7% at step 40 of the 2D dam break).
#ifndef SPH_SPLIT_SKIN_RATIO
#define SPH_SPLIT_SKIN_RATIO 0.12
#endif
#ifndef SPH_SPLIT_2D
#define SPH_SPLIT_2D 0
#endif
static bool split_filter(const SphEngine* e)
{
    if (e->dim == 2 && !SPH_SPLIT_2D) return false;
    return e->skin > SPH_SPLIT_SKIN_RATIO * e->cutoff;
}

// sub-step path: only the invalid lists are rebuilt up front; valid skin
// lists are filtered inside the continuity / wall sweeps
template <class T, int D>
static void mark_and_fix(const SphEngine* e, cudaStream_t s)
{
    Eng<T> E = eng_of<T>(e);
    if (e->n <= 0) return;
    // few refreshes expected (host hint from the previous step): check +
    // refresh in one pass; otherwise the queue spreads the (spatially
    // clustered) refreshes over more warps (measured with the one-pass
    // kernel: 2D at rest -3 us per sub-step, at step 40 +27 us)
    if (SPH_MARK_FUSED && e->few_refreshes) {
        const int64_t want = (e->n + 4 * kNlThreads - 1) / (4 * kNlThreads);
        const int blocks = (int)(want < 148 * 4 ? want : 148 * 4);
        launch_pdl(pdl_for(e), k_mark_refresh<T, D>, blocks, kNlThreads, s, acc_of_engine<T>(e),
                   grid_of_engine<T>(e), E, skin_cs2<T>(e), skin_eff<T>(e));
        return;
    }
    cudaMemsetAsync(e->qcount, 0, sizeof(uint32_t), s);
    launch_pdl(pdl_for(e), k_mark<T>, grid_for((e->n + 3) / 4, 256), 256, s, E, skin_eff<T>(e));
    launch_fix<T, D>(e, s);
}

static int require_lists(const SphEngine* e)
{
    if (!e->lists_ready) {
        set_error("engine: neighbour lists not built since the last CLL rebuild");
        return SPH_ERR_INVALID;
    }
    return SPH_OK;
}

template <class T, int D>
static void launch_wall(const SphEngine* e, int b, int zero_drho, int count_factor, int filter,
                        int cvn, cudaStream_t s)
{
    const int64_t nw = e->n - e->nf;
    const Eng<T> E = eng_of<T>(e);
    const PhysT<T> P = make_phys<T>(phys_of_engine(e));
    const GridP<T> g = grid_of_engine<T>(e);
    // a thread per wall: a warp per wall with an ordered shuffle chain for
    // the sums measured 1.4x (2D) to 7x (3D) slower
    if (SPH_WALL_LANES > 1)
        launch_pdl(pdl_for(e), k_wall_g<T, D, (SPH_WALL_LANES > 1 ? SPH_WALL_LANES : 2)>,
                   grid_for(nw * SPH_WALL_LANES, kSweepThreads), kSweepThreads, s, E, P, g, b,
                   zero_drho, count_factor, filter, cvn);
    else
        launch_pdl(pdl_for(e), k_wall<T, D>, grid_for(nw, kSweepThreads), kSweepThreads, s, E, P, g, b,
                   zero_drho, count_factor, filter, cvn);
}

// physics.py:460-467 initialize, in its two halo-exchange phases: exact
// lists + WALL_PRESSURE into the current buffer, then MOMENTUM (no kick)
template <class T, int D>
static void init_wall(SphEngine* e, cudaStream_t s)
{
    prepare_lists<T, D>(e, s);
    const int64_t nw = e->n - e->nf;
    if (nw > 0)
        launch_wall<T, D>(e, e->cur_rp, 0, 1, 0, -1, s);
}

template <class T, int D>
static void init_momentum(SphEngine* e, cudaStream_t s)
{
    Eng<T> E = eng_of<T>(e);
    const int64_t nw = e->n - e->nf;
    if (e->nf > 0) {
        note_launch(), k_rq_fill<T><<<grid_for(e->nf, 256), 256, 0, s>>>(E, e->cur_rp, e->nf);
        note_launch(), k_mom<T, D><<<grid_for(e->nf, kSweepThreads), kSweepThreads, 0, s>>>(
            E, make_phys<T>(phys_of_engine(e)), e->cur_v, e->cur_rp, 0, T(0), 1,
            grid_of_engine<T>(e), 0, T(0));
    }
    // momentum writes dvdt = 0 for walls (physics.py:128-131)
    if (nw > 0)
        cudaMemsetAsync((char*)e->dvdt + sizeof(vec4<T>) * (size_t)e->nf, 0,
                        sizeof(vec4<T>) * (size_t)nw, s);
}

template <class T, int D>
static int initialize_impl(SphEngine* e, cudaStream_t s)
{
    init_wall<T, D>(e, s);
    init_momentum<T, D>(e, s);
    return check_launch("engine_initialize");
}

extern "C" int sph_engine_initialize(SphEngine* e, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    return SPH_DISPATCH(e, initialize_impl, e, s);
}

template <class T, int D>
static int shepard_impl(SphEngine* e, cudaStream_t s)
{
    if (e->n <= 0) return SPH_OK;
    prepare_lists<T, D>(e, s);
    Eng<T> E = eng_of<T>(e);
    const PhysT<T> P = make_phys<T>(phys_of_engine(e));
    note_launch(), k_shepard<T, D><<<grid_for(e->n, kSweepThreads), kSweepThreads, 0, s>>>(
        E, P, e->cur_rp);
    e->cur_rp ^= 1;
    return check_launch("engine_shepard");
}

extern "C" int sph_engine_shepard(SphEngine* e, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    return SPH_DISPATCH(e, shepard_impl, e, s);
}

// physics.py:522-548, one acoustic sub-step in the phases between which a
// multi-rank run exchanges halo data
template <class T, int D>
static void sub_kick_drift(SphEngine* e, T half, T full, cudaStream_t s)
{
    if (e->n > 0)
        launch_pdl(pdl_for(e), k_kick_drift<T, D>, grid_for(e->n, 256), 256, s, eng_of<T>(e), e->cur_v,
                   e->cur_rp, grid_of_engine<T>(e), half, full);
}

// list upkeep of a sub-step: exact lists for all (split) or for the
// particles whose skin list is no longer valid
template <class T, int D>
static void sub_lists(SphEngine* e, cudaStream_t s)
{
    launch_blockmax<T, D>(e, s);   // local displacement bounds after the drift
    if (split_filter(e)) prepare_lists<T, D>(e, s);
    else mark_and_fix<T, D>(e, s);
}

// Walls' continuity operand m/rho from the current (rho, p) buffer.  After a
// fused MOMENTUM_NEXT phase of a slab rank the KICK_DRIFT phase (which sets
// it for walls and ghosts) is skipped; k_wall set it for every wall from
// this rank's own wall pressure, which for WALL GHOSTS is superseded by the
// owner's (rho, p) refresh -- so it is recomputed here from the refreshed
// buffer (owned walls get the value they already hold).
template <class T>
__global__ void __launch_bounds__(256) k_wall_operands(Eng<T> E, int cv, int crp)
{
    pdl_begin();   // PDL: wait for the previous kernel, let the next one launch
    const int64_t i = E.nf + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < E.n)
        reinterpret_cast<T*>(&E.vel[cv][i])[3] = RN<T>::div(E.pos[i].w, E.rp[crp][i].x);
}

template <class T>
static void sub_wall_operands(SphEngine* e, cudaStream_t s)
{
    const int64_t nw = e->n - e->nf;
    if (nw > 0)
        launch_pdl(pdl_for(e), k_wall_operands<T>, grid_for(nw, 256), 256, s, eng_of<T>(e), e->cur_v,
                   e->cur_rp);
}

template <class T, int D>
static void sub_continuity(SphEngine* e, T full, cudaStream_t s)
{
    Eng<T> E = eng_of<T>(e);
    const int crp = e->cur_rp;
    if (e->nf > 0 && split_filter(e))
        launch_pdl(pdl_for(e), k_cont_du<T, D, true>, grid_for(e->nf, kSweepThreads), kSweepThreads, s, E,
                   make_phys<T>(phys_of_engine(e)), grid_of_engine<T>(e), e->cur_v, crp, full);
    else if (e->nf > 0)
        launch_pdl(pdl_for(e), k_cont_du<T, D, false>, grid_for(e->nf, kSweepThreads), kSweepThreads, s, E,
                   make_phys<T>(phys_of_engine(e)), grid_of_engine<T>(e), e->cur_v, crp, full);
    else if (e->n > 0)   // no fluid: the other rp buffer must still carry walls
        cudaMemcpyAsync(E.rp[crp ^ 1], E.rp[crp], sizeof(vec2<T>) * (size_t)e->n,
                        cudaMemcpyDeviceToDevice, s);
}

template <class T, int D>
static void sub_wall(SphEngine* e, cudaStream_t s)
{
    const int64_t nw = e->n - e->nf;
    if (nw > 0)
        launch_wall<T, D>(e, e->cur_rp ^ 1, 1, 1, split_filter(e) ? 0 : 1, e->cur_v ^ 1, s);
}

// zero_walls: the reference's momentum body writes dvdt = 0 for walls
// (physics.py:128-131); only a host edit can make it non-zero, and nothing
// reads it within a step, so once per step suffices
template <class T, int D>
static void sub_momentum(SphEngine* e, T half, T next_full, bool fuse, bool zero_walls,
                         cudaStream_t s)
{
    Eng<T> E = eng_of<T>(e);
    const int cv = e->cur_v;
    fuse = fuse && e->nf > 0;
    if (zero_walls && e->n > e->nf)
        cudaMemsetAsync((char*)e->dvdt + sizeof(vec4<T>) * (size_t)e->nf, 0,
                        sizeof(vec4<T>) * (size_t)(e->n - e->nf), s);
    if (e->nf > 0)
        launch_pdl(pdl_for(e), k_mom<T, D>, grid_for(e->nf, kSweepThreads), kSweepThreads, s, E,
                   make_phys<T>(phys_of_engine(e)), cv, e->cur_rp ^ 1, 1, half, 2,
                   grid_of_engine<T>(e), fuse ? 1 : 0, next_full);
    else if (e->n > 0)
        cudaMemcpyAsync(E.vel[cv ^ 1], E.vel[cv], sizeof(vec4<T>) * (size_t)e->n,
                        cudaMemcpyDeviceToDevice, s);
    e->cur_v = cv ^ 1;
    e->cur_rp ^= 1;
    if (fuse) {
        e->cur_pos ^= 1;
        e->drifted = 1;
    }
}

// One sub-step; fuse: its momentum sweep also applies the next sub-step's
// kick + drift.  ev (optional, 6 events) brackets: kick+drift | list filter
// + fix-ups | continuity+DU | wall pressure | momentum+kick (bench.py timing)
template <class T, int D>
static void substep_parts(SphEngine* e, T half, T full, bool fuse, cudaEvent_t* ev,
                          cudaStream_t s, cudaEvent_t* marks = nullptr)
{
    if (ev) cudaEventRecord(ev[0], s);
    e->cll_fresh = 0;   // particles move from here on
    if (!e->drifted) sub_kick_drift<T, D>(e, half, full, s);
    e->drifted = 0;
    if (marks) cudaEventRecord(marks[0], s);   // positions final
    if (ev) cudaEventRecord(ev[1], s);
    sub_lists<T, D>(e, s);
    if (ev) cudaEventRecord(ev[2], s);
    sub_continuity<T, D>(e, full, s);
    if (ev) cudaEventRecord(ev[3], s);
    sub_wall<T, D>(e, s);
    if (marks) cudaEventRecord(marks[1], s);   // rho, p (fluid and walls), drho final
    if (ev) cudaEventRecord(ev[4], s);
    sub_momentum<T, D>(e, half, full, fuse, !fuse, s);
    if (ev) cudaEventRecord(ev[5], s);
}

template <class T, int D>
static int substep_impl(SphEngine* e, double half_d, double full_d, cudaEvent_t* ev,
                        cudaStream_t s)
{
    substep_parts<T, D>(e, T(half_d), T(full_d), false, ev, s);
    return check_launch("engine_substep");
}

extern "C" int sph_engine_substep(SphEngine* e, double half_dt, double full_dt, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    return SPH_DISPATCH(e, substep_impl, e, half_dt, full_dt, (cudaEvent_t*)nullptr, s);
}

extern "C" int sph_engine_substep_timed(SphEngine* e, double half_dt, double full_dt,
                                        float* ms_out, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    cudaEvent_t ev[6];
    for (int k = 0; k < 6; k++) cudaEventCreate(&ev[k]);
    rc = SPH_DISPATCH(e, substep_impl, e, half_dt, full_dt, ev, s);
    if (rc == SPH_OK) {
        cudaEventSynchronize(ev[5]);
        for (int k = 0; k < 5; k++) cudaEventElapsedTime(&ms_out[k], ev[k], ev[k + 1]);
    }
    for (int k = 0; k < 6; k++) cudaEventDestroy(ev[k]);
    return rc ? rc : check_launch("engine_substep_timed");
}

// physics.py:522-548 for the nsub sub-steps of one advective step.  ms
// (optional): per-part CUDA-event times summed over the sub-steps; the
// events are only recorded between the launches (no host synchronisation
// until the last sub-step), so the timed step runs as the untimed one does
template <class T, int D>
static int substeps_impl(SphEngine* e, double half_d, double full_d, int nsub, float* ms,
                         cudaStream_t s, cudaEvent_t* marks = nullptr)
{
    const T half = T(half_d), full = T(full_d);
    cudaEvent_t* ev = nullptr;
    if (ms) {
        ev = new cudaEvent_t[6 * (size_t)(nsub > 0 ? nsub : 1)];
        for (int k = 0; k < 6 * nsub; k++) cudaEventCreate(&ev[k]);
        for (int k = 0; k < 5; k++) ms[k] = 0.0f;
    }
    for (int k = 0; k < nsub; k++)
        substep_parts<T, D>(e, half, full, k + 1 < nsub, ms ? ev + 6 * k : nullptr, s,
                            k + 1 == nsub ? marks : nullptr);
    if (marks && nsub == 0) {
        cudaEventRecord(marks[0], s);
        cudaEventRecord(marks[1], s);
    }
    if (ms) {
        if (nsub > 0) cudaEventSynchronize(ev[6 * nsub - 1]);
        for (int k = 0; k < nsub; k++)
            for (int q = 0; q < 5; q++) {
                float t = 0.0f;
                cudaEventElapsedTime(&t, ev[6 * k + q], ev[6 * k + q + 1]);
                ms[q] += t;
            }
        for (int k = 0; k < 6 * nsub; k++) cudaEventDestroy(ev[k]);
        delete[] ev;
    }
    return check_launch("engine_substeps");
}

extern "C" int sph_engine_substeps(SphEngine* e, double half_dt, double full_dt, int32_t nsub,
                                   cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    if (nsub < 0 || e->drifted) return SPH_ERR_INVALID;
    return SPH_DISPATCH(e, substeps_impl, e, half_dt, full_dt, (int)nsub, (float*)nullptr, s);
}

extern "C" int sph_engine_substeps_marked(SphEngine* e, double half_dt, double full_dt,
                                          int32_t nsub, cudaEvent_t x_final,
                                          cudaEvent_t rp_final, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    if (nsub < 0 || e->drifted || !x_final || !rp_final) return SPH_ERR_INVALID;
    cudaEvent_t marks[2] = {x_final, rp_final};
    return SPH_DISPATCH(e, substeps_impl, e, half_dt, full_dt, (int)nsub, (float*)nullptr, s,
                        marks);
}

extern "C" int sph_engine_substeps_timed(SphEngine* e, double half_dt, double full_dt,
                                         int32_t nsub, float* ms_out, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    if (nsub < 0 || e->drifted) return SPH_ERR_INVALID;
    return SPH_DISPATCH(e, substeps_impl, e, half_dt, full_dt, (int)nsub, ms_out, s);
}

template <class T, int D>
static int phase_impl(SphEngine* e, int phase, double half_d, double full_d, cudaStream_t s)
{
    e->cll_fresh = 0;   // a phase may move particles (kick + drift)
    const T half = T(half_d), full = T(full_d);
    switch (phase) {
    case SPH_PHASE_KICK_DRIFT:   // already applied by a MOMENTUM_NEXT phase?
        if (!e->drifted) sub_kick_drift<T, D>(e, half, full, s);
        else sub_wall_operands<T>(e, s);
        e->drifted = 0;
        break;
    case SPH_PHASE_CONTINUITY:
        sub_lists<T, D>(e, s);
        sub_continuity<T, D>(e, full, s);
        break;
    case SPH_PHASE_WALL: sub_wall<T, D>(e, s); break;
    case SPH_PHASE_MOMENTUM: sub_momentum<T, D>(e, half, T(0), false, true, s); break;
    case SPH_PHASE_MOMENTUM_NEXT: sub_momentum<T, D>(e, half, full, true, false, s); break;
    case SPH_PHASE_INIT_WALL: init_wall<T, D>(e, s); break;
    case SPH_PHASE_INIT_MOMENTUM: init_momentum<T, D>(e, s); break;
    default: set_error("engine_phase: unknown phase"); return SPH_ERR_INVALID;
    }
    return check_launch("engine_phase");
}

extern "C" int sph_engine_phase(SphEngine* e, int32_t phase, double half_dt, double full_dt,
                                cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc || (rc = require_lists(e))) return rc;
    return SPH_DISPATCH(e, phase_impl, e, phase, half_dt, full_dt, s);
}

// ---------------------------------------------------------------------------
// halo records (multi-rank slabs)
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256)
k_pack(Eng<T> E, int kind, int cv, int b, const int32_t* __restrict__ phys, int64_t count,
       T* __restrict__ out)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const int64_t i = phys[k];
    if (kind == SPH_HALO_XV) {
        const vec4<T> P4 = E.pos[i], V4 = E.vel[cv][i];
        T* o = out + 9 * k;
        o[0] = P4.x; o[1] = P4.y; o[2] = P4.z; o[3] = P4.w;
        o[4] = V4.x; o[5] = V4.y; o[6] = V4.z; o[7] = V4.w;
        o[8] = E.disp[i];
    } else {
        const vec2<T> RP = E.rp[b][i];
        out[2 * k] = RP.x;
        out[2 * k + 1] = RP.y;
    }
}

template <class T, int D>
__global__ void __launch_bounds__(256)
k_unpack(Eng<T> E, GridP<T> g, int kind, int cv, int b, const int32_t* __restrict__ phys,
         int64_t count, const T* __restrict__ in)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    T dsp = T(0);
    if (k < count) {
        const int64_t i = phys[k];
        if (kind == SPH_HALO_XV) {
            const T* r = in + 9 * k;
            vec4<T> P4, V4;
            P4.x = r[0]; P4.y = r[1]; P4.z = r[2]; P4.w = r[3];
            V4.x = r[4]; V4.y = r[5]; V4.z = r[6]; V4.w = r[7];
            dsp = r[8];
            E.pos[i] = P4;
            E.vel[cv][i] = V4;
            E.disp[i] = dsp;
            // the ghost's list stays valid only in the cell it was built for
            const T xn[3] = {P4.x, P4.y, P4.z};
            int c[3];
            if (cell_key_of<T, D>(xn, g, c) != E.cell0[i]) E.cell0[i] = kInvalidCell;
        } else {
            vec2<T> RP;
            RP.x = in[2 * k];
            RP.y = in[2 * k + 1];
            E.rp[b][i] = RP;
            E.rq[i] = rq_of<T>(RP);
        }
    }
    if (kind == SPH_HALO_XV) {
        const unsigned long long m = warp_max_u64(dbits(double(dsp)));
        if (lane_id() == 0 && m) atomicMax(&E.stats->dmax_bits, m);
    }
}

extern "C" int32_t sph_engine_halo_width(int32_t kind)
{
    return kind == SPH_HALO_XV ? 9 : (kind == SPH_HALO_RP_NEXT || kind == SPH_HALO_RP_CUR) ? 2
                                                                                         : -1;
}

template <class T, int D>
static int pack_impl(const SphEngine* e, int kind, const int32_t* phys, int64_t count, void* out,
                     cudaStream_t s)
{
    if (count > 0)
        note_launch(), k_pack<T><<<grid_for(count, 256), 256, 0, s>>>(
            eng_of<T>(e), kind, e->cur_v, kind == SPH_HALO_RP_NEXT ? e->cur_rp ^ 1 : e->cur_rp,
            phys, count, (T*)out);
    return check_launch("engine_pack");
}

template <class T, int D>
static int unpack_impl(SphEngine* e, int kind, const int32_t* phys, int64_t count,
                       const void* in, cudaStream_t s)
{
    if (count > 0)
        note_launch(), k_unpack<T, D><<<grid_for(count, 256), 256, 0, s>>>(
            eng_of<T>(e), grid_of_engine<T>(e), kind, e->cur_v,
            kind == SPH_HALO_RP_NEXT ? e->cur_rp ^ 1 : e->cur_rp, phys, count, (const T*)in);
    return check_launch("engine_unpack");
}

extern "C" int sph_engine_pack(const SphEngine* e, int32_t kind, const int32_t* phys,
                               int64_t count, void* out, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc) return rc;
    if (sph_engine_halo_width(kind) < 0 || count < 0) return SPH_ERR_INVALID;
    return SPH_DISPATCH(e, pack_impl, e, kind, phys, count, out, s);
}

extern "C" int sph_engine_unpack(SphEngine* e, int32_t kind, const int32_t* phys, int64_t count,
                                 const void* in, cudaStream_t s)
{
    int rc = engine_begin(e, s);
    if (rc) return rc;
    if (sph_engine_halo_width(kind) < 0 || count < 0) return SPH_ERR_INVALID;
    if (kind == SPH_HALO_XV) e->cll_fresh = 0;   // ghosts' positions change
    return SPH_DISPATCH(e, unpack_impl, e, kind, phys, count, in, s);
}
