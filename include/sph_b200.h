/* sph_b200.h -- C ABI of the B200-native SPH particle-step library
 * (libsphb200.so, built for sm_100a).
 *
 * Drop-in boundary for the reference's hot path (reference package `minisph`,
 * /root/reference/pkg/src/minisph).  The reference crosses from Python into
 * native code at exactly two call sites: `kernel.driver()(range_size, args)`
 * (execution.py:129, particle_for) and the reduce driver (execution.py:206,
 * particle_reduce); plus the CLL build and sort drivers it calls from the
 * step (neighborhood.py:149-173, sorting.py:46-70).  Each entry point below
 * names the reference interface it replaces.
 *
 * Conventions
 *  - extern "C", plain pointers + sizes; every pointer marked (dev) is device
 *    memory, everything else host memory.
 *  - Every call enqueues work on the caller's stream and returns an int
 *    status (SPH_OK == 0); it never throws and never allocates persistent
 *    memory.  Scratch comes from the caller, sized by the *_bytes queries.
 *  - `_f32` entry points implement the reference's precision="f32" run
 *    (binary32 storage with the binary64 temporaries numba infers, no FMA);
 *    `_f64` ones the precision="f64" run.  Results are bit-identical to the
 *    reference on the same inputs.
 */
#ifndef SPH_B200_H
#define SPH_B200_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_ABI_VERSION 16
#define SPH_NEIGHBOR_CAPACITY 256   /* neighborhood.py:30 NEIGHBOR_CAPACITY */

/* status codes; mapped to the reference's exception classes by the host */
enum {
    SPH_OK = 0,
    SPH_ERR_INVALID = 1,        /* bad argument (TypeError/ValueError)       */
    SPH_ERR_CUDA = 2,           /* CUDA launch/runtime error                  */
    SPH_ERR_NEGATIVE_KEY = 3,   /* ValueError, sorting.py:52-53               */
    SPH_ERR_WORKSPACE = 4,      /* workspace smaller than *_bytes query       */
    SPH_ERR_UNSUPPORTED = 5     /* grid too large for 32-bit cell keys, ...   */
};

int sph_abi_version(void);
const char* sph_last_error(void);
/* kernels launched by this library since load (bench gpu_launches) */
long long sph_kernel_launches(void);

/* ---------------------------------------------------------------------------
 * Generic kernel-dispatch boundary: particle_for(policy, n, KERNEL, args)
 * with args == force_args(registry, cll) (physics.py:315-330), arrays in the
 * reference layout (vectors (n, d) row-major, index fields uint32) and the
 * caller's CellLinkedList (offsets int64[C+1], particle_ids int64[n]).
 * -------------------------------------------------------------------------*/
typedef struct {
    /* per-particle (dev) */
    const float* x; const float* v; float* rho; float* p; const float* m;
    const uint32_t* wall; const uint32_t* ids;
    const int64_t* offsets; const int64_t* pids;
    float* drho; float* dvdt; uint32_t* nnb; uint32_t* oflow;
    float* rho_new;                 /* Shepard target, physics.py:222 */
    /* host values */
    float g[3]; float origin[3]; int64_t shape[3];
    float cell_size, cutoff, h, alpha_d, c0, rho0, alpha_visc, eps_h2;
    int64_t n; int32_t dim; int32_t reserved;
} SphSweepArgs_f32;

typedef struct {
    const double* x; const double* v; double* rho; double* p; const double* m;
    const uint32_t* wall; const uint32_t* ids;
    const int64_t* offsets; const int64_t* pids;
    double* drho; double* dvdt; uint32_t* nnb; uint32_t* oflow;
    double* rho_new;
    double g[3]; double origin[3]; int64_t shape[3];
    double cell_size, cutoff, h, alpha_d, c0, rho0, alpha_visc, eps_h2;
    int64_t n; int32_t dim; int32_t reserved;
} SphSweepArgs_f64;

/* scratch for the ordered neighbour lists the sweeps build */
size_t sph_sweep_workspace_bytes(int64_t n);

/* physics.py:94-119 CONTINUITY / :122-158 MOMENTUM / :161-194 WALL_PRESSURE /
 * :197-217 DENSITY_SUMMATION / :220-247 SHEPARD, each over i in [0, n) */
int sph_continuity_f32(const SphSweepArgs_f32* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_momentum_f32(const SphSweepArgs_f32* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_wall_pressure_f32(const SphSweepArgs_f32* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_density_summation_f32(const SphSweepArgs_f32* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_shepard_f32(const SphSweepArgs_f32* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_continuity_f64(const SphSweepArgs_f64* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_momentum_f64(const SphSweepArgs_f64* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_wall_pressure_f64(const SphSweepArgs_f64* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_density_summation_f64(const SphSweepArgs_f64* a, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_shepard_f64(const SphSweepArgs_f64* a, void* ws, size_t ws_bytes, cudaStream_t s);

/* neighborhood.py:176-227 collect_neighbors for particles i0..i0+count-1:
 * out_lists (dev, count x 256 int32) = physical j in ascending-id order,
 * out_counts (dev, count) = count or -1 on overflow. */
int sph_neighbors_f32(const SphSweepArgs_f32* a, int64_t i0, int64_t count,
                      int32_t* out_lists, int32_t* out_counts, cudaStream_t s);
int sph_neighbors_f64(const SphSweepArgs_f64* a, int64_t i0, int64_t count,
                      int32_t* out_lists, int32_t* out_counts, cudaStream_t s);

/* physics.py:250-256 KICK, :259-265 DRIFT, :268-274 DENSITY_UPDATE,
 * :277-280 COPY_SCALAR (all dev arrays, reference layout) */
int sph_kick_f32(float* v, const float* dvdt, const uint32_t* wall, int64_t n, int dim, float half_dt, cudaStream_t s);
int sph_drift_f32(float* x, const float* v, const uint32_t* wall, int64_t n, int dim, float dt, cudaStream_t s);
int sph_density_update_f32(float* rho, float* p, const float* drho, const uint32_t* wall, int64_t n,
                           float dt, float c0, float rho0, cudaStream_t s);
int sph_kick_f64(double* v, const double* dvdt, const uint32_t* wall, int64_t n, int dim, double half_dt, cudaStream_t s);
int sph_drift_f64(double* x, const double* v, const uint32_t* wall, int64_t n, int dim, double dt, cudaStream_t s);
int sph_density_update_f64(double* rho, double* p, const double* drho, const uint32_t* wall, int64_t n,
                           double dt, double c0, double rho0, cudaStream_t s);
int sph_copy(void* dst, const void* src, int64_t nbytes, cudaStream_t s);

/* diagnostic: count (into *bad, dev) quotients a/h where the kernels'
 * reciprocal-based division differs from IEEE __fdiv_rn / __ddiv_rn, over n
 * pseudo-random a (binary32 h = (float)h and binary64 h) */
int sph_selftest_div(double h, int64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t s);
/* test support: the f32 sweeps' straight-line pair factor (physics.cuh
 * pair_fac_spec) against the per-operation IEEE sequence for every binary32
 * r2 bit pattern in [lo_bits, hi_bits); *bad += mismatches, *first_bad =
 * min mismatching pattern (initialise to 0xffffffff) */
int sph_selftest_pair_fac(double h, double alpha_d, uint32_t lo_bits, uint32_t hi_bits,
                          unsigned long long* bad, unsigned int* first_bad, cudaStream_t s);
/* test support: the momentum sweep's binary32 rounding done in the FP64
 * adder (physics.cuh rn_f32_in_f64) against __double2float_rn on n random
 * binary64 values (half of them binary32 ties); *bad += mismatches where the
 * fast path claims validity, *fast += values it handled */
int sph_selftest_round_f32(int64_t n, uint64_t seed, unsigned long long* bad,
                           unsigned long long* fast, cudaStream_t s);

/* physics.py:296-310 VMAX_SPEC through particle_reduce (execution.py:191-209):
 * *out (dev double) = max_i sqrt(sum_k f64(v_ik*v_ik)), identity 0.0 */
int sph_vmax_f32(const float* v, int64_t n, int dim, double* out, cudaStream_t s);
int sph_vmax_f64(const double* v, int64_t n, int dim, double* out, cudaStream_t s);

/* ---------------------------------------------------------------------------
 * Cell linked list and sort (neighborhood.py:105-173, sorting.py:46-81)
 * -------------------------------------------------------------------------*/
/* neighborhood.py:137-146 compute_cell_keys: keys (dev int64[n]) and the
 * clamp count (*oob_count, dev uint32) */
int sph_cell_keys_f32(const float* x, int64_t n, int dim, const float* origin, float cell_size,
                      const int64_t* shape, int64_t* keys, uint32_t* oob_count, cudaStream_t s);
int sph_cell_keys_f64(const double* x, int64_t n, int dim, const double* origin, double cell_size,
                      const int64_t* shape, int64_t* keys, uint32_t* oob_count, cudaStream_t s);

/* neighborhood.py:149-173 build_cell_linked_list: offsets (dev int64[C+1]),
 * particle_ids (dev int64[n]) == argsort(keys, kind="stable"). */
size_t sph_cll_workspace_bytes(int64_t n, int64_t ncells);
int sph_cll_build_f32(const float* x, int64_t n, int dim, const float* origin, float cell_size,
                      const int64_t* shape, int64_t* offsets, int64_t* particle_ids,
                      uint32_t* oob_count, void* ws, size_t ws_bytes, cudaStream_t s);
int sph_cll_build_f64(const double* x, int64_t n, int dim, const double* origin, double cell_size,
                      const int64_t* shape, int64_t* offsets, int64_t* particle_ids,
                      uint32_t* oob_count, void* ws, size_t ws_bytes, cudaStream_t s);

/* sorting.py:46-70 radix_sort_permutation: stable LSD radix (8-bit digits)
 * of non-negative int64 keys; perm (dev int64[n]).  *max_key_out (host) may
 * be NULL.  Returns SPH_ERR_NEGATIVE_KEY on a negative key. */
size_t sph_sort_workspace_bytes(int64_t n);
int sph_radix_sort_perm(const int64_t* keys, int64_t n, int64_t* perm,
                        void* ws, size_t ws_bytes, cudaStream_t s);

/* variables.py:132-145 apply_permutation: dst[k] = src[perm[k]] for
 * elements of elem_bytes (4, 8, 12, 16, 24 or 32). */
int sph_gather(void* dst, const void* src, const int64_t* perm, int64_t n, int elem_bytes,
               cudaStream_t s);

/* ---------------------------------------------------------------------------
 * Case placement on the device (cases.py:129-161 _lattice, _tank_wall_points,
 * _box_points; the obstacle cut of build_case_dambreak, cases.py:227-233).
 * Lattice points anchor[k] + (i_k + 0.5)*dp (binary64) over the index box
 * lo[k] <= i_k < hi[k] (host arrays of d), kept by mode and compacted in the
 * lattice's C order (last axis fastest, np.meshgrid(indexing="ij").ravel())
 * into out (dev, (count, d) binary64; NULL = count only).  *count (dev int64)
 * receives the number kept; *ilast_max (dev u64, caller-zeroed) the
 * order-preserving key (i ^ 2^63) of the largest kept last-axis index.
 * -------------------------------------------------------------------------*/
#define SPH_LATTICE_ALL 0      /* every point (_lattice, _box_points)                 */
#define SPH_LATTICE_TANK 1     /* _tank_wall_points' outside test, counts[0..d)       */
#define SPH_LATTICE_NOT_IN 2   /* not strictly inside the open box (box_lo, box_hi)   */
size_t sph_lattice_workspace_bytes(int32_t d, const int64_t* lo, const int64_t* hi);
int sph_lattice_points(int32_t d, const int64_t* lo, const int64_t* hi, double dp,
                       const double* anchor, int32_t mode, const int64_t* counts,
                       const double* box_lo, const double* box_hi, double* out,
                       int64_t* count, unsigned long long* ilast_max, void* ws,
                       size_t ws_bytes, cudaStream_t s);

/* ---------------------------------------------------------------------------
 * Device-resident step engine: the B200 restatement of Simulation.advance
 * (physics.py:489-552).  Particles live in two segments -- fluid [0, nf),
 * walls [nf, n) -- each ordered by grid cell; the fluid segment is re-sorted
 * by cell every advective step, the static walls once.  All accumulation
 * runs in ascending original-id order, so every field is bit-identical to
 * the reference for any physical order.
 * -------------------------------------------------------------------------*/
typedef struct {
    unsigned long long vmax_bits;     /* exact max |v|   (f64 bits)            */
    unsigned long long amax_bits;     /* exact max |dvdt| (f64 bits)           */
    unsigned long long interactions;  /* report.py:20-21 directed visits       */
    unsigned long long rho_min_key;   /* order-preserving key of min rho (f64) */
    unsigned long long v2max_key;     /* key of max run-precision |v|^2        */
    unsigned long long dmax_bits;     /* max path length since the skin build  */
    unsigned int overflow;            /* particles over NEIGHBOR_CAPACITY      */
    unsigned int oob;                 /* fluid out-of-bounds clamps            */
    unsigned int oob_walls;           /* wall clamps (counted once, at push)   */
    unsigned int nfix;                /* list refreshes (cell change / skin)   */
    unsigned int nan_flags;           /* bit0: a NaN rho, bit1: a NaN |v|^2    */
    unsigned int push_error;          /* push: ids not a permutation of 0..n-1 */
    unsigned int fluid_seen;          /* push: particles with wall == 0        */
    unsigned int ndisp;               /* of which displacement-triggered       */
} SphStepStats;

typedef struct {
    /* sizes */
    int64_t n, nf, ncells; int32_t dim; int32_t key_bits;
    /* per-particle SoA, physical order (dev).  f32 run: float4/float2,
     * f64 run: double4/double2 (reinterpret). pos.w == m; pos, vel and rp
     * are double buffers (cur_pos / cur_v / cur_rp select); vel.w is scratch
     * (m/rho of the sub-step's continuity sweep); rq = (rho, p/rho^2) of the
     * sub-step's momentum sweep (library-maintained, no host meaning). */
    void* pos[2]; void* vel[2]; void* rp[2]; void* rq; void* dvdt; void* drho;
    uint32_t* id; uint32_t* nnb; uint32_t* refpos;
    /* by-id cold fields (dev) */
    void* rho_scratch_id; uint32_t* oflow_id; uint32_t* wall_id; void* vol_id;
    /* multi-rank slabs: 1 for particles this rank owns, 0 for halo ghosts,
     * by id; NULL = every particle is owned.  Ghosts are not integrated and
     * count in no counter or reduction (their state arrives by unpack). */
    uint8_t* owned_id;
    /* cell offsets into each segment (dev, ncells+1 each) */
    uint32_t* offs_f; uint32_t* offs_w;
    /* ascending-id Verlet (skin) lists and this sub-step's exact lists, both
     * tile-ELL [slots/32][256][32] int32; per slot: skin entries (lcount),
     * exact count or -1 on overflow (acount), static wall-wall count of walls
     * (nww); per particle: list cell (cell0) and path length since the list
     * build (disp, run precision); fix-up queue */
    int32_t* lists; int32_t* lcount; int32_t* acount; int32_t* nww; int32_t* elist;
    uint32_t* cell0; void* disp; uint32_t* queue; uint32_t* qcount;
    /* scratch (dev): keys/values x2 for the radix sort + gather staging */
    void* ws; size_t ws_bytes;
    SphStepStats* stats;              /* dev */
    /* physics scalars (run precision, passed as double for both runs) */
    double g[3]; double origin[3]; int64_t shape[3];
    double cell_size, cutoff, h, alpha_d, c0, rho0, alpha_visc, eps_h2;
    double skin;                      /* Verlet skin of the current lists    */
    /* double-buffer selectors and list state, maintained by the library */
    int32_t cur_v, cur_rp, cur_pos;
    int32_t drifted;                  /* next sub-step's kick+drift already applied */
    int32_t f64;                      /* 0: f32 run, 1: f64 run */
    int32_t lists_ready;
    /* periodic box (beyond the reference): per axis the
     * period L (run precision value; 0 = bounded as in the reference).  A
     * periodic axis wraps over [origin, origin + L), needs shape >= 3 and
     * L <= shape * cell_size; only libsphb200_periodic.so accepts L > 0. */
    double period[3];
    /* per particle (dev, run precision): the value of disp when the
     * particle's own skin list was last built (a mid-step refresh after a
     * cell change re-bases it; disp itself always measures the path since
     * the step's list build, which bounds every neighbour's motion) */
    void* disp0;
    /* host hint: 1 when the previous step refreshed few lists, so the
     * sub-step's list check and refreshes run as one queue-free pass */
    int32_t few_refreshes;
    /* library state: the walls' static wall-wall neighbour counts (nww) are
     * valid (computed by the first list build after a push; walls never
     * move), so later builds skip wall-only candidate blocks */
    int32_t nww_ready;
    /* id space: 0 = ids are a permutation of 0..n-1 (checked at push);
     * > 0 = ids are distinct values below id_range (multi-rank slabs use
     * GLOBAL ids, so the by-id arrays -- rho_scratch_id, oflow_id, wall_id,
     * vol_id, owned_id -- hold id_range entries; only the range is checked) */
    int64_t id_range;
    /* skin lists kept across advective steps (sph_engine_maintain_lists):
     * per particle in physical order (dev) the cell key of the current CLL
     * (key_sorted; walls: their static cell), the key of the PREVIOUS CLL
     * (key_prev, fluid), the last re-sort's permutation (new i <- old
     * perm[i]) and its inverse; the second list / count buffers the
     * maintenance writes (swapped with lists / lcount).  NULL: lists are
     * rebuilt every step.  lists_stale: the lists were valid before the last
     * CLL rebuild (library state). */
    uint32_t* key_sorted; uint32_t* key_prev; uint32_t* perm; uint32_t* inv;
    int32_t* lists_alt; int32_t* lcount_alt;
    int32_t lists_stale;
    /* library state: 1 while the cell order and offsets were computed from
     * the current positions (set by a push or a CLL rebuild, cleared by
     * anything that moves particles), so a list build can take each
     * particle's cell from the CLL instead of recomputing it */
    int32_t cll_fresh;
    /* local displacement bound (f32 runs with the persistent arrays): per
     * grid cell (dev, ncells) the largest path length since the lists' build
     * of the particles whose CLL cell it is (cellmax, float bits) and its
     * maximum over the cell's 3^d block (blockmax); a list's validity test
     * then uses its own block's bound instead of the global maximum.  NULL:
     * the global bound (SphStepStats.dmax_bits). */
    uint32_t* cellmax; uint32_t* blockmax;
} SphEngine;

size_t sph_engine_workspace_bytes(int64_t n, int64_t ncells, int32_t f64);
/* the same for an engine with SphEngine.id_range > 0 */
size_t sph_engine_workspace_bytes_ids(int64_t n, int64_t ncells, int32_t f64, int64_t id_range);
/* Registry-order (n,d)/(n,) device arrays <-> engine SoA.  push lays the
 * particles out (fluid/wall split, cell order) and records refpos. */
int sph_engine_push(SphEngine* e, const void* x, const void* v, const void* rho, const void* p,
                    const void* m, const void* vol, const void* drho, const void* dvdt,
                    const void* rho_scratch, const uint32_t* id, const uint32_t* wall,
                    const uint32_t* nnb, const uint32_t* oflow, cudaStream_t s);
/* the same push in two halves, so that the registry's upload can overlap
 * the first step's list build: push_begin needs only x, id and wall (id
 * range check, fluid count, cell order, positions, refpos; counts the fluid
 * clamps of this cell order into stats->oob, which the following step's CLL
 * would count); push_end gathers every other field by refpos and checks the
 * ids for duplicates.  push_begin + push_end on one stream ==
 * sph_engine_push; stats->push_error / fluid_seen are final after push_end. */
int sph_engine_push_begin(SphEngine* e, const void* x, const uint32_t* id, const uint32_t* wall,
                          cudaStream_t s);
int sph_engine_push_end(SphEngine* e, const void* v, const void* rho, const void* p,
                        const void* m, const void* vol, const void* drho, const void* dvdt,
                        const void* rho_scratch, const uint32_t* nnb, const uint32_t* oflow,
                        cudaStream_t s);
/* push_end may leave vol, rho_scratch and oflow NULL and deliver them later
 * with push_tail (registry-order ids + those fields; any may be NULL), e.g.
 * after the step's sub-steps: the step reads none of them (rho_scratch only
 * on a Shepard step, which must not defer it); a deferred oflow yields
 * to the overflow flags (1) the step set meanwhile, as the pushed value
 * would have. */
int sph_engine_push_tail(SphEngine* e, const uint32_t* id, const void* vol,
                         const void* rho_scratch, const uint32_t* oflow, cudaStream_t s);
int sph_engine_pull(const SphEngine* e, void* x, void* v, void* rho, void* p, void* m, void* vol,
                    void* drho, void* dvdt, void* rho_scratch, uint32_t* id, uint32_t* wall,
                    uint32_t* nnb, uint32_t* oflow, cudaStream_t s);
/* the fields of mask only (bit k = the k-th array argument of
 * sph_engine_pull: x, v, rho, p, m, vol, drho, dvdt, rho_scratch, id, wall,
 * nnb, oflow); the others may be NULL */
int sph_engine_pull_fields(const SphEngine* e, uint32_t mask, void* x, void* v, void* rho,
                           void* p, void* m, void* vol, void* drho, void* dvdt,
                           void* rho_scratch, uint32_t* id, uint32_t* wall, uint32_t* nnb,
                           uint32_t* oflow, cudaStream_t s);
/* physics.py:446-449 _rebuild_cll on the engine layout: re-sort the fluid
 * segment by cell, rebuild the segment offsets; counts clamps into stats. */
int sph_engine_rebuild_cll(SphEngine* e, cudaStream_t s);
/* sorting.py:84-87 sort_particles_by_cell, tracked for the registry mirror */
int sph_engine_ref_sort(SphEngine* e, cudaStream_t s);
/* Verlet skin lists for the step (after every rebuild): for each particle the
 * ascending-id list of CLL-block neighbours within cutoff + skin of its
 * current position; resets the displacement bounds.  Every later sweep
 * filters them exactly (0 < r2 < cutoff^2 on current positions) and falls
 * back to an exact rebuild for a particle whose cell changed or whose
 * displacement bound exceeds the skin, so results are the reference's. */
int sph_engine_build_lists(SphEngine* e, double skin, cudaStream_t s);
/* carry the skin lists of the previous advective step across this step's
 * CLL rebuild instead of rebuilding them (same skin; needs the persistent
 * arrays above): entries are renumbered through the re-sort, entries whose
 * current CLL cell left the particle's 3^d block are dropped, particles
 * that moved INTO the block since the previous CLL are merged in id order
 * when within cutoff + skin; particles whose list is no longer valid (cell
 * change, displacement since the list build + the largest displacement
 * since the full build > skin) get a fresh list of their current block */
int sph_engine_maintain_lists(SphEngine* e, cudaStream_t s);
/* physics.py:460-467 initialize: wall pressure + momentum + counts */
int sph_engine_initialize(SphEngine* e, cudaStream_t s);
/* physics.py:469-487 _shepard_filter (SHEPARD, COPY_SCALAR, DENSITY_UPDATE) */
int sph_engine_shepard(SphEngine* e, cudaStream_t s);
/* physics.py:522-548 one acoustic sub-step: KICK, DRIFT, CONTINUITY,
 * DENSITY_UPDATE, WALL_PRESSURE, MOMENTUM, KICK (fused) */
int sph_engine_substep(SphEngine* e, double half_dt, double full_dt, cudaStream_t s);
/* nsub consecutive sub-steps of one advective step (physics.py:522-548): the
 * momentum sweep of every sub-step but the last also applies the next
 * sub-step's KICK + DRIFT (same dt), writing positions to the other buffer,
 * so one pass over the particles disappears per sub-step */
int sph_engine_substeps(SphEngine* e, double half_dt, double full_dt, int32_t nsub,
                        cudaStream_t s);
/* the same, synchronised, with the CUDA-event time of each of the five
 * parts summed over the sub-steps (ms_out[5]; see sph_engine_substep_timed) */
/* sph_engine_substeps, recording x_final on s once the last sub-step's
 * positions are final and rp_final once its rho, p and drho are (after its
 * wall-pressure sweep): a registry pull of those fields can start there,
 * overlapping the step's momentum sweep */
int sph_engine_substeps_marked(SphEngine* e, double half_dt, double full_dt, int32_t nsub,
                               cudaEvent_t x_final, cudaEvent_t rp_final, cudaStream_t s);
int sph_engine_substeps_timed(SphEngine* e, double half_dt, double full_dt, int32_t nsub,
                              float* ms_out, cudaStream_t s);
/* the same sub-step, synchronised, with CUDA-event times (ms) of its five
 * kernels: kick+drift, neighbour lists, continuity+density update, wall
 * pressure, momentum+kick (bench.py per-kernel roofline) */
int sph_engine_substep_timed(SphEngine* e, double half_dt, double full_dt, float* ms_out,
                             cudaStream_t s);
/* flags & 1: reset the per-step counters (interactions, overflow, oob, nfix);
 * flags & 2: recompute the exact vmax/amax (physics.py:390-391) and the
 * stability inputs (physics.py:554-564) into e->stats */
int sph_engine_stats(SphEngine* e, int flags, cudaStream_t s);
/* binary snapshot (report.py:187-205 fields, by original id): out (dev) is
 * an (n, 2*dim + 2) run-precision row-major array, row = particle id,
 * columns x[dim], v[dim], rho, p of the current state */
int sph_engine_snapshot(const SphEngine* e, void* out, cudaStream_t s);
/* physics.py:589-606 sample_pressure, device half: records (registry
 * position, x, y, z, m, rho, p) as binary64 of the fluid particles with
 * |x - loc| < radius (binary64), at most cap of them (*count = all found;
 * loc: host array of 3) */
int sph_engine_probe(const SphEngine* e, const double* loc, double radius, double* out,
                     int32_t cap, unsigned int* count, cudaStream_t s);

/* ---- multi-rank slab decomposition ------------------------
 * The sub-step and initialize split at the points where halo data must be
 * exchanged between ranks; sph_engine_substep == phases 0..3. */
#define SPH_PHASE_KICK_DRIFT 0      /* KICK + DRIFT of owned fluid, m/rho operands  */
#define SPH_PHASE_CONTINUITY 1      /* list upkeep, CONTINUITY + DENSITY_UPDATE      */
#define SPH_PHASE_WALL 2            /* WALL_PRESSURE into the sub-step's rp buffer   */
#define SPH_PHASE_MOMENTUM 3        /* MOMENTUM + KICK; the sub-step's buffers become
                                       current                                      */
#define SPH_PHASE_INIT_WALL 4       /* initialize: exact lists + WALL_PRESSURE       */
#define SPH_PHASE_INIT_MOMENTUM 5   /* initialize: MOMENTUM (no kick)                */
#define SPH_PHASE_MOMENTUM_NEXT 6   /* MOMENTUM + KICK + the NEXT sub-step's KICK +
                                       DRIFT of owned fluid (same dt); the next
                                       KICK_DRIFT phase is then a no-op           */
int sph_engine_phase(SphEngine* e, int32_t phase, double half_dt, double full_dt,
                     cudaStream_t s);
/* Halo records of the particles at physical indices phys[0..count), packed
 * as count x width run-precision values (owner side) and written back into
 * the ghosts (receiver side):
 *   XV      pos (x, y, z, m), current vel (x, y, z, m/rho), displacement
 *           bound since the list build; unpack re-checks the ghost's list
 *           cell and folds the bound into the step's maximum displacement
 *   RP_NEXT (rho, p) of the in-flight sub-step buffer (after CONTINUITY or
 *           WALL phases)
 *   RP_CUR  (rho, p) of the current buffer (after Shepard / INIT_WALL) */
#define SPH_HALO_XV 0
#define SPH_HALO_RP_NEXT 1
#define SPH_HALO_RP_CUR 2
int32_t sph_engine_halo_width(int32_t kind);
int sph_engine_pack(const SphEngine* e, int32_t kind, const int32_t* phys, int64_t count,
                    void* out, cudaStream_t s);
int sph_engine_unpack(SphEngine* e, int32_t kind, const int32_t* phys, int64_t count,
                      const void* in, cudaStream_t s);

/* Halo plan of one rank for one advective step: per record class (0 = fluid
 * ghosts, 1 = wall ghosts) the physical indices of the records this rank
 * sends (its owned particles in the neighbours' halos) and of its ghosts,
 * each concatenated over the peers in peer order, with per-peer record
 * offsets; send_buf / recv_buf are device staging of >= 9 run-precision
 * values per record of the larger class total. */
#define SPH_MAX_PEERS 8
typedef struct {
    int32_t npeers;
    int32_t peer[SPH_MAX_PEERS];
    const int32_t* send_phys[2];
    const int32_t* recv_phys[2];
    int64_t send_off[2][SPH_MAX_PEERS + 1];
    int64_t recv_off[2][SPH_MAX_PEERS + 1];
    void* send_buf;
    void* recv_buf;
} SphHaloPlan;
/* pack every record of class cls into send_buf / unpack recv_buf into the
 * ghosts (the transport in between is the caller's: NCCL below, or any
 * host-staged one) */
int sph_halo_pack(const SphEngine* e, const SphHaloPlan* plan, int32_t kind, int32_t cls,
                  cudaStream_t s);
int sph_halo_unpack(SphEngine* e, const SphHaloPlan* plan, int32_t kind, int32_t cls,
                    cudaStream_t s);
/* NCCL communicator among the ranks (libnccl.so.2 is opened on first use:
 * the copy the process already loaded, e.g. torch's, else the system one) */
size_t sph_comm_id_bytes(void);
int sph_comm_unique_id(void* id_out);
int sph_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm_out);
int sph_comm_destroy(void* comm);
/* pack, grouped ncclSend/ncclRecv with every peer, unpack -- all on s */
int sph_halo_exchange(SphEngine* e, void* comm, const SphHaloPlan* plan, int32_t kind,
                      int32_t cls, cudaStream_t s);
/* the step statistics (e->stats) of all ranks reduced in place with NCCL
 * on s: flags & 1 vmax / amax (max); & 2 interactions, overflow and
 * refresh counts (sum); & 4 min rho (min), max run-precision |v|^2 (max)
 * and the NaN flags (or) -- the host then reads global values once */
int sph_stats_allreduce(SphEngine* e, void* comm, int32_t flags, cudaStream_t s);
/* the nsub sub-steps of a slab rank with the halo refreshes between the
 * phases (XV of fluid ghosts after KICK_DRIFT, RP_NEXT of fluid ghosts after
 * CONTINUITY, RP_NEXT of wall ghosts after WALL), one host call per step */
int sph_engine_substeps_slab(SphEngine* e, void* comm, const SphHaloPlan* plan, double half_dt,
                             double full_dt, int32_t nsub, cudaStream_t s);

/* ---- slab bookkeeping (distributed.py) ---------------------
 * A rank's particles in registry layout (distributed.FIELDS order): x[d],
 * v[d], rho, p, m, Vol, drho, dvdt[d], rho_scratch (run precision), id,
 * wall, nnb, oflow (uint32); device pointers, row-major. */
typedef struct {
    void* f[13];
} SphRows;
#define SPH_MAX_RANKS 64
/* slab layout seen by one rank: rank r owns axis-0 cell planes
 * [cuts[r], cuts[r+1]); halo = planes within `halo` outside a slab (ring
 * distance when periodic); peers = the ranks exchanged with */
typedef struct {
    int64_t nplanes;                  /* == shape[0] */
    double origin[3], cell_size;      /* grid (run-precision values) */
    int64_t shape[3];
    int32_t nranks, rank, periodic, halo;
    int64_t cuts[SPH_MAX_RANKS + 1];
    int32_t npeers;
    int32_t peer[SPH_MAX_PEERS];
} SphSlabGeom;
/* int32 words of one packed row record */
int32_t sph_slab_record_words(int32_t dim, int32_t f64);
/* classify rows [0, n) by the axis-0 cell plane of x (neighborhood.py:76-84
 * binning): lists (dev, (3 npeers + 1) x n) get per peer k the rows moving to
 * peer k (list 3k), the kept rows in peer k's halo, fluid (3k+1) and wall
 * (3k+2), and all kept rows (list 3 npeers); counts (dev, 3 npeers + 3) the
 * list lengths, then counts[3 npeers + 1] > 0 when a row's new owner is no
 * peer and counts[3 npeers + 2] = rows whose cell key clamps on some axis
 * (the reference's out-of-bounds count, neighborhood.py:79-84) */
int sph_slab_classify(const SphSlabGeom* g, const void* x, const uint32_t* wall, int64_t n,
                      int32_t dim, int32_t f64, int32_t* lists, int32_t* counts, cudaStream_t s);
/* records (n x words int32) <- rows[k] of in (rows == NULL: rows 0..n-1) */
int sph_slab_pack(const SphRows* in, int32_t dim, int32_t f64, const int32_t* rows, int64_t n,
                  void* out, cudaStream_t s);
/* rows [dst_off, dst_off + n) of out <- records */
int sph_slab_unpack(const void* records, int64_t n, const SphRows* out, int32_t dim, int32_t f64,
                    int64_t dst_off, cudaStream_t s);
/* rows [dst_off, dst_off + n) of out <- rows[k] of in */
int sph_slab_gather(const SphRows* in, const int32_t* rows, int64_t n, const SphRows* out,
                    int32_t dim, int32_t f64, int64_t dst_off, cudaStream_t s);

#ifdef __cplusplus
}
#endif
#endif /* SPH_B200_H */
