/* sph_oracle.c -- CPU restatement of the reference WCSPH hot path.
 *
 * TEST INFRASTRUCTURE: the parity checker for the CUDA product path and the
 * CPU baseline arm of bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline / --impl reference) may load it.  It is never on the
 * product path.
 *
 * The reference (/root/reference/pkg/src/minisph) is Python + numba; this file
 * restates the algorithm of each @njit body in C, one function per reference
 * symbol, each citing file:line.  The arithmetic contract (which operations are
 * binary32 and which binary64) is the numba typing of those bodies; see
 * sph_oracle_impl.h.  Pinned against fixtures generated from the reference
 * itself (tests/golden/make_goldens.py).
 */

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_CAP 256            /* neighborhood.py:30 NEIGHBOR_CAPACITY */
#define ORC_ERR_OVERFLOW 1     /* NeighborOverflowError */
#define ORC_ERR_UNSTABLE_RHO 2 /* SimulationUnstableError, rho <= 0 */
#define ORC_ERR_UNSTABLE_V 3   /* SimulationUnstableError, runaway velocity */

int orc_abi_version(void) { return 1; }

/* Ascending sort of packed (id << 32 | j) keys; every key is unique, so any
 * correct sort reproduces numpy's buf[:n].sort() (neighborhood.py:226). */
void orc_sort_i64(int64_t *a, int n)
{
    /* insertion sort on runs of 16, then bottom-up merges */
    int64_t tmp[ORC_CAP];
    const int RUN = 16;
    for (int lo = 0; lo < n; lo += RUN) {
        int hi = lo + RUN < n ? lo + RUN : n;
        for (int i = lo + 1; i < hi; i++) {
            int64_t v = a[i];
            int j = i - 1;
            while (j >= lo && a[j] > v) { a[j + 1] = a[j]; j--; }
            a[j + 1] = v;
        }
    }
    int64_t *src = a, *dst = tmp;
    for (int w = RUN; w < n; w *= 2) {
        for (int lo = 0; lo < n; lo += 2 * w) {
            int mid = lo + w < n ? lo + w : n;
            int hi = lo + 2 * w < n ? lo + 2 * w : n;
            int p = lo, q = mid, o = lo;
            while (p < mid && q < hi) dst[o++] = src[p] <= src[q] ? src[p++] : src[q++];
            while (p < mid) dst[o++] = src[p++];
            while (q < hi) dst[o++] = src[q++];
        }
        int64_t *t = src; src = dst; dst = t;
    }
    if (src != a) memcpy(a, src, sizeof(int64_t) * (size_t)n);
}

/* neighborhood.py:120-173 count / exclusive prefix / scatter: a stable
 * counting sort by key.  particle_ids == argsort(keys, kind="stable"),
 * offsets = exclusive prefix of per-cell counts (offsets[C] = n). */
void orc_counting_sort(const int64_t *keys, int64_t n, int64_t ncells,
                       int64_t *offsets, int64_t *pids)
{
    memset(offsets, 0, sizeof(int64_t) * (size_t)(ncells + 1));
    for (int64_t i = 0; i < n; i++) offsets[keys[i] + 1]++;
    for (int64_t c = 0; c < ncells; c++) offsets[c + 1] += offsets[c];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncells ? ncells : 1));
    memcpy(cursor, offsets, sizeof(int64_t) * (size_t)ncells);
    for (int64_t i = 0; i < n; i++) pids[cursor[keys[i]]++] = i;
    free(cursor);
}

/* sorting.py:46-70 radix_sort_permutation: LSD passes of 8-bit digits,
 * passes = max(1, ceil(bit_length(max_key) / 8)); each pass a stable
 * counting scatter.  Returns -1 on a negative key (sorting.py:52-53). */
int orc_radix_sort_perm(const int64_t *keys, int64_t n, int64_t *perm)
{
    if (n == 0) return 0;
    int64_t mx = 0;
    for (int64_t i = 0; i < n; i++) {
        if (keys[i] < 0) return -1;
        if (keys[i] > mx) mx = keys[i];
    }
    int bits = 0;
    while (bits < 64 && (mx >> bits) != 0) bits++;
    int passes = (bits + 7) / 8;
    if (passes < 1) passes = 1;
    int64_t *out = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *cur = perm;
    for (int64_t i = 0; i < n; i++) cur[i] = i;
    for (int p = 0; p < passes; p++) {
        int shift = p * 8;
        int64_t count[257];
        memset(count, 0, sizeof(count));
        for (int64_t s = 0; s < n; s++) count[((keys[cur[s]] >> shift) & 255) + 1]++;
        for (int b = 0; b < 256; b++) count[b + 1] += count[b];
        for (int64_t s = 0; s < n; s++) {
            int64_t q = cur[s];
            out[count[(keys[q] >> shift) & 255]++] = q;
        }
        int64_t *t = cur; cur = out; out = t;
    }
    if (cur != perm) { memcpy(perm, cur, sizeof(int64_t) * (size_t)n); out = cur; }
    free(out);
    return 0;
}

/* sorting.py:22-24 comparison_sort_permutation == stable argsort; the same
 * permutation as the radix route. */
void orc_stable_argsort(const int64_t *keys, int64_t n, int64_t *perm)
{
    int64_t mn = 0;
    for (int64_t i = 0; i < n; i++) if (keys[i] < mn) mn = keys[i];
    if (mn >= 0) { orc_radix_sort_perm(keys, n, perm); return; }
    /* negative keys: bias into the unsigned range first */
    int64_t *k2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; i++) k2[i] = keys[i] - mn;
    orc_radix_sort_perm(k2, n, perm);
    free(k2);
}

/* physics.py:386-400 compute_timestep host arithmetic (Python doubles). */
void orc_timestep_formula(double vmax, double amax, double h, double c0,
                          double dt_max, double cfl_acoustic,
                          double cfl_advective, double *dt_ac, double *dt_adv)
{
    double dt_acoustic = cfl_acoustic * h / (c0 + vmax);
    double dt_advective = dt_max;
    if (vmax > 0.0) {
        double c = cfl_advective * h / vmax;
        if (c < dt_advective) dt_advective = c;
    }
    if (amax > 0.0) {
        double c = cfl_advective * sqrt(h / amax);
        if (c < dt_advective) dt_advective = c;
    }
    *dt_ac = dt_acoustic;
    *dt_adv = dt_advective;
}

#define R float
#define SFX _f32
#define SQRT sqrtf
#define FLOOR floorf
#include "sph_oracle_impl.h"
#undef R
#undef SFX
#undef SQRT
#undef FLOOR

#define R double
#define SFX _f64
#define SQRT sqrt
#define FLOOR floor
#include "sph_oracle_impl.h"
#undef R
#undef SFX
#undef SQRT
#undef FLOOR
