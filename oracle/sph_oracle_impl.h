/* CPU restatement of the reference WCSPH particle step, one precision.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/README.md): included twice by
 * sph_oracle.c with R = float (suffix _f32, the reference's precision="f32"
 * run) and R = double (suffix _f64).  In the f32 instantiation every
 * expression follows the numba typing of the reference bodies: operations on
 * array elements / f32 scalars are binary32, any operand that meets a Python
 * float literal is widened to binary64.  Built with
 * -ffp-contract=off and without -ffast-math so no FMA contraction happens,
 * exactly like the numba-compiled kernels (0 vfmadd in every JIT kernel).
 *
 * Reference line numbers: /root/reference/pkg/src/minisph/<file>:<line>.
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)

/* force_args field order, physics.py:77-80 / 315-330 (+ rho_new for the
 * Shepard shell, physics.py:473-478). Vectors are (n, d) row-major. */
typedef struct {
    int64_t n; int d;
    R *x, *v, *rho, *p, *m;
    uint32_t *wall, *ids;
    R *g;
    int64_t *offsets, *pids;
    R *origin; int64_t *shape;
    R *drho, *dvdt;
    uint32_t *nnb, *oflow;
    R cell_size, cutoff, h, alpha_d, c0, rho0, alpha_visc, eps_h2;
    R *rho_new;
} FN(orc_args);

/* ---- periodic boxes: NOT in the reference ---------------
 * The builder's own extension, restated here so the CUDA periodic build has
 * a checker (parity of this part is against this restatement only).  Per
 * axis k: L > 0 makes the axis periodic over [lo, hi) (hi = RN(lo + L),
 * both run precision, set by the caller).  Pair differences take the
 * minimum image (dx > L/2: dx - L; dx < -L/2: dx + L; one rounding), the
 * 3^d block wraps on periodic axes (shape >= 3), and a drift leaving
 * [lo, hi) re-enters by one +-L.  All zero = the reference's bounded box. */
static R FN(box_L)[3], FN(box_hL)[3], FN(box_lo)[3], FN(box_hi)[3];

void FN(orc_set_box)(const R *L, const R *lo, const R *hi, int d)
{
    for (int k = 0; k < 3; k++) {
        FN(box_L)[k] = (L && k < d) ? L[k] : (R)0;
        FN(box_hL)[k] = (R)(FN(box_L)[k] * (R)0.5);
        FN(box_lo)[k] = (L && k < d) ? lo[k] : (R)0;
        FN(box_hi)[k] = (L && k < d) ? hi[k] : (R)0;
    }
}

static inline R FN(min_image)(R dx, int k)
{
    R L = FN(box_L)[k];
    if (L > (R)0) {
        if (dx > FN(box_hL)[k]) dx = (R)(dx - L);
        else if (dx < -FN(box_hL)[k]) dx = (R)(dx + L);
    }
    return dx;
}

static inline R FN(wrap_coord)(R x, int k)
{
    R L = FN(box_L)[k];
    if (L > (R)0) {
        if (x >= FN(box_hi)[k]) x = (R)(x - L);
        else if (x < FN(box_lo)[k]) x = (R)(x + L);
    }
    return x;
}

/* the cells of axis k around c: *n of them into a[] (wrapped or clamped) */
static inline int FN(block_axis)(int64_t c, int64_t s, int k, int64_t *a)
{
    if (FN(box_L)[k] > (R)0) {
        a[0] = c == 0 ? s - 1 : c - 1; a[1] = c; a[2] = c + 1 == s ? 0 : c + 1;
        return 3;
    }
    int n = 0;
    for (int64_t t = c - 1; t <= c + 1; t++)
        if (t >= 0 && t < s) a[n++] = t;
    return n;
}

/* neighborhood.py:76-84  _cell_coord: floor((x - origin) / cell_size),
 * clamped to [0, ncells-1]; *clamped set on a clamp. */
static inline int64_t FN(cell_coord)(R x, R origin, R cell_size,
                                     int64_t ncells, int *clamped)
{
    R t = (R)(x - origin);
    t = (R)(t / cell_size);
    R f = FLOOR(t);
    /* x86 cvttss2si/cvttsd2si (numba's int()) yields INT64_MIN for NaN and
     * out-of-range values; C leaves that undefined, so spell it out. */
    int64_t c = (f >= (R)-9.2233720368547758e18 && f < (R)9.2233720368547758e18)
                    ? (int64_t)f : INT64_MIN;
    if (c < 0) { *clamped = 1; return 0; }
    if (c >= ncells) { *clamped = 1; return ncells - 1; }
    return c;
}

/* neighborhood.py:105-117  _compute_keys */
void FN(orc_compute_keys)(const R *pos, int64_t n, int d, const R *origin,
                          R cell_size, const int64_t *shape, int64_t *keys,
                          uint8_t *oob)
{
    for (int64_t i = 0; i < n; i++) {
        int64_t lin = 0;
        int clamped = 0;
        for (int k = 0; k < d; k++) {
            int cl = 0;
            int64_t c = FN(cell_coord)(pos[i * d + k], origin[k], cell_size,
                                       shape[k], &cl);
            clamped |= cl;
            lin = lin * shape[k] + c;
        }
        keys[i] = lin;
        oob[i] = (uint8_t)clamped;
    }
}

/* neighborhood.py:176-227  collect_neighbors.  Packs (id << 32 | j) for every
 * j != i of the clamped 3^d block around i's CURRENT cell with 0 < r2 < c2
 * (binary32 r2, dx0^2 + dx1^2 [+ dx2^2] left to right), sorts ascending.
 * Returns the count, or -1 when more than cap neighbours qualify. */
int FN(orc_collect_neighbors)(int64_t i, const R *pos, int d,
                              const uint32_t *ids, const int64_t *offsets,
                              const int64_t *pids, const R *origin,
                              R cell_size, const int64_t *shape, R cutoff,
                              int64_t *buf, int cap)
{
    R c2 = (R)(cutoff * cutoff);
    int n = 0;
    int cl = 0;
    int64_t cx = FN(cell_coord)(pos[i * d + 0], origin[0], cell_size, shape[0], &cl);
    int64_t cy = FN(cell_coord)(pos[i * d + 1], origin[1], cell_size, shape[1], &cl);
    int64_t cz = 0;
    if (d == 3)
        cz = FN(cell_coord)(pos[i * d + 2], origin[2], cell_size, shape[2], &cl);
    /* the clamped (or, on periodic axes, wrapped) 3^d block */
    int64_t bx[3], by[3], bz[3] = {0, 0, 0};
    int nx = FN(block_axis)(cx, shape[0], 0, bx);
    int ny = FN(block_axis)(cy, shape[1], 1, by);
    int nz = d == 3 ? FN(block_axis)(cz, shape[2], 2, bz) : 1;
    for (int tx = 0; tx < nx; tx++)
        for (int ty = 0; ty < ny; ty++)
            for (int tz = 0; tz < nz; tz++) {
                int64_t ax = bx[tx], ay = by[ty], az = bz[tz];
                int64_t lin = (d == 3) ? (ax * shape[1] + ay) * shape[2] + az
                                       : ax * shape[1] + ay;
                for (int64_t s = offsets[lin]; s < offsets[lin + 1]; s++) {
                    int64_t j = pids[s];
                    if (j == i) continue;
                    R r2;
                    R dx = FN(min_image)((R)(pos[i * d + 0] - pos[j * d + 0]), 0);
                    R dy = FN(min_image)((R)(pos[i * d + 1] - pos[j * d + 1]), 1);
                    r2 = (R)((R)(dx * dx) + (R)(dy * dy));
                    if (d == 3) {
                        R dz = FN(min_image)((R)(pos[i * d + 2] - pos[j * d + 2]), 2);
                        r2 = (R)(r2 + (R)(dz * dz));
                    }
                    if (r2 < c2 && (double)r2 > 0.0) {
                        if (n >= cap) return -1;
                        buf[n++] = ((int64_t)ids[j] << 32) | j;
                    }
                }
            }
    orc_sort_i64(buf, n);
    return n;
}

/* physics.py:82-91  _pair_geometry (binary32, accumulated from 0) */
static inline void FN(pair_geometry)(int64_t i, int64_t j, int d, const R *x,
                                     const R *v, R *r2o, R *vxo)
{
    R r2 = (R)(x[i * d] - x[i * d]);
    R vx = r2;
    for (int k = 0; k < d; k++) {
        R dxk = FN(min_image)((R)(x[i * d + k] - x[j * d + k]), k);
        r2 = (R)(r2 + (R)(dxk * dxk));
        vx = (R)(vx + (R)((R)(v[i * d + k] - v[j * d + k]) * dxk));
    }
    *r2o = r2;
    *vxo = vx;
}

/* gw/r factor of the Wendland C2 gradient, physics.py:113-117 / 146-150:
 * tq = 1.0 - 0.5*q; gw = -5.0*alpha_d*q*tq*tq*tq/h; fac = gw/r (binary64). */
static inline double FN(grad_fac)(R r, R q, R h, R alpha_d)
{
    double tq = 1.0 - 0.5 * (double)q;
    double gw = -5.0 * (double)alpha_d;
    gw = gw * (double)q;
    gw = gw * tq;
    gw = gw * tq;
    gw = gw * tq;
    gw = gw / (double)h;
    return gw / (double)r;
}

/* Wendland C2 value, physics.py:184-186: alpha_d*tq^4*(2q+1) (binary64). */
static inline double FN(kernel_w)(R q, R alpha_d)
{
    double tq = 1.0 - 0.5 * (double)q;
    double w = (double)alpha_d * tq;
    w = w * tq;
    w = w * tq;
    w = w * tq;
    return w * (2.0 * (double)q + 1.0);
}

#define SWEEP_PRELUDE                                                       \
    int64_t buf[ORC_CAP];                                                   \
    int cnt = FN(orc_collect_neighbors)(i, a->x, a->d, a->ids, a->offsets,  \
                                        a->pids, a->origin, a->cell_size,   \
                                        a->shape, a->cutoff, buf, ORC_CAP);

/* physics.py:94-119  _continuity_body */
static void FN(continuity_one)(const FN(orc_args) *a, int64_t i)
{
    if (a->wall[i] != 0) { a->drho[i] = 0; return; }
    SWEEP_PRELUDE
    if (cnt < 0) { a->oflow[i] = 1; return; }
    const int d = a->d;
    R rho_i = a->rho[i];
    double acc = (double)(R)(rho_i - rho_i);
    for (int t = 0; t < cnt; t++) {
        int64_t j = buf[t] & 0xFFFFFFFFLL;
        R r2, vx;
        FN(pair_geometry)(i, j, d, a->x, a->v, &r2, &vx);
        R r = SQRT(r2);
        R q = (R)(r / a->h);
        double fac = FN(grad_fac)(r, q, a->h, a->alpha_d);
        R mr = (R)(a->m[j] / a->rho[j]);
        R mv = (R)(mr * vx);
        acc = acc + (double)mv * fac;
    }
    a->drho[i] = (R)((double)rho_i * acc);
}

/* physics.py:122-158  _momentum_body */
static void FN(momentum_one)(const FN(orc_args) *a, int64_t i)
{
    const int d = a->d;
    if (a->wall[i] != 0) {
        for (int k = 0; k < d; k++) a->dvdt[i * d + k] = 0;
        return;
    }
    SWEEP_PRELUDE
    if (cnt < 0) { a->oflow[i] = 1; return; }
    R rho_i = a->rho[i];
    R p_i = a->p[i];
    R pi_rr = (R)(p_i / (R)(rho_i * rho_i));
    for (int k = 0; k < d; k++) a->dvdt[i * d + k] = a->g[k];
    R avc = (R)(a->alpha_visc * a->c0);
    R avch = (R)(avc * a->h);
    for (int t = 0; t < cnt; t++) {
        int64_t j = buf[t] & 0xFFFFFFFFLL;
        R r2, vx;
        FN(pair_geometry)(i, j, d, a->x, a->v, &r2, &vx);
        R r = SQRT(r2);
        R q = (R)(r / a->h);
        double fac = FN(grad_fac)(r, q, a->h, a->alpha_d);
        R rho_j = a->rho[j];
        double pij = (double)(R)(pi_rr + (R)(a->p[j] / (R)(rho_j * rho_j)));
        if ((double)vx < 0.0) {
            R num = (R)(-(R)(avch * vx));
            double den = 0.5 * (double)(R)(rho_i + rho_j);
            den = den * (double)(R)(r2 + a->eps_h2);
            pij = pij + (double)num / den;
        }
        double f = (double)(R)(-a->m[j]) * pij;
        f = f * fac;
        for (int k = 0; k < d; k++) {
            R dxk = FN(min_image)((R)(a->x[i * d + k] - a->x[j * d + k]), k);
            a->dvdt[i * d + k] = (R)((double)a->dvdt[i * d + k] + f * (double)dxk);
        }
    }
    a->nnb[i] = (uint32_t)cnt;
}

/* physics.py:161-194  _wall_pressure_body */
static void FN(wall_pressure_one)(const FN(orc_args) *a, int64_t i)
{
    if (a->wall[i] == 0) return;
    SWEEP_PRELUDE
    if (cnt < 0) { a->oflow[i] = 1; return; }
    const int d = a->d;
    double num = (double)(R)(a->rho[i] - a->rho[i]);
    double den = num;
    uint32_t visits = 0;
    for (int t = 0; t < cnt; t++) {
        int64_t j = buf[t] & 0xFFFFFFFFLL;
        if (a->wall[j] != 0) continue;
        visits++;
        R r2, vx;
        FN(pair_geometry)(i, j, d, a->x, a->v, &r2, &vx);
        R r = SQRT(r2);
        R q = (R)(r / a->h);
        double w = FN(kernel_w)(q, a->alpha_d);
        num = num + (double)a->p[j] * w;
        den = den + w;
    }
    if (den > 0.0) a->p[i] = (R)(num / den);
    else a->p[i] = 0;
    a->rho[i] = (R)(a->rho0 + (R)(a->p[i] / (R)(a->c0 * a->c0)));
    a->nnb[i] = visits;
}

/* physics.py:197-217  _density_summation_body (overflow: self term only) */
static void FN(density_summation_one)(const FN(orc_args) *a, int64_t i)
{
    SWEEP_PRELUDE
    if (cnt < 0) cnt = 0;
    const int d = a->d;
    double acc = (double)(R)(a->m[i] * a->alpha_d);
    for (int t = 0; t < cnt; t++) {
        int64_t j = buf[t] & 0xFFFFFFFFLL;
        R r2 = (R)(a->x[i * d] - a->x[i * d]);
        for (int k = 0; k < d; k++) {
            R dxk = FN(min_image)((R)(a->x[i * d + k] - a->x[j * d + k]), k);
            r2 = (R)(r2 + (R)(dxk * dxk));
        }
        R r = SQRT(r2);
        R q = (R)(r / a->h);
        double tq = 1.0 - 0.5 * (double)q;
        double term = (double)(R)(a->m[j] * a->alpha_d) * tq;
        term = term * tq;
        term = term * tq;
        term = term * tq;
        term = term * (2.0 * (double)q + 1.0);
        acc = acc + term;
    }
    a->rho[i] = (R)acc;
}

/* physics.py:220-247  _shepard_body, result into a->rho_new */
static void FN(shepard_one)(const FN(orc_args) *a, int64_t i)
{
    if (a->wall[i] != 0) { a->rho_new[i] = a->rho[i]; return; }
    SWEEP_PRELUDE
    if (cnt < 0) { a->rho_new[i] = a->rho[i]; return; }
    const int d = a->d;
    double num = (double)(R)(a->m[i] * a->alpha_d);
    double den = (double)(R)((R)(a->m[i] / a->rho[i]) * a->alpha_d);
    for (int t = 0; t < cnt; t++) {
        int64_t j = buf[t] & 0xFFFFFFFFLL;
        R r2 = (R)(a->x[i * d] - a->x[i * d]);
        for (int k = 0; k < d; k++) {
            R dxk = FN(min_image)((R)(a->x[i * d + k] - a->x[j * d + k]), k);
            r2 = (R)(r2 + (R)(dxk * dxk));
        }
        R r = SQRT(r2);
        R q = (R)(r / a->h);
        double w = FN(kernel_w)(q, a->alpha_d);
        num = num + (double)a->m[j] * w;
        den = den + (double)(R)(a->m[j] / a->rho[j]) * w;
    }
    a->rho_new[i] = (R)(num / den);
}

#define DEFINE_SWEEP(NAME)                                                  \
    void FN(orc_##NAME)(const FN(orc_args) *a)                              \
    {                                                                       \
        _Pragma("omp parallel for schedule(dynamic, 256)")                  \
        for (int64_t i = 0; i < a->n; i++) FN(NAME##_one)(a, i);            \
    }
DEFINE_SWEEP(continuity)
DEFINE_SWEEP(momentum)
DEFINE_SWEEP(wall_pressure)
DEFINE_SWEEP(density_summation)
DEFINE_SWEEP(shepard)

/* physics.py:250-256  _kick_body */
void FN(orc_kick)(int64_t n, int d, R *v, const R *dvdt, const uint32_t *wall,
                  R half_dt)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (wall[i] != 0) continue;
        for (int k = 0; k < d; k++)
            v[i * d + k] = (R)(v[i * d + k] + (R)(half_dt * dvdt[i * d + k]));
    }
}

/* physics.py:259-265  _drift_body */
void FN(orc_drift)(int64_t n, int d, R *x, const R *v, const uint32_t *wall,
                   R dt)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (wall[i] != 0) continue;
        for (int k = 0; k < d; k++)
            x[i * d + k] = FN(wrap_coord)((R)(x[i * d + k] + (R)(dt * v[i * d + k])), k);
    }
}

/* physics.py:268-274  _density_update_body */
void FN(orc_density_update)(int64_t n, R *rho, R *p, const R *drho,
                            const uint32_t *wall, R dt, R c0, R rho0)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (wall[i] != 0) continue;
        rho[i] = (R)(rho[i] + (R)(dt * drho[i]));
        p[i] = (R)((R)(c0 * c0) * (R)(rho[i] - rho0));
    }
}

/* physics.py:296-310  VMAX_SPEC: exact max over i of sqrt(sum_k f64(v_k*v_k))
 * (binary32 products, binary64 accumulation); identity 0.0.  The fold order
 * does not matter for an exact max. */
double FN(orc_vmax)(int64_t n, int d, const R *v)
{
    double best = 0.0;
    #pragma omp parallel for reduction(max:best) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double acc = 0.0;
        for (int k = 0; k < d; k++)
            acc = acc + (double)(R)(v[i * d + k] * v[i * d + k]);
        double s = sqrt(acc);
        if (s > best) best = s;
    }
    return best;
}

/* physics.py:554-564 _stability_check inputs: min rho and the binary32
 * max row norm sqrt(max_i sum_k v_k^2) numpy computes. */
void FN(orc_stability)(int64_t n, int d, const R *rho, const R *v,
                       double *rho_min, double *vmax)
{
    /* numpy min/max propagate NaN */
    R rmin = n ? rho[0] : 0;
    R s2max = 0;
    int nan_r = 0, nan_v = 0;
    for (int64_t i = 0; i < n; i++) {
        if (rho[i] != rho[i]) nan_r = 1;
        if (rho[i] < rmin) rmin = rho[i];
        R s = 0;
        for (int k = 0; k < d; k++) s = (R)(s + (R)(v[i * d + k] * v[i * d + k]));
        if (s != s) nan_v = 1;
        if (s > s2max) s2max = s;
    }
    *rho_min = nan_r ? NAN : (double)rmin;
    *vmax = nan_v ? NAN : (double)SQRT(s2max);
}

/* neighborhood.py:149-173  build_cell_linked_list on this precision's
 * positions; returns the out-of-bounds clamp count. */
int64_t FN(orc_build_cll)(const R *pos, int64_t n, int d, const R *origin,
                          R cell_size, const int64_t *shape, int64_t ncells,
                          int64_t *offsets, int64_t *pids, int64_t *keys_tmp)
{
    uint8_t *oob = (uint8_t *)malloc(n ? (size_t)n : 1);
    FN(orc_compute_keys)(pos, n, d, origin, cell_size, shape, keys_tmp, oob);
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; i++) cnt += oob[i];
    free(oob);
    orc_counting_sort(keys_tmp, n, ncells, offsets, pids);
    return cnt;
}

/* ---- whole advective step (physics.py:416-564) --------------------------- */

typedef struct {
    int64_t n; int d;
    R *x, *v, *rho, *p, *m, *Vol, *drho, *dvdt, *rho_scratch;
    uint32_t *id, *wall, *nnb, *oflow;
    R g[3];
    /* force_args host scalars, computed by the caller with NumPy-2 scalar
     * rules exactly as physics.py:315-330 does */
    R origin[3]; R cell_size, cutoff, h, alpha_d, c0, rho0, alpha_visc, eps_h2;
    int64_t shape[3]; int64_t ncells;
    /* host doubles (physics.py:392-393 float(h), float(c0)) */
    double h_d, c0_d;
    double dt_max, cfl_acoustic, cfl_advective, fixed_dt; int has_fixed_dt;
    int64_t sort_every, shepard_every;
    /* state */
    int64_t step_count; double time; int64_t interaction_count, out_of_bounds;
    int64_t *offsets, *pids, *keys;  /* CLL storage: ncells+1, n, n */
    double last_nsub;
    int sort_with_radix;   /* device policy in the reference -> radix */
} FN(orc_sim);

static void FN(sim_args)(FN(orc_sim) *s, FN(orc_args) *a)
{
    a->n = s->n; a->d = s->d;
    a->x = s->x; a->v = s->v; a->rho = s->rho; a->p = s->p; a->m = s->m;
    a->wall = s->wall; a->ids = s->id; a->g = s->g;
    a->offsets = s->offsets; a->pids = s->pids;
    a->origin = s->origin; a->shape = s->shape;
    a->drho = s->drho; a->dvdt = s->dvdt; a->nnb = s->nnb; a->oflow = s->oflow;
    a->rho_new = s->rho_scratch;
    a->cell_size = s->cell_size; a->cutoff = s->cutoff; a->h = s->h;
    a->alpha_d = s->alpha_d; a->c0 = s->c0; a->rho0 = s->rho0;
    a->alpha_visc = s->alpha_visc; a->eps_h2 = s->eps_h2;
}

static int FN(check_overflow)(FN(orc_sim) *s)
{
    for (int64_t i = 0; i < s->n; i++)
        if (s->oflow[i]) return ORC_ERR_OVERFLOW;
    return 0;
}

static void FN(rebuild_cll)(FN(orc_sim) *s)
{
    s->out_of_bounds += FN(orc_build_cll)(s->x, s->n, s->d, s->origin,
                                          s->cell_size, s->shape, s->ncells,
                                          s->offsets, s->pids, s->keys);
}

static void FN(count_interactions)(FN(orc_sim) *s, int continuity_pass)
{
    int64_t total = 0;
    for (int64_t i = 0; i < s->n; i++) total += s->nnb[i];
    if (continuity_pass)
        for (int64_t i = 0; i < s->n; i++)
            if (s->wall[i] == 0) total += s->nnb[i];
    s->interaction_count += total;
}

/* physics.py:460-467 */
int FN(orc_sim_initialize)(FN(orc_sim) *s)
{
    FN(orc_args) a;
    FN(rebuild_cll)(s);
    FN(sim_args)(s, &a);
    FN(orc_wall_pressure)(&a);
    if (FN(check_overflow)(s)) return ORC_ERR_OVERFLOW;
    FN(orc_momentum)(&a);
    if (FN(check_overflow)(s)) return ORC_ERR_OVERFLOW;
    FN(count_interactions)(s, 0);
    return 0;
}

/* sorting.py:84-87 + variables.py:132-145: reorder every discrete variable */
static void FN(sort_by_cell)(FN(orc_sim) *s)
{
    int64_t n = s->n; int d = s->d;
    uint8_t *oob = (uint8_t *)malloc(n ? (size_t)n : 1);
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    FN(orc_compute_keys)(s->x, n, d, s->origin, s->cell_size, s->shape,
                         s->keys, oob);
    free(oob);
    orc_stable_argsort(s->keys, n, perm);
    R *tr = (R *)malloc(sizeof(R) * (size_t)(n ? n : 1) * d);
    uint32_t *tu = (uint32_t *)malloc(sizeof(uint32_t) * (n ? n : 1));
#define PERM_VEC(arr) do { \
        for (int64_t k = 0; k < n; k++) \
            for (int c = 0; c < d; c++) tr[k * d + c] = arr[perm[k] * d + c]; \
        memcpy(arr, tr, sizeof(R) * n * d); \
    } while (0)
#define PERM_SCL(arr, tmp, T) do { \
        for (int64_t k = 0; k < n; k++) tmp[k] = arr[perm[k]]; \
        memcpy(arr, tmp, sizeof(T) * n); \
    } while (0)
    PERM_VEC(s->x); PERM_VEC(s->v); PERM_VEC(s->dvdt);
    PERM_SCL(s->rho, tr, R); PERM_SCL(s->p, tr, R); PERM_SCL(s->m, tr, R);
    PERM_SCL(s->Vol, tr, R); PERM_SCL(s->drho, tr, R);
    PERM_SCL(s->rho_scratch, tr, R);
    PERM_SCL(s->id, tu, uint32_t); PERM_SCL(s->wall, tu, uint32_t);
    PERM_SCL(s->nnb, tu, uint32_t); PERM_SCL(s->oflow, tu, uint32_t);
#undef PERM_VEC
#undef PERM_SCL
    free(tr); free(tu); free(perm);
}

/* physics.py:386-400 compute_timestep (host doubles) */
void FN(orc_sim_timestep)(FN(orc_sim) *s, double *dt_ac, double *dt_adv)
{
    double vmax = FN(orc_vmax)(s->n, s->d, s->v);
    double amax = FN(orc_vmax)(s->n, s->d, s->dvdt);
    orc_timestep_formula(vmax, amax, s->h_d, s->c0_d, s->dt_max,
                         s->cfl_acoustic, s->cfl_advective, dt_ac, dt_adv);
}

/* physics.py:489-552 Simulation.advance; end_time NaN == None.
 * Returns 0 or an ORC_ERR_* code; *dt_out = the advective dt taken. */
int FN(orc_sim_advance)(FN(orc_sim) *s, double end_time, double *dt_out)
{
    FN(orc_args) a;
    int64_t n = s->n; int d = s->d;
    if (s->sort_every && s->step_count > 0 && s->step_count % s->sort_every == 0)
        FN(sort_by_cell)(s);
    FN(rebuild_cll)(s);
    FN(sim_args)(s, &a);
    if (s->shepard_every && s->step_count > 0
            && s->step_count % s->shepard_every == 0) {
        FN(orc_shepard)(&a);                                  /* :479 */
        memcpy(s->rho, s->rho_scratch, sizeof(R) * n);        /* :480 */
        FN(orc_density_update)(n, s->rho, s->p, s->drho, s->wall, (R)0,
                               s->c0, s->rho0);               /* :485 */
    }
    double dt_ac, dt_adv;
    if (s->has_fixed_dt) { dt_ac = dt_adv = s->fixed_dt; }
    else FN(orc_sim_timestep)(s, &dt_ac, &dt_adv);
    double dt = dt_adv;
    if (!isnan(end_time)) { double rem = end_time - s->time; if (rem < dt) dt = rem; }
    double q = ceil(dt / dt_ac);
    int64_t nsub = (int64_t)q; if (nsub < 1) nsub = 1;
    double dts = dt / (double)nsub;
    s->last_nsub = (double)nsub;
    for (int64_t sub = 0; sub < nsub; sub++) {
        R half = (R)(0.5 * dts);
        R full = (R)dts;
        FN(orc_kick)(n, d, s->v, s->dvdt, s->wall, half);
        FN(orc_drift)(n, d, s->x, s->v, s->wall, full);
        FN(orc_continuity)(&a);
        if (FN(check_overflow)(s)) return ORC_ERR_OVERFLOW;
        FN(orc_density_update)(n, s->rho, s->p, s->drho, s->wall, full, s->c0,
                               s->rho0);
        FN(orc_wall_pressure)(&a);
        if (FN(check_overflow)(s)) return ORC_ERR_OVERFLOW;
        FN(orc_momentum)(&a);
        if (FN(check_overflow)(s)) return ORC_ERR_OVERFLOW;
        FN(count_interactions)(s, 1);
        FN(orc_kick)(n, d, s->v, s->dvdt, s->wall, half);
    }
    s->step_count += 1;
    s->time += dt;
    *dt_out = dt;
    double rmin, vm;
    FN(orc_stability)(n, d, s->rho, s->v, &rmin, &vm);
    if (n && rmin <= 0.0) return ORC_ERR_UNSTABLE_RHO;
    if (n && vm > 10.0 * s->c0_d) return ORC_ERR_UNSTABLE_V;
    return 0;
}

#undef SWEEP_PRELUDE
#undef DEFINE_SWEEP
#undef FN
#undef CAT
#undef CAT_
