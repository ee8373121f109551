// sweeps.cu -- the particle_for kernel-dispatch boundary on the reference
// layout (execution.py:121-129 driving physics.py:94-280 bodies).
//
// Each entry point takes the force_args tuple as SphSweepArgs_*, builds the
// ascending-id neighbour lists from the caller's CellLinkedList (one warp per
// particle, nlist.cuh) and runs the body thread-per-particle with the exact
// per-pair arithmetic of physics.cuh.  Bodies write only their own slots, as
// the reference's do, so no ordering between threads matters.
#include "common.cuh"
#include "internal.cuh"
#include "nlist.cuh"
#include "physics.cuh"

namespace sph {

template <class T> struct ArgsOf;
template <> struct ArgsOf<float> { using type = SphSweepArgs_f32; };
template <> struct ArgsOf<double> { using type = SphSweepArgs_f64; };

template <class T>
struct GenView {
    const T* x; const T* v; T* rho; T* p; const T* m;
    const uint32_t* wall; const uint32_t* ids;
    T* drho; T* dvdt; uint32_t* nnb; uint32_t* oflow; T* rho_new;
    int64_t n;
};

template <class T>
static PhysP phys_of(const typename ArgsOf<T>::type& a)
{
    PhysP P;
    P.cell_size = a.cell_size; P.cutoff = a.cutoff; P.h = a.h; P.alpha_d = a.alpha_d;
    P.c0 = a.c0; P.rho0 = a.rho0; P.alpha_visc = a.alpha_visc; P.eps_h2 = a.eps_h2;
    P.g[0] = a.g[0]; P.g[1] = a.g[1]; P.g[2] = a.dim == 3 ? a.g[2] : 0.0;
    return P;
}

template <class T, int D>
__device__ __forceinline__ void load3(const T* a, int64_t i, T (&o)[3])
{
    o[0] = a[i * D]; o[1] = a[i * D + 1]; o[2] = D == 3 ? a[i * D + 2] : T(0);
}

// physics.py:94-119
template <class T, int D>
__global__ void k_gen_continuity(GenView<T> a, PhysT<T> P, const int32_t* __restrict__ lists,
                                 const int32_t* __restrict__ lcount)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    if (a.wall[i] != 0) { a.drho[i] = T(0); return; }
    int cnt = lcount[i];
    if (cnt < 0) { a.oflow[i] = 1; return; }
    T xi[3], vi[3];
    load3<T, D>(a.x, i, xi);
    load3<T, D>(a.v, i, vi);
    T rho_i = a.rho[i];
    double acc = double(RN<T>::sub(rho_i, rho_i));
    for (int t = 0; t < cnt; t++) {
        int64_t j = lists[ell_index(i, t)];
        T xj[3], vj[3], dx[3], r2, vx;
        load3<T, D>(a.x, j, xj);
        load3<T, D>(a.v, j, vj);
        pair_geometry<T, D>(xi, xj, vi, vj, r2, vx, dx);
        acc = dadd(acc, continuity_term<T>(r2, vx, RN<T>::div(a.m[j], a.rho[j]), P));
    }
    a.drho[i] = RN<T>::from_d(dmul(double(rho_i), acc));
}

// physics.py:122-158
template <class T, int D>
__global__ void k_gen_momentum(GenView<T> a, PhysT<T> P, const int32_t* __restrict__ lists,
                               const int32_t* __restrict__ lcount)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    if (a.wall[i] != 0) {
        for (int k = 0; k < D; k++) a.dvdt[i * D + k] = T(0);
        return;
    }
    int cnt = lcount[i];
    if (cnt < 0) { a.oflow[i] = 1; return; }
    T xi[3], vi[3];
    load3<T, D>(a.x, i, xi);
    load3<T, D>(a.v, i, vi);
    const T rho_i = a.rho[i], p_i = a.p[i];
    const T pi_rr = RN<T>::div(p_i, RN<T>::mul(rho_i, rho_i));
    T acc[3] = {P.g[0], P.g[1], P.g[2]};
    for (int t = 0; t < cnt; t++) {
        int64_t j = lists[ell_index(i, t)];
        T xj[3], vj[3], dx[3], r2, vx;
        load3<T, D>(a.x, j, xj);
        load3<T, D>(a.v, j, vj);
        pair_geometry<T, D>(xi, xj, vi, vj, r2, vx, dx);
        momentum_pair<T, D>(r2, vx, dx, rho_i, pi_rr, a.rho[j],
                            RN<T>::div(a.p[j], RN<T>::mul(a.rho[j], a.rho[j])), a.m[j], P, acc);
    }
    for (int k = 0; k < D; k++) a.dvdt[i * D + k] = acc[k];
    a.nnb[i] = (uint32_t)cnt;
}

// physics.py:161-194 (walls read fluid neighbours' p only, write their own
// p/rho: no read-after-write hazard between threads)
template <class T, int D>
__global__ void k_gen_wall_pressure(GenView<T> a, PhysT<T> P, const int32_t* __restrict__ lists,
                                    const int32_t* __restrict__ lcount)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    if (a.wall[i] == 0) return;
    int cnt = lcount[i];
    if (cnt < 0) { a.oflow[i] = 1; return; }
    T xi[3];
    load3<T, D>(a.x, i, xi);
    T rho_i = a.rho[i];
    double num = double(RN<T>::sub(rho_i, rho_i));
    double den = num;
    uint32_t visits = 0;
    for (int t = 0; t < cnt; t++) {
        int64_t j = lists[ell_index(i, t)];
        if (a.wall[j] != 0) continue;
        visits++;
        T xj[3];
        load3<T, D>(a.x, j, xj);
        double w = wall_weight<T>(pair_r2<T, D>(xi, xj), P);
        num = dadd(num, dmul(double(a.p[j]), w));
        den = dadd(den, w);
    }
    T pw = den > 0.0 ? RN<T>::from_d(ddiv(num, den)) : T(0);
    a.p[i] = pw;
    a.rho[i] = RN<T>::add(P.rho0, RN<T>::div(pw, RN<T>::mul(P.c0, P.c0)));
    a.nnb[i] = visits;
}

// physics.py:197-217 (overflow: self term only)
template <class T, int D>
__global__ void k_gen_density_summation(GenView<T> a, PhysT<T> P,
                                        const int32_t* __restrict__ lists,
                                        const int32_t* __restrict__ lcount)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    int cnt = lcount[i];
    if (cnt < 0) cnt = 0;
    T xi[3];
    load3<T, D>(a.x, i, xi);
    double acc = double(RN<T>::mul(a.m[i], P.alpha_d));
    for (int t = 0; t < cnt; t++) {
        int64_t j = lists[ell_index(i, t)];
        T xj[3];
        load3<T, D>(a.x, j, xj);
        acc = dadd(acc, summation_term<T>(pair_r2<T, D>(xi, xj), a.m[j], P));
    }
    a.rho[i] = RN<T>::from_d(acc);
}

// physics.py:220-247
template <class T, int D>
__global__ void k_gen_shepard(GenView<T> a, PhysT<T> P, const int32_t* __restrict__ lists,
                              const int32_t* __restrict__ lcount)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    if (a.wall[i] != 0) { a.rho_new[i] = a.rho[i]; return; }
    int cnt = lcount[i];
    if (cnt < 0) { a.rho_new[i] = a.rho[i]; return; }
    T xi[3];
    load3<T, D>(a.x, i, xi);
    const T m_i = a.m[i];
    double num = double(RN<T>::mul(m_i, P.alpha_d));
    double den = double(RN<T>::mul(RN<T>::div(m_i, a.rho[i]), P.alpha_d));
    for (int t = 0; t < cnt; t++) {
        int64_t j = lists[ell_index(i, t)];
        T xj[3];
        load3<T, D>(a.x, j, xj);
        double w = wall_weight<T>(pair_r2<T, D>(xi, xj), P);
        num = dadd(num, dmul(double(a.m[j]), w));
        den = dadd(den, dmul(double(RN<T>::div(a.m[j], a.rho[j])), w));
    }
    a.rho_new[i] = RN<T>::from_d(ddiv(num, den));
}

// ---- integration bodies (physics.py:250-280) --------------------------------
template <class T>
__global__ void k_gen_kick(T* v, const T* dvdt, const uint32_t* wall, int64_t n, int dim, T half)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || wall[i] != 0) return;
    for (int k = 0; k < dim; k++)
        v[i * dim + k] = RN<T>::add(v[i * dim + k], RN<T>::mul(half, dvdt[i * dim + k]));
}

template <class T>
__global__ void k_gen_drift(T* x, const T* v, const uint32_t* wall, int64_t n, int dim, T dt)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || wall[i] != 0) return;
    for (int k = 0; k < dim; k++)
        x[i * dim + k] = RN<T>::add(x[i * dim + k], RN<T>::mul(dt, v[i * dim + k]));
}

template <class T>
__global__ void k_gen_density_update(T* rho, T* p, const T* drho, const uint32_t* wall, int64_t n,
                                     T dt, T c0, T rho0)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || wall[i] != 0) return;
    T r = RN<T>::add(rho[i], RN<T>::mul(dt, drho[i]));
    rho[i] = r;
    p[i] = RN<T>::mul(RN<T>::mul(c0, c0), RN<T>::sub(r, rho0));
}

// physics.py:296-310 VMAX_SPEC: exact max of sqrt(sum_k f64(v_k*v_k))
template <class T>
__global__ void k_gen_vmax(const T* v, int64_t n, int dim, unsigned long long* out)
{
    double best = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < dim; k++) {
            T c = v[i * dim + k];
            acc = dadd(acc, double(RN<T>::mul(c, c)));
        }
        double s = __dsqrt_rn(acc);
        best = s > best ? s : best;
    }
    unsigned long long b = warp_max_u64(dbits(best));
    if (lane_id() == 0) atomicMax(out, b);
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// ---- dispatch helpers --------------------------------------------------------
template <class T>
static GenView<T> view_of(const typename ArgsOf<T>::type& a)
{
    GenView<T> g;
    g.x = a.x; g.v = a.v; g.rho = a.rho; g.p = a.p; g.m = a.m; g.wall = a.wall; g.ids = a.ids;
    g.drho = a.drho; g.dvdt = a.dvdt; g.nnb = a.nnb; g.oflow = a.oflow; g.rho_new = a.rho_new;
    g.n = a.n;
    return g;
}

template <class T>
static GridP<T> grid_of(const typename ArgsOf<T>::type& a)
{
    GridP<T> g;
    for (int k = 0; k < 3; k++) {
        g.o[k] = k < a.dim ? a.origin[k] : T(0);
        g.s[k] = k < a.dim ? (int)a.shape[k] : 1;
    }
    g.cs = a.cell_size;
    g.c2 = a.cutoff * a.cutoff;   // binary32 product, neighborhood.py:185
    return g;
}

size_t lists_bytes(int64_t n)
{
    int64_t tiles = (n + 31) / 32;
    if (tiles < 1) tiles = 1;
    return align_up(sizeof(int32_t) * (size_t)tiles * kCap * 32) +
           align_up(sizeof(int32_t) * (size_t)tiles * 32);
}

template <class T>
static int gen_build(const typename ArgsOf<T>::type& a, int64_t i0, int64_t count,
                     int32_t* lists, int32_t* lcount, cudaStream_t s)
{
    GridP<T> g = grid_of<T>(a);
    if (a.dim == 2) {
        GenAcc<T, 2> acc{a.x, a.ids, a.offsets, a.pids};
        launch_build_lists<T, 2>(acc, g, i0, count, 0, lists, lcount, s);
    } else {
        GenAcc<T, 3> acc{a.x, a.ids, a.offsets, a.pids};
        launch_build_lists<T, 3>(acc, g, i0, count, 0, lists, lcount, s);
    }
    return check_launch("build_lists");
}

enum SweepKind { kContinuity, kMomentum, kWallPressure, kDensitySummation, kShepard };

template <class T, int D>
static void launch_sweep(SweepKind kind, GenView<T> v, PhysT<T> P, const int32_t* lists,
                         const int32_t* lcount, cudaStream_t s)
{
    int g = grid_for(v.n, 128);
    switch (kind) {
    case kContinuity: note_launch(), k_gen_continuity<T, D><<<g, 128, 0, s>>>(v, P, lists, lcount); break;
    case kMomentum: note_launch(), k_gen_momentum<T, D><<<g, 128, 0, s>>>(v, P, lists, lcount); break;
    case kWallPressure: note_launch(), k_gen_wall_pressure<T, D><<<g, 128, 0, s>>>(v, P, lists, lcount); break;
    case kDensitySummation:
        note_launch(), k_gen_density_summation<T, D><<<g, 128, 0, s>>>(v, P, lists, lcount);
        break;
    case kShepard: note_launch(), k_gen_shepard<T, D><<<g, 128, 0, s>>>(v, P, lists, lcount); break;
    }
}

template <class T>
static int gen_sweep(SweepKind kind, const typename ArgsOf<T>::type* a, void* ws, size_t ws_bytes,
                     cudaStream_t s)
{
    if (!a || (a->dim != 2 && a->dim != 3)) return SPH_ERR_INVALID;
    if (a->n <= 0) return SPH_OK;
    if (ws_bytes < lists_bytes(a->n)) return SPH_ERR_WORKSPACE;
    int64_t ncells = a->shape[0] * a->shape[1] * (a->dim == 3 ? a->shape[2] : 1);
    if (ncells >= (int64_t)UINT32_MAX || a->n >= (int64_t)INT32_MAX) return SPH_ERR_UNSUPPORTED;
    int64_t tiles = (a->n + 31) / 32;
    int32_t* lists = static_cast<int32_t*>(ws);
    int32_t* lcount = reinterpret_cast<int32_t*>(
        static_cast<char*>(ws) + align_up(sizeof(int32_t) * (size_t)tiles * kCap * 32));
    int rc = gen_build<T>(*a, 0, a->n, lists, lcount, s);
    if (rc) return rc;
    GenView<T> v = view_of<T>(*a);
    const PhysT<T> P = make_phys<T>(phys_of<T>(*a));
    if (a->dim == 2) launch_sweep<T, 2>(kind, v, P, lists, lcount, s);
    else launch_sweep<T, 3>(kind, v, P, lists, lcount, s);
    return check_launch("sweep");
}

}  // namespace sph

using namespace sph;

extern "C" size_t sph_sweep_workspace_bytes(int64_t n) { return lists_bytes(n); }

#define SPH_SWEEP_ENTRY(NAME, KIND)                                                          \
    extern "C" int sph_##NAME##_f32(const SphSweepArgs_f32* a, void* ws, size_t b,            \
                                    cudaStream_t s)                                           \
    {                                                                                         \
        return gen_sweep<float>(KIND, a, ws, b, s);                                           \
    }                                                                                         \
    extern "C" int sph_##NAME##_f64(const SphSweepArgs_f64* a, void* ws, size_t b,            \
                                    cudaStream_t s)                                           \
    {                                                                                         \
        return gen_sweep<double>(KIND, a, ws, b, s);                                          \
    }
SPH_SWEEP_ENTRY(continuity, kContinuity)
SPH_SWEEP_ENTRY(momentum, kMomentum)
SPH_SWEEP_ENTRY(wall_pressure, kWallPressure)
SPH_SWEEP_ENTRY(density_summation, kDensitySummation)
SPH_SWEEP_ENTRY(shepard, kShepard)

extern "C" int sph_neighbors_f32(const SphSweepArgs_f32* a, int64_t i0, int64_t count,
                                 int32_t* out_lists, int32_t* out_counts, cudaStream_t s)
{
    if (!a || (a->dim != 2 && a->dim != 3)) return SPH_ERR_INVALID;
    return gen_build<float>(*a, i0, count, out_lists, out_counts, s);
}

extern "C" int sph_neighbors_f64(const SphSweepArgs_f64* a, int64_t i0, int64_t count,
                                 int32_t* out_lists, int32_t* out_counts, cudaStream_t s)
{
    if (!a || (a->dim != 2 && a->dim != 3)) return SPH_ERR_INVALID;
    return gen_build<double>(*a, i0, count, out_lists, out_counts, s);
}

#define SPH_INTEG_ENTRY(SFX, T)                                                                \
    extern "C" int sph_kick_##SFX(T* v, const T* dvdt, const uint32_t* wall, int64_t n,        \
                                  int dim, T half_dt, cudaStream_t s)                          \
    {                                                                                          \
        if (n <= 0) return SPH_OK;                                                             \
        note_launch(), k_gen_kick<T><<<grid_for(n, 256), 256, 0, s>>>(v, dvdt, wall, n, dim, half_dt);        \
        return check_launch("kick");                                                           \
    }                                                                                          \
    extern "C" int sph_drift_##SFX(T* x, const T* v, const uint32_t* wall, int64_t n, int dim, \
                                   T dt, cudaStream_t s)                                       \
    {                                                                                          \
        if (n <= 0) return SPH_OK;                                                             \
        note_launch(), k_gen_drift<T><<<grid_for(n, 256), 256, 0, s>>>(x, v, wall, n, dim, dt);               \
        return check_launch("drift");                                                          \
    }                                                                                          \
    extern "C" int sph_density_update_##SFX(T* rho, T* p, const T* drho, const uint32_t* wall, \
                                            int64_t n, T dt, T c0, T rho0, cudaStream_t s)     \
    {                                                                                          \
        if (n <= 0) return SPH_OK;                                                             \
        note_launch(), k_gen_density_update<T><<<grid_for(n, 256), 256, 0, s>>>(rho, p, drho, wall, n, dt,    \
                                                                 c0, rho0);                    \
        return check_launch("density_update");                                                 \
    }                                                                                          \
    extern "C" int sph_vmax_##SFX(const T* v, int64_t n, int dim, double* out, cudaStream_t s) \
    {                                                                                          \
        note_launch(), k_set_u64<<<1, 1, 0, s>>>((unsigned long long*)out, 0ull);                             \
        if (n > 0)                                                                             \
            note_launch(), k_gen_vmax<T><<<grid_for(n, 256, 4 * 148), 256, 0, s>>>(                           \
                v, n, dim, (unsigned long long*)out);                                          \
        return check_launch("vmax");                                                           \
    }
SPH_INTEG_ENTRY(f32, float)
SPH_INTEG_ENTRY(f64, double)

// ---------------------------------------------------------------------------
// self-test of the reciprocal divisions (common.cuh) against the IEEE ones
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t& s)
{
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void k_selftest_div(float hf, double hd, int64_t n, uint64_t seed,
                               unsigned long long* bad)
{
    const float yf = __frcp_rn(hf);
    const double yd = __drcp_rn(hd);
    const bool okf = rcp_ok<float>(hf), okd = rcp_ok<double>(hd);
    unsigned long long nb = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t st = seed ^ (uint64_t)k * 0x2545f4914f6cdd1dull;
        const uint64_t u = splitmix64(st);
        // random significands; binary32 exponents over 2^-64 .. 2^63 and
        // binary64 ones over 2^-470 .. 2^470, both across the edges of the
        // reciprocal path's range tests (2^+-59 / 2^+-465)
        const double sig = 1.0 + (double)(u >> 11) * 0x1.0p-53;
        const double magf = ldexp(sig, (int)(u & 127) - 64);
        const double magd = ldexp(sig, (int)((u >> 16) % 941) - 470);
        const bool neg = (u >> 7) & 1;
        const float af = (float)(neg ? -magf : magf);
        const double a = neg ? -magd : magd;
        if (__float_as_uint(fdiv_rcp(af, hf, yf, okf)) != __float_as_uint(__fdiv_rn(af, hf))) nb++;
        if (__double_as_longlong(ddiv_rcp(a, hd, yd, okd)) !=
            __double_as_longlong(__ddiv_rn(a, hd)))
            nb++;
    }
    nb = warp_sum(nb);
    if (lane_id() == 0 && nb) atomicAdd(bad, nb);
}

extern "C" int sph_selftest_div(double h, int64_t n, uint64_t seed, unsigned long long* bad,
                                cudaStream_t s)
{
    note_launch(), k_selftest_div<<<148 * 8, 256, 0, s>>>((float)h, h, n, seed, bad);
    return check_launch("selftest_div");
}

// pair_fac_spec (physics.cuh, the straight-line f32 pair factor) against the
// per-operation reference sequence for EVERY binary32 bit pattern in
// [lo_bits, hi_bits) (positive r2; the sweeps see 0 < r2 < c^2).
__global__ void k_selftest_pair_fac(PhysT<float> P, uint32_t lo, uint32_t hi,
                                    unsigned long long* bad, unsigned int* first)
{
    unsigned long long nb = 0;
    for (uint64_t u = (uint64_t)lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
         u < (uint64_t)hi; u += (uint64_t)gridDim.x * blockDim.x) {
        const float r2 = __uint_as_float((uint32_t)u);
        const double a = pair_fac_spec(r2, P), b = pair_fac_ref<float>(r2, P);
        if (__double_as_longlong(a) != __double_as_longlong(b)) {
            nb++;
            atomicMin(first, (unsigned int)u);
        }
    }
    nb = warp_sum(nb);
    if (lane_id() == 0 && nb) atomicAdd(bad, nb);
}

extern "C" int sph_selftest_pair_fac(double h, double alpha_d, uint32_t lo_bits,
                                     uint32_t hi_bits, unsigned long long* bad,
                                     unsigned int* first_bad, cudaStream_t s)
{
    PhysP p{};
    p.h = (double)(float)h;
    p.alpha_d = (double)(float)alpha_d;
    note_launch(), k_selftest_pair_fac<<<148 * 16, 256, 0, s>>>(make_phys<float>(p), lo_bits,
                                                                hi_bits, bad, first_bad);
    return check_launch("selftest_pair_fac");
}

// rn_f32_in_f64 (physics.cuh, the momentum sweep's binary32 rounding in the
// FP64 adder) against __double2float_rn: random significands over the
// binade band [2^-160, 2^140), half of them made exact binary32 ties (the
// 29 low significand bits set to 1 << 28), both signs, zeros.  *bad +=
// mismatches of the fast path where it claims validity; *fast += values it
// handled (the rest take the conversion fallback).
__global__ void k_selftest_round_f32(int64_t n, uint64_t seed, unsigned long long* bad,
                                     unsigned long long* fast)
{
    unsigned long long nb = 0, nf = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t st = seed ^ (uint64_t)k * 0x9e3779b97f4a7c15ull;
        const uint64_t u = splitmix64(st), v = splitmix64(st);
        uint64_t mant = u & 0xfffffffffffffull;
        if (v & 1) mant = (mant & ~0x1fffffffull) | 0x10000000ull;   // a binary32 tie
        const int e = (int)((v >> 1) % 300) - 160;
        uint64_t bits = ((uint64_t)(e + 1023) << 52) | mant | ((v >> 20) & 1 ? (1ull << 63) : 0);
        if ((v >> 21) % 1000 == 0) bits &= (1ull << 63);              // +-0
        const double s = __longlong_as_double((long long)bits);
        bool ok = true;
        const double r = rn_f32_in_f64(s, ok);
        if (ok) {
            nf++;
            if (__double_as_longlong(r) != __double_as_longlong(double(__double2float_rn(s))))
                nb++;
        }
    }
    nb = warp_sum(nb);
    nf = warp_sum(nf);
    if (lane_id() == 0) {
        if (nb) atomicAdd(bad, nb);
        atomicAdd(fast, nf);
    }
}

extern "C" int sph_selftest_round_f32(int64_t n, uint64_t seed, unsigned long long* bad,
                                      unsigned long long* fast, cudaStream_t s)
{
    note_launch(), k_selftest_round_f32<<<148 * 16, 256, 0, s>>>(n, seed, bad, fast);
    return check_launch("selftest_round_f32");
}

