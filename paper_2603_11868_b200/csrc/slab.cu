// slab.cu -- the per-step bookkeeping of a slab rank (distributed.py,
// SURVEY.md 8e) as device kernels instead of host-synchronised tensor
// algebra: one pass classifies the rank's owned rows by the axis-0 cell
// plane of their position into per-peer mover lists, per-peer halo lists
// (fluid and wall records apart) and the kept list; registry-layout rows
// then move as fixed-width int32 records (pack -> transport -> unpack), and
// kept rows are gathered straight into the next push's input.
//
// Row order inside a list follows warp-aggregated atomics (not fixed): the
// engine accumulates every neighbour sum in ascending ORIGINAL id, so the
// physical order of a rank's particles never changes a result bit.
#include "engine.cuh"

namespace sph {

// registry field order (distributed.FIELDS): widths in elements
//   x[d] v[d] rho p m Vol drho dvdt[d] rho_scratch  (run precision)
//   id wall nnb oflow                                 (uint32)
__host__ __device__ inline int rows_field_elems(int f, int d)
{
    return (f == 0 || f == 1 || f == 7) ? d : 1;
}
__host__ __device__ inline bool rows_field_real(int f) { return f < 9; }
constexpr int kRowFields = 13;

__host__ __device__ inline int rows_words(int d, int f64)
{
    return (3 * d + 6) * (f64 ? 2 : 1) + 4;
}

__device__ __forceinline__ bool slab_halo(const SphSlabGeom& g, int q, int64_t p)
{
    const int64_t a = g.cuts[q], b = g.cuts[q + 1], H = g.halo, P = g.nplanes;
    if (g.periodic) {
        const bool inside = p >= a && p < b;
        const int64_t below = ((a - p) % P + P) % P;
        const int64_t above = ((p - b) % P + P) % P;
        return !inside && ((below >= 1 && below <= H) || above < H);
    }
    return (p >= a - H && p < a) || (p >= b && p < b + H);
}

__device__ __forceinline__ void slab_append(int32_t* list, int32_t* count, bool take, int32_t row)
{
    const unsigned b = __ballot_sync(0xffffffffu, take);
    if (!b) return;
    const int leader = __ffs(b) - 1;
    int base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(count, __popc(b));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (take) list[base + __popc(b & lanemask_lt())] = row;
}

// list c of cls 3k (movers to peer k), 3k+1 (fluid halo of k), 3k+2 (wall
// halo of k), 3 npeers (kept); counts[3 npeers + 1] flags a row whose new
// owner is no peer (a particle crossed more than one slab in a step)
template <class T>
__global__ void __launch_bounds__(256)
k_slab_classify(SphSlabGeom g, const T* __restrict__ x, const uint32_t* __restrict__ wall,
                int64_t n, int d, int32_t* __restrict__ lists, int32_t* __restrict__ counts)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = r < n;
    int64_t p = 0;
    int owner = g.rank;
    bool w = false;
    int cl = 0;
    if (live) {
        const T cs = T(g.cell_size);
        p = cell_coord<T>(x[r * d], T(g.origin[0]), cs, (int)g.shape[0], cl);
        for (int k = 1; k < d; k++) cell_coord<T>(x[r * d + k], T(g.origin[k]), cs, (int)g.shape[k], cl);
        int lo = 0, hi = g.nranks;   // owner = last q with cuts[q] <= p
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (g.cuts[mid] <= p) lo = mid;
            else hi = mid;
        }
        owner = lo;
        w = wall[r] != 0;
    }
    const bool keep = live && owner == g.rank;
    bool lost = live && !keep;
    for (int k = 0; k < g.npeers; k++) {
        const int q = g.peer[k];
        const bool mv = live && !keep && owner == q;
        lost = lost && !mv;
        slab_append(lists + (size_t)(3 * k) * n, counts + 3 * k, mv, (int32_t)r);
        const bool h = keep && slab_halo(g, q, p);
        slab_append(lists + (size_t)(3 * k + 1) * n, counts + 3 * k + 1, h && !w, (int32_t)r);
        slab_append(lists + (size_t)(3 * k + 2) * n, counts + 3 * k + 2, h && w, (int32_t)r);
    }
    slab_append(lists + (size_t)(3 * g.npeers) * n, counts + 3 * g.npeers, keep, (int32_t)r);
    if (__any_sync(0xffffffffu, lost) && lane_id() == 0) atomicAdd(counts + 3 * g.npeers + 1, 1);
    const unsigned oob = __ballot_sync(0xffffffffu, live && cl);
    if (oob && lane_id() == 0) atomicAdd(counts + 3 * g.npeers + 2, __popc(oob));
}

// record k <- row rows[k] of in (all fields, as 32-bit words)
__global__ void __launch_bounds__(256)
k_slab_pack(SphRows in, int d, int f64, const int32_t* __restrict__ rows, int64_t n,
            uint32_t* __restrict__ out)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t r = rows ? rows[k] : k;
    const int W = rows_words(d, f64);
    uint32_t* o = out + (size_t)k * W;
    int c = 0;
    for (int f = 0; f < kRowFields; f++) {
        const int wpe = rows_field_real(f) ? (f64 ? 2 : 1) : 1;
        const int nw = rows_field_elems(f, d) * wpe;
        const uint32_t* src = (const uint32_t*)in.f[f] + (size_t)r * nw;
        for (int t = 0; t < nw; t++) o[c + t] = src[t];
        c += nw;
    }
}

// rows [off, off + n) of out <- records (rows == nullptr) or <- rows of in
__global__ void __launch_bounds__(256)
k_slab_put(const uint32_t* __restrict__ rec, SphRows in, const int32_t* __restrict__ rows,
           int64_t n, SphRows out, int d, int f64, int64_t off)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int W = rows_words(d, f64);
    int c = 0;
    for (int f = 0; f < kRowFields; f++) {
        const int wpe = rows_field_real(f) ? (f64 ? 2 : 1) : 1;
        const int nw = rows_field_elems(f, d) * wpe;
        uint32_t* dst = (uint32_t*)out.f[f] + (size_t)(off + k) * nw;
        const uint32_t* src = rec ? rec + (size_t)k * W + c
                                  : (const uint32_t*)in.f[f] + (size_t)rows[k] * nw;
        for (int t = 0; t < nw; t++) dst[t] = src[t];
        c += nw;
    }
}

}  // namespace sph

using namespace sph;

extern "C" int32_t sph_slab_record_words(int32_t dim, int32_t f64)
{
    return rows_words(dim, f64);
}

extern "C" int sph_slab_classify(const SphSlabGeom* g, const void* x, const uint32_t* wall,
                                 int64_t n, int32_t dim, int32_t f64, int32_t* lists,
                                 int32_t* counts, cudaStream_t s)
{
    if (!g || g->nranks < 1 || g->nranks > SPH_MAX_RANKS || g->npeers < 0 ||
        g->npeers > SPH_MAX_PEERS || (dim != 2 && dim != 3) || n < 0)
        return SPH_ERR_INVALID;
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)(3 * g->npeers + 3), s);
    if (n > 0) {
        if (f64)
            note_launch(), k_slab_classify<double><<<grid_for(n, 256), 256, 0, s>>>(
                *g, (const double*)x, wall, n, dim, lists, counts);
        else
            note_launch(), k_slab_classify<float><<<grid_for(n, 256), 256, 0, s>>>(
                *g, (const float*)x, wall, n, dim, lists, counts);
    }
    return check_launch("slab_classify");
}

extern "C" int sph_slab_pack(const SphRows* in, int32_t dim, int32_t f64, const int32_t* rows,
                             int64_t n, void* out, cudaStream_t s)
{
    if (!in || n < 0) return SPH_ERR_INVALID;
    if (n > 0)
        note_launch(), k_slab_pack<<<grid_for(n, 256), 256, 0, s>>>(*in, dim, f64, rows, n,
                                                                    (uint32_t*)out);
    return check_launch("slab_pack");
}

extern "C" int sph_slab_unpack(const void* records, int64_t n, const SphRows* out, int32_t dim,
                               int32_t f64, int64_t dst_off, cudaStream_t s)
{
    if (!out || n < 0 || !records) return SPH_ERR_INVALID;
    if (n > 0)
        note_launch(), k_slab_put<<<grid_for(n, 256), 256, 0, s>>>(
            (const uint32_t*)records, *out, nullptr, n, *out, dim, f64, dst_off);
    return check_launch("slab_unpack");
}

extern "C" int sph_slab_gather(const SphRows* in, const int32_t* rows, int64_t n,
                               const SphRows* out, int32_t dim, int32_t f64, int64_t dst_off,
                               cudaStream_t s)
{
    if (!in || !out || !rows || n < 0) return SPH_ERR_INVALID;
    if (n > 0)
        note_launch(), k_slab_put<<<grid_for(n, 256), 256, 0, s>>>(nullptr, *in, rows, n, *out,
                                                                   dim, f64, dst_off);
    return check_launch("slab_gather");
}
