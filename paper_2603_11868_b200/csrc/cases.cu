// cases.cu -- case placement on the device.
//
// Replaces the host lattice builders of the reference case setup
// (cases.py:129-161 _lattice / _tank_wall_points / _box_points and the fluid
// cut of build_case_dambreak, cases.py:217-238): a 64M-particle tank
// materialises ~275M host lattice points (meshgrid, index arrays, masks);
// here every point is generated from its lattice index in registers, tested,
// and compacted in lattice order straight into HBM.
//
// Arithmetic (binary64, round to nearest, no FMA -- the build uses
// --fmad=false and explicit intrinsics): a point is anchor + (i + 0.5)*dp,
// numpy's `anchor + (idx + 0.5) * dp` with idx converted to float64 exactly;
// the tank test recomputes idx = round(pt/dp - 0.5) (np.round: half to
// even == rint) exactly as _tank_wall_points does.
//
// Two passes over tiles of kLatTile lattice points: per-tile kept counts,
// an exclusive scan (sort.cu), then per tile a block-ordered compaction
// (warp ballots + a block prefix), so the output order is the lattice's C
// order (last axis fastest), the order of np.meshgrid(indexing="ij").ravel().
#include "common.cuh"
#include "internal.cuh"

namespace sph {

constexpr int kLatThreads = 256;
constexpr int kLatRounds = 8;
constexpr int kLatTile = kLatThreads * kLatRounds;

struct LatP {
    int d, mode;
    int64_t lo[3], ext[3];       // index box [lo, lo + ext)
    double dp, anchor[3];
    int64_t counts[3];           // SPH_LATTICE_TANK: inner tank counts
    double box_lo[3], box_hi[3]; // SPH_LATTICE_NOT_IN: open box
    int64_t npts;
};

__device__ __forceinline__ bool lat_point(const LatP& P, int64_t p, double (&pt)[3],
                                          int64_t& ilast)
{
    int64_t idx[3] = {0, 0, 0};
    int64_t r = p;
    for (int k = P.d - 1; k >= 0; k--) {
        idx[k] = P.lo[k] + r % P.ext[k];
        r /= P.ext[k];
    }
    for (int k = 0; k < P.d; k++)
        pt[k] = dadd(P.anchor[k], dmul(dadd((double)idx[k], 0.5), P.dp));
    ilast = idx[P.d - 1];
    if (P.mode == SPH_LATTICE_TANK) {
        // cases.py:146-150: outside = any(idx < 0) | any(idx[:, k] >= counts[k], k < d-1)
        bool outside = false;
        for (int k = 0; k < P.d; k++) {
            const double t = rint(dsub(ddiv(pt[k], P.dp), 0.5));
            const int64_t ik = (int64_t)t;
            outside |= ik < 0;
            if (k < P.d - 1) outside |= ik >= P.counts[k];
        }
        return outside;
    }
    if (P.mode == SPH_LATTICE_NOT_IN) {
        // cases.py:230-232: inside = ((fluid > lo) & (fluid < hi)).all(axis=1)
        bool inside = true;
        for (int k = 0; k < P.d; k++) inside &= (pt[k] > P.box_lo[k]) && (pt[k] < P.box_hi[k]);
        return !inside;
    }
    return true;
}

__global__ void __launch_bounds__(kLatThreads) k_lat_count(LatP P, uint32_t* __restrict__ cnt)
{
    const int64_t base = (int64_t)blockIdx.x * kLatTile;
    int c = 0;
    for (int r = 0; r < kLatRounds; r++) {
        const int64_t p = base + r * kLatThreads + threadIdx.x;
        double pt[3];
        int64_t il;
        if (p < P.npts && lat_point(P, p, pt, il)) c++;
    }
    c = warp_sum(c);
    __shared__ int ws[kLatThreads / 32];
    if (lane_id() == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kLatThreads / 32; w++) t += ws[w];
        cnt[blockIdx.x] = (uint32_t)t;
    }
}

__global__ void __launch_bounds__(kLatThreads)
k_lat_write(LatP P, const uint32_t* __restrict__ off, double* __restrict__ out,
            unsigned long long* __restrict__ ilast_max)
{
    const int64_t base = (int64_t)blockIdx.x * kLatTile;
    __shared__ int wsum[kLatThreads / 32];
    __shared__ int total;
    int64_t run = off[blockIdx.x];
    long long imax = LLONG_MIN;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    for (int r = 0; r < kLatRounds; r++) {
        const int64_t p = base + r * kLatThreads + threadIdx.x;
        double pt[3];
        int64_t il = 0;
        const bool keep = p < P.npts && lat_point(P, p, pt, il);
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[warp] = __popc(b);
        __syncthreads();
        int before = 0;
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < kLatThreads / 32; w++) t += wsum[w];
            total = t;
        }
        for (int w = 0; w < (int)warp; w++) before += wsum[w];
        if (keep) {
            const int64_t q = run + before + __popc(b & lanemask_lt());
            if (out)
                for (int k = 0; k < P.d; k++) out[q * P.d + k] = pt[k];
            imax = il > imax ? il : imax;
        }
        __syncthreads();
        run += total;
        __syncthreads();
    }
    // order-preserving u64 key of the largest kept last-axis index
    for (int o = 16; o > 0; o >>= 1) {
        const long long v = __shfl_xor_sync(0xffffffffu, imax, o);
        imax = v > imax ? v : imax;
    }
    if (lane == 0 && imax != LLONG_MIN)
        atomicMax(ilast_max, (unsigned long long)imax ^ 0x8000000000000000ull);
}

__global__ void k_lat_total(const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                            int64_t tiles, int64_t* __restrict__ count)
{
    count[0] = tiles ? (int64_t)off[tiles - 1] + cnt[tiles - 1] : 0;
}

static bool lat_params(int32_t d, const int64_t* lo, const int64_t* hi, LatP& P)
{
    if (d < 1 || d > 3 || !lo || !hi) return false;
    P.d = d;
    P.npts = 1;
    for (int k = 0; k < 3; k++) {
        P.lo[k] = k < d ? lo[k] : 0;
        P.ext[k] = k < d ? hi[k] - lo[k] : 1;
        if (P.ext[k] <= 0) { P.npts = 0; P.ext[k] = 1; }
    }
    if (P.npts)
        for (int k = 0; k < d; k++) P.npts *= P.ext[k];
    return true;
}

}  // namespace sph

using namespace sph;

extern "C" size_t sph_lattice_workspace_bytes(int32_t d, const int64_t* lo, const int64_t* hi)
{
    LatP P;
    if (!lat_params(d, lo, hi, P)) return 0;
    const int64_t tiles = (P.npts + kLatTile - 1) / kLatTile;
    const size_t t = (size_t)(tiles > 0 ? tiles : 1);
    return 2 * align_up(sizeof(uint32_t) * t) + scan_scratch_bytes(tiles);
}

extern "C" int sph_lattice_points(int32_t d, const int64_t* lo, const int64_t* hi, double dp,
                                  const double* anchor, int32_t mode, const int64_t* counts,
                                  const double* box_lo, const double* box_hi, double* out,
                                  int64_t* count, unsigned long long* ilast_max, void* ws,
                                  size_t ws_bytes, cudaStream_t s)
{
    LatP P;
    if (!lat_params(d, lo, hi, P) || !count || !ilast_max || !anchor ||
        (mode != SPH_LATTICE_ALL && mode != SPH_LATTICE_TANK && mode != SPH_LATTICE_NOT_IN) ||
        (mode == SPH_LATTICE_TANK && !counts) ||
        (mode == SPH_LATTICE_NOT_IN && (!box_lo || !box_hi))) {
        set_error("lattice_points: bad arguments");
        return SPH_ERR_INVALID;
    }
    if (P.npts >= ((int64_t)1 << 32)) {
        set_error("lattice_points: more than 2^32 lattice points");
        return SPH_ERR_UNSUPPORTED;
    }
    P.mode = mode;
    P.dp = dp;
    for (int k = 0; k < 3; k++) {
        P.anchor[k] = k < d ? anchor[k] : 0.0;
        P.counts[k] = (k < d && counts) ? counts[k] : 0;
        P.box_lo[k] = (k < d && box_lo) ? box_lo[k] : 0.0;
        P.box_hi[k] = (k < d && box_hi) ? box_hi[k] : 0.0;
    }
    if (ws_bytes < sph_lattice_workspace_bytes(d, lo, hi)) return SPH_ERR_WORKSPACE;
    const int64_t tiles = (P.npts + kLatTile - 1) / kLatTile;
    if (tiles == 0) {
        cudaMemsetAsync(count, 0, sizeof(int64_t), s);
        return check_launch("lattice_points");
    }
    Bump bump(ws, ws_bytes);
    uint32_t* cnt = bump.take<uint32_t>(tiles);
    uint32_t* off = bump.take<uint32_t>(tiles);
    void* scan_tmp = bump.take<char>(scan_scratch_bytes(tiles));
    note_launch(), k_lat_count<<<(unsigned)tiles, kLatThreads, 0, s>>>(P, cnt);
    int rc = exclusive_scan_u32(cnt, off, tiles, scan_tmp, s);
    if (rc) return rc;
    note_launch(), k_lat_write<<<(unsigned)tiles, kLatThreads, 0, s>>>(P, off, out, ilast_max);
    note_launch(), k_lat_total<<<1, 1, 0, s>>>(off, cnt, tiles, count);
    return check_launch("lattice_points");
}
