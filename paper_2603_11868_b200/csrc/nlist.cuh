// nlist.cuh -- ordered neighbour lists (neighborhood.py:176-227).
//
// The reference collects, for each particle i, every j != i of the clamped
// 3^d cell block around i's CURRENT cell (membership from the cell linked
// list built at the start of the advective step, neighborhood.py:188-213)
// with 0 < r2 < cutoff^2, and visits them in ascending ORIGINAL id.  That
// order fixes every floating-point accumulation, so it is reproduced exactly.
//
// B200 mapping: one warp per particle.  Row-major cell keys make each (ax,
// ay) column of the block one contiguous key range (3 in 2D, 9 in 3D), i.e.
// one contiguous run of the cell-sorted particle array per segment.  All
// run bounds are fetched in one round trip (one lane per run), a warp scan
// flattens the runs into one candidate index space, and every 32-candidate
// step finds its run with a 5-step shuffle binary search -- so a particle
// costs two dependent memory round trips plus one per 32 candidates, not two
// per run.  Survivors are compacted by ballot into a per-warp shared buffer
// of packed (id << 32 | j) and sorted by a warp bitonic network (registers
// for <= 32 survivors, shared memory above).
//
// Two acceptance modes:
//   exact: 0 < r2 < cutoff^2 (the reference's test), and
//   skin:  r2 < (cutoff + skin)^2 -- a Verlet superset built once per
//          advective step; engine.cu filters it exactly every sub-step.
#pragma once

#include "common.cuh"
#include "physics.cuh"

namespace sph {

constexpr int kNlWarps = 8;
constexpr int kNlThreads = kNlWarps * 32;
constexpr int kStagePitch = 33;   // conflict-free transposition
struct WarpBuf;
constexpr size_t kWarpBufBytes = sizeof(uint32_t) * (2 * kCap + 4);
constexpr size_t kNlSmem = sizeof(int32_t) * kCap * kStagePitch + kWarpBufBytes * kNlWarps +
                           sizeof(int) * 64;

template <class T>
struct GridP {
    T o[3]; T cs; T c2; int s[3];
};

#if SPH_PERIODIC
// The 3^d block of cell cc with periodic axes wrapped: a
// periodic column axis (all but the last) contributes cc-1, cc, cc+1 mod s;
// along the last axis each column is one key run [zlo, zhi] plus, at a
// periodic edge, a one-cell run zw on the far side.  Periodic axes have
// s >= 3 (no cell repeats); bounded axes clamp like neighborhood.py:188-196.
struct PerBlock {
    int ax0, ax1, ax2, ay0, ay1, ay2;
    int nx, ny, nz, zlo, zhi, zw;
};
__device__ __forceinline__ int pick3(int a, int b, int c, int i)
{
    return i == 0 ? a : (i == 1 ? b : c);
}
template <class T>
__device__ __forceinline__ void per_axis(int c, int s, bool periodic, int& n, int& a0, int& a1,
                                         int& a2)
{
    if (periodic) {
        n = 3;
        a0 = c == 0 ? s - 1 : c - 1;
        a1 = c;
        a2 = c + 1 == s ? 0 : c + 1;
    } else {
        const int lo = max(c - 1, 0), hi = min(c + 1, s - 1);
        n = hi - lo + 1;
        a0 = lo; a1 = lo + 1; a2 = lo + 2;
    }
}
template <class T, int D>
__device__ __forceinline__ PerBlock per_block(const GridP<T>& g, const int (&cc)[3])
{
    PerBlock b;
    per_axis<T>(cc[0], g.s[0], BoxOf<T>::L(0) > T(0), b.nx, b.ax0, b.ax1, b.ax2);
    if (D == 3) per_axis<T>(cc[1], g.s[1], BoxOf<T>::L(1) > T(0), b.ny, b.ay0, b.ay1, b.ay2);
    else { b.ny = 1; b.ay0 = b.ay1 = b.ay2 = 0; }
    constexpr int r = D - 1;
    const int s = g.s[r];
    int lo = cc[r] - 1, hi = cc[r] + 1;
    b.nz = 1;
    b.zw = 0;
    if (BoxOf<T>::L(r) > T(0)) {
        if (lo < 0) { b.nz = 2; b.zw = s - 1; lo = 0; }
        else if (hi > s - 1) { b.nz = 2; b.zw = 0; hi = s - 1; }
    } else {
        lo = max(lo, 0);
        hi = min(hi, s - 1);
    }
    b.zlo = lo;
    b.zhi = hi;
    return b;
}
__device__ __forceinline__ int per_runs(const PerBlock& b) { return b.nx * b.ny * b.nz; }
// run rr in [0, per_runs(b)) -> inclusive key range [klo, khi]
template <class T, int D>
__device__ __forceinline__ void per_run(const GridP<T>& g, const PerBlock& b, int rr,
                                        uint32_t& klo, uint32_t& khi)
{
    const int col = rr / b.nz, z = rr - col * b.nz;
    const int cx = col / b.ny, cy = col - cx * b.ny;
    const int ax = pick3(b.ax0, b.ax1, b.ax2, cx), ay = pick3(b.ay0, b.ay1, b.ay2, cy);
    const int zl = z ? b.zw : b.zlo, zh = z ? b.zw : b.zhi;
    if (D == 3) {
        const uint32_t rowk = ((uint32_t)ax * g.s[1] + ay) * g.s[2];
        klo = rowk + zl;
        khi = rowk + zh;
    } else {
        klo = (uint32_t)ax * g.s[1] + zl;
        khi = (uint32_t)ax * g.s[1] + zh;
    }
}
#endif

// Quad tile-ELL: a 32-particle tile stores entry t of particle (lane) s at
// [s/32][t/4][s%32][t%4], so one int4 load per lane fetches 4 consecutive
// entries and a warp's int4 loads cover one contiguous 512-byte block.
__device__ __forceinline__ size_t ell_base(int64_t slot)
{
    return (size_t)(slot >> 5) * (kCap * 32) + (size_t)(slot & 31) * 4;
}
__device__ __forceinline__ int ell_off(int t) { return (t >> 2) * 128 + (t & 3); }
__device__ __forceinline__ size_t ell_index(int64_t slot, int t)
{
    return ell_base(slot) + (size_t)ell_off(t);
}

// ascending bitonic sort of sb[0..np), np a power of two in [64, 256]
__device__ __forceinline__ void warp_bitonic_smem(unsigned long long* sb, int np, unsigned lane)
{
    for (int k = 2; k <= np; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int q = lane; q < (np >> 1); q += 32) {
                int lo = ((q & ~(j - 1)) << 1) | (q & (j - 1));
                int hi = lo + j;
                unsigned long long a = sb[lo], b = sb[hi];
                bool up = (lo & k) == 0;
                if ((a > b) == up) { sb[lo] = b; sb[hi] = a; }
            }
            __syncwarp();
        }
    }
}

// ascending bitonic sort of one value per lane
__device__ __forceinline__ unsigned long long warp_bitonic_reg(unsigned long long v,
                                                               unsigned lane)
{
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            unsigned long long o = __shfl_xor_sync(0xffffffffu, v, j);
            bool up = (lane & k) == 0;
            bool lower = (lane & j) == 0;
            unsigned long long mn = o < v ? o : v, mx = o < v ? v : o;
            v = (lower == up) ? mn : mx;
        }
    }
    return v;
}

// Register bitonic sort of 32*PER values held blocked (lane owns elements
// lane*PER .. lane*PER+PER-1): partners closer than PER are exchanged inside
// a lane, farther ones through shuffles.  Fully unrolled; ~5x cheaper than a
// shared-memory network for 128 elements.
template <int PER>
__device__ __forceinline__ void warp_bitonic_blocked(unsigned long long (&v)[PER], unsigned lane)
{
    constexpr int N = 32 * PER;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= PER) {
#pragma unroll
                for (int r = 0; r < PER; r++) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[r], j / PER);
                    const int e = (int)lane * PER + r;
                    const bool up = (e & k) == 0, lower = (e & j) == 0;
                    const unsigned long long mn = o < v[r] ? o : v[r];
                    const unsigned long long mx = o < v[r] ? v[r] : o;
                    v[r] = (lower == up) ? mn : mx;
                }
            } else {
#pragma unroll
                for (int r = 0; r < PER; r++) {
                    if (r & j) continue;
                    const int e = (int)lane * PER + r;
                    const bool up = (e & k) == 0;
                    const unsigned long long a = v[r], b = v[r ^ j];
                    const bool sw = (a > b) == up;
                    v[r] = sw ? b : a;
                    v[r ^ j] = sw ? a : b;
                }
            }
        }
    }
}

template <int PER>
__device__ __forceinline__ void warp_sort_blocked_smem(unsigned long long* sb, int n,
                                                       unsigned lane)
{
    unsigned long long v[PER];
#pragma unroll
    for (int r = 0; r < PER; r++) {
        const int e = (int)lane * PER + r;
        v[r] = e < n ? sb[e] : ~0ull;
    }
    warp_bitonic_blocked<PER>(v, lane);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < PER; r++) {
        const int e = (int)lane * PER + r;
        if (e < n) sb[e] = v[r];
    }
}

// Per-warp survivor buffer: original ids and physical indices (compacted).
struct __align__(16) WarpBuf {
    uint32_t id[kCap + 4];   // +4: padding so 128-bit loads may read past n
    uint32_t j[kCap];
};

// Rank by counting: survivor e goes to position #{f : id_f < id_e} (ids are
// unique).  Each lane owns E survivors; the ids are streamed from shared
// memory four at a time as broadcasts.  For n <= 128 this is cheaper than a
// bitonic network (2 ALU ops per comparison, no data movement).
template <int E, class Emit>
__device__ __forceinline__ void rank_emit(WarpBuf& b, int n, unsigned lane, Emit emit)
{
    if (lane < 4) b.id[n + lane] = 0xffffffffu;
    __syncwarp();
    uint32_t my[E];
    int rank[E];
#pragma unroll
    for (int k = 0; k < E; k++) {
        const int e = (int)lane + 32 * k;
        my[k] = e < n ? b.id[e] : 0xffffffffu;
        rank[k] = 0;
    }
    const uint4* ids4 = reinterpret_cast<const uint4*>(b.id);
    for (int f = 0; f < n; f += 4) {
        const uint4 q = ids4[f >> 2];
#pragma unroll
        for (int k = 0; k < E; k++)
            rank[k] += (int)(q.x < my[k]) + (int)(q.y < my[k]) + (int)(q.z < my[k]) +
                       (int)(q.w < my[k]);
    }
#pragma unroll
    for (int k = 0; k < E; k++) {
        const int e = (int)lane + 32 * k;
        if (e < n) emit(rank[k], b.j[e]);
    }
}

// Emit the n survivors of b in ascending original id: emit(position, j).
template <class Emit>
__device__ __forceinline__ void warp_emit_sorted(WarpBuf& b, int n, unsigned lane, Emit emit)
{
    __syncwarp();
    if (n <= 32) rank_emit<1>(b, n, lane, emit);
    else if (n <= 64) rank_emit<2>(b, n, lane, emit);
    else if (n <= 96) rank_emit<3>(b, n, lane, emit);
    else if (n <= 128) rank_emit<4>(b, n, lane, emit);
    else {   // long skin lists: register bitonic network over (id, j) pairs
        unsigned long long v[8];
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int e = (int)lane * 8 + r;
            v[r] = e < n ? (((unsigned long long)b.id[e] << 32) | b.j[e]) : ~0ull;
        }
        warp_bitonic_blocked<8>(v, lane);
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const int e = (int)lane * 8 + r;
            if (e < n) emit(e, (uint32_t)v[r]);
        }
    }
    __syncwarp();
}

// Engine layout: segment 0 = fluid [0, nf), segment 1 = walls [nf, n); each
// cell-sorted with offsets relative to its segment start.  pos.w = mass.
template <class T>
struct EngAcc {
    static constexpr int kSegs = 2;
    const vec4<T>* __restrict__ pos;
    const uint32_t* __restrict__ id;
    const uint32_t* __restrict__ offs_f;
    const uint32_t* __restrict__ offs_w;
    int64_t nf;
#if SPH_PERIODIC
    int segs;   // 1 when there are no walls (keeps periodic blocks within a warp's runs)
    __device__ __forceinline__ int nsegs() const { return segs; }
#else
    __device__ __forceinline__ static constexpr int nsegs() { return kSegs; }
#endif
    __device__ __forceinline__ void position(int64_t j, T (&x)[3]) const
    {
        vec4<T> p = pos[j];
        x[0] = p.x; x[1] = p.y; x[2] = p.z;
    }
    __device__ __forceinline__ uint32_t idof(int64_t j) const { return id[j]; }
    __device__ __forceinline__ void run(int seg, uint32_t klo, uint32_t khi, int64_t& s0,
                                        int64_t& s1) const
    {
        if (seg == 0) { s0 = offs_f[klo]; s1 = offs_f[khi + 1]; }
        else { s0 = nf + offs_w[klo]; s1 = nf + offs_w[khi + 1]; }
    }
    __device__ __forceinline__ int64_t cand(int64_t s) const { return s; }
};

// Reference layout: x (n, d) row-major, CellLinkedList offsets / particle_ids.
template <class T, int D>
struct GenAcc {
    static constexpr int kSegs = 1;
    const T* __restrict__ x;
    const uint32_t* __restrict__ id;
    const int64_t* __restrict__ offsets;
    const int64_t* __restrict__ pids;
    __device__ __forceinline__ static constexpr int nsegs() { return kSegs; }
    __device__ __forceinline__ void position(int64_t j, T (&p)[3]) const
    {
        p[0] = x[j * D + 0]; p[1] = x[j * D + 1]; p[2] = D == 3 ? x[j * D + 2] : T(0);
    }
    __device__ __forceinline__ uint32_t idof(int64_t j) const { return id[j]; }
    __device__ __forceinline__ void run(int, uint32_t klo, uint32_t khi, int64_t& s0,
                                        int64_t& s1) const
    {
        s0 = offsets[klo]; s1 = offsets[khi + 1];
    }
    __device__ __forceinline__ int64_t cand(int64_t s) const { return pids[s]; }
};

// cell of a position and its row-major key (neighborhood.py:76-84, 112-116)
template <class T, int D>
__device__ __forceinline__ uint32_t cell_key_of(const T (&x)[3], const GridP<T>& g, int (&c)[3])
{
    int cl = 0;
    c[0] = cell_coord<T>(x[0], g.o[0], g.cs, g.s[0], cl);
    c[1] = cell_coord<T>(x[1], g.o[1], g.cs, g.s[1], cl);
    c[2] = D == 3 ? cell_coord<T>(x[2], g.o[2], g.cs, g.s[2], cl) : 0;
    uint32_t k = (uint32_t)c[0] * g.s[1] + c[1];
    if (D == 3) k = k * g.s[2] + c[2];
    return k;
}

struct CollectCounts {
    int stored;     // packed entries written to sb (may exceed kCap: overflow)
    int accepted;   // exact-test accepted neighbours over ALL segments
};

// Collect the neighbours of particle i (position xi) into sb.
//   SKIN == false: store j of storing segments with 0 < r2 < c2;
//   SKIN == true : store j of storing segments with r2 < cs2 (a superset).
// `accepted` counts exact-test neighbours of every segment (the reference's
// capacity count); with SKIN it counts only the non-storing segments.
// store_mask bit s: segment s is stored.
template <class T, int D, bool SKIN, class Acc>
__device__ __forceinline__ CollectCounts warp_collect(const Acc& acc, const GridP<T>& g,
                                                      int64_t i, const T (&xi)[3], T cs2,
                                                      unsigned store_mask, WarpBuf& buf)
{
    const unsigned lane = lane_id();
    const unsigned lt = lanemask_lt();
    int c[3];
    cell_key_of<T, D>(xi, g, c);
#if SPH_PERIODIC
    const PerBlock pb = per_block<T, D>(g, c);
    const int runs_per_seg = per_runs(pb);
#else
    const int xlo = max(c[0] - 1, 0), xhi = min(c[0] + 1, g.s[0] - 1);
    const int ylo = max(c[1] - 1, 0), yhi = min(c[1] + 1, g.s[1] - 1);
    const int zlo = D == 3 ? max(c[2] - 1, 0) : 0, zhi = D == 3 ? min(c[2] + 1, g.s[2] - 1) : 0;
    const int nxr = xhi - xlo + 1;
    const int nyr = D == 3 ? (yhi - ylo + 1) : 1;
    const int runs_per_seg = nxr * nyr;
#endif
    const int nruns = runs_per_seg * acc.nsegs();
    // lane r < nruns owns run r: (seg, ax, ay) -> candidate range [s0, s1)
    int64_t s0 = 0, s1 = 0;
    int seg = 0;
    if ((int)lane < nruns) {
        seg = (int)lane / runs_per_seg;
        const int rr = (int)lane - seg * runs_per_seg;
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
    // flatten: exclusive prefix of run lengths
    const uint32_t len = (uint32_t)(s1 - s0);
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    const uint32_t start = incl - len;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t seg_s0 = (uint32_t)s0 | ((uint32_t)seg << 31);   // index < 2^31
    CollectCounts out{0, 0};
    // each lane tracks the run of its candidate index; indices grow by 32
    // per chunk, so the run only ever moves forward (usually 0-1 runs)
    int r[2] = {0, 0};
    for (uint32_t base = 0; base < total; base += 64) {
        int64_t jj[2];
        int sg[2];
        bool valid[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const uint32_t idx = base + 32 * h + lane;
            while (true) {
                const int nr = r[h] + 1;
                const uint32_t sv = __shfl_sync(0xffffffffu, start, nr & 31);
                const bool adv = nr < nruns && sv <= idx;
                if (!__any_sync(0xffffffffu, adv)) break;
                if (adv) r[h] = nr;
            }
            const uint32_t rss = __shfl_sync(0xffffffffu, seg_s0, r[h]);
            const uint32_t rstart = __shfl_sync(0xffffffffu, start, r[h]);
            sg[h] = (int)(rss >> 31);
            valid[h] = idx < total;
            jj[h] = valid[h] ? acc.cand((int64_t)(rss & 0x7fffffffu) + (idx - rstart)) : 0;
            valid[h] = valid[h] && jj[h] != i;
        }
        T xj[2][3];
        uint32_t idj[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            if (valid[h]) {
                acc.position(jj[h], xj[h]);
                idj[h] = acc.idof(jj[h]);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            bool ok_store = false, ok_count = false;
            if (valid[h]) {
                const T r2 = accept_r2<T, D>(xi, xj[h]);
                const bool exact = (r2 < g.c2) && (r2 > T(0));
                const bool stores = (store_mask >> sg[h]) & 1u;
                if (SKIN) {
                    ok_store = stores && (r2 < cs2);
                    ok_count = !stores && exact;
                } else {
                    ok_store = stores && exact;
                    ok_count = exact;
                }
            }
            const unsigned bs = __ballot_sync(0xffffffffu, ok_store);
            if (ok_store) {
                const int p = out.stored + __popc(bs & lt);
                if (p < kCap) {
                    buf.id[p] = idj[h];
                    buf.j[p] = (uint32_t)jj[h];
                }
            }
            out.stored += __popc(bs);
            out.accepted += __popc(__ballot_sync(0xffffffffu, ok_count));
        }
    }
    return out;
}

// Build exact ordered lists of particles first .. first+count-1 into slots
// slot_first .. (slot_first % 32 == 0), staged per 32-particle tile so the
// block writes lists[tile][t][lane] coalesced.  lcount[slot] = count, or -1
// when more than kCap neighbours qualify (neighborhood.py:200-202).
template <class T, int D, class Acc>
__global__ void __launch_bounds__(kNlThreads, 4)
k_build_lists(const Acc acc, const GridP<T> g, int64_t first, int64_t count,
              int64_t slot_first, int32_t* __restrict__ lists, int32_t* __restrict__ lcount)
{
    extern __shared__ __align__(16) unsigned char nl_smem[];
    int32_t* stage = reinterpret_cast<int32_t*>(nl_smem);
    WarpBuf* bufs =
        reinterpret_cast<WarpBuf*>(nl_smem + sizeof(int32_t) * kCap * kStagePitch);
    int* scnt = reinterpret_cast<int*>(bufs + kNlWarps);

    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    WarpBuf& sb = bufs[warp];
    const int64_t t0 = (int64_t)blockIdx.x * 32;

    for (int p = warp; p < 32; p += kNlWarps) {
        const int64_t t = t0 + p;
        if (t >= count) {
            if (lane == 0) scnt[p] = 0;
            continue;
        }
        const int64_t i = first + t;
        T xi[3];
        acc.position(i, xi);
        CollectCounts cc = warp_collect<T, D, false>(acc, g, i, xi, T(0), 1u, sb);
        if (cc.accepted > kCap) {
            if (lane == 0) scnt[p] = -1;
            __syncwarp();
            continue;
        }
        warp_emit_sorted(sb, cc.stored, lane, [&](int pos, uint32_t j) {
            stage[pos * kStagePitch + p] = (int32_t)j;
        });
        if (lane == 0) scnt[p] = cc.stored;
        __syncwarp();
    }
    __syncthreads();
    int mc = 0;
#pragma unroll 4
    for (int q = 0; q < 32; q++) mc = max(mc, scnt[q]);
    int32_t* dst = lists + (size_t)((slot_first + t0) >> 5) * (kCap * 32);
    for (int idx = threadIdx.x; idx < mc * 32; idx += kNlThreads) {
        const int t = idx >> 5, q = idx & 31;
        dst[ell_off(t) + q * 4] = stage[t * kStagePitch + q];
    }
    if (threadIdx.x < 32 && t0 + threadIdx.x < count)
        lcount[slot_first + t0 + threadIdx.x] = scnt[threadIdx.x];
}

template <class T, int D, class Acc>
inline int launch_build_lists(const Acc& acc, const GridP<T>& g, int64_t first, int64_t count,
                              int64_t slot_first, int32_t* lists, int32_t* lcount,
                              cudaStream_t s)
{
    if (count <= 0) return 0;
    cudaFuncSetAttribute(k_build_lists<T, D, Acc>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kNlSmem);
    int64_t tiles = (count + 31) / 32;
    note_launch(), k_build_lists<T, D, Acc><<<(unsigned)tiles, kNlThreads, kNlSmem, s>>>(
        acc, g, first, count, slot_first, lists, lcount);
    return 0;
}

}  // namespace sph
