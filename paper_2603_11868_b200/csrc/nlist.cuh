// nlist.cuh -- ordered neighbour lists (neighborhood.py:176-227).
//
// The reference collects, for each particle i, every j != i of the clamped
// 3^d cell block around i's CURRENT cell (membership from the cell linked
// list built at the start of the advective step, neighborhood.py:188-213)
// with 0 < r2 < cutoff^2, and visits them in ascending ORIGINAL id.  That
// order fixes every floating-point accumulation, so it is reproduced exactly.
//
// B200 mapping: one warp per particle.  The block's row-major cell keys make
// each (ax, ay) column of the block one contiguous key range (3 ranges in
// 2D, 9 in 3D), i.e. one contiguous run of the cell-sorted particle array
// per segment; lanes test 32 candidates per step, survivors are compacted by
// ballot into a per-warp shared buffer of packed (id << 32 | j), sorted by a
// warp bitonic network (registers for <= 32 survivors, shared memory above),
// then staged so the block writes its 32-particle tile of lists coalesced in
// a tile-ELL layout: lists[tile][t][lane].  The thread-per-particle sweeps
// then read entry t of 32 consecutive particles as one 128-byte line.
#pragma once

#include "common.cuh"
#include "physics.cuh"

namespace sph {

constexpr int kNlWarps = 8;
constexpr int kNlThreads = kNlWarps * 32;
constexpr int kStagePitch = 33;   // conflict-free transposition
constexpr size_t kNlSmem = sizeof(int32_t) * kCap * kStagePitch +
                           sizeof(unsigned long long) * kNlWarps * kCap + sizeof(int) * 32;

template <class T>
struct GridP {
    T o[3]; T cs; T c2; int s[3];
};

__device__ __forceinline__ size_t ell_index(int64_t slot, int t)
{
    return (size_t)(slot >> 5) * (kCap * 32) + (size_t)t * 32 + (size_t)(slot & 31);
}

// ascending bitonic sort of sb[0..np), np a power of two in [32, 256]
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
            bool take_min = (lower == up);
            unsigned long long mn = o < v ? o : v, mx = o < v ? v : o;
            v = take_min ? mn : mx;
        }
    }
    return v;
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
    bool store_walls;   // walls' own lists keep fluid neighbours only
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
    __device__ __forceinline__ bool store(int seg) const { return seg == 0 || store_walls; }
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
    __device__ __forceinline__ bool store(int) const { return true; }
    __device__ __forceinline__ int64_t cand(int64_t s) const { return pids[s]; }
};

// Build the ordered lists of particles first .. first+count-1 into slots
// slot_first .. (slot_first % 32 == 0).  lcount[slot] = stored count, or -1
// when more than kCap neighbours qualify (neighborhood.py:200-202).
template <class T, int D, class Acc>
__global__ void __launch_bounds__(kNlThreads)
k_build_lists(const Acc acc, const GridP<T> g, int64_t first, int64_t count,
              int64_t slot_first, int32_t* __restrict__ lists, int32_t* __restrict__ lcount)
{
    extern __shared__ __align__(16) unsigned char nl_smem[];
    int32_t* stage = reinterpret_cast<int32_t*>(nl_smem);
    unsigned long long* sbuf_all =
        reinterpret_cast<unsigned long long*>(nl_smem + sizeof(int32_t) * kCap * kStagePitch);
    int* scnt = reinterpret_cast<int*>(sbuf_all + kNlWarps * kCap);

    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    unsigned long long* sb = sbuf_all + warp * kCap;
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
        int cl = 0;
        const int cx = cell_coord<T>(xi[0], g.o[0], g.cs, g.s[0], cl);
        const int cy = cell_coord<T>(xi[1], g.o[1], g.cs, g.s[1], cl);
        const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.s[0] - 1);
        const int ylo = max(cy - 1, 0), yhi = min(cy + 1, g.s[1] - 1);
        int zlo = 0, zhi = 0;
        if (D == 3) {
            const int cz = cell_coord<T>(xi[2], g.o[2], g.cs, g.s[2], cl);
            zlo = max(cz - 1, 0);
            zhi = min(cz + 1, g.s[2] - 1);
        }
        int n_tot = 0, n_st = 0;
        for (int ax = xlo; ax <= xhi; ax++) {
            const int ay_end = D == 3 ? yhi : ylo;   // 2D: one key range per ax
            for (int ay = ylo; ay <= ay_end; ay++) {
                uint32_t klo, khi;
                if (D == 3) {
                    uint32_t rowk = ((uint32_t)ax * g.s[1] + ay) * g.s[2];
                    klo = rowk + zlo;
                    khi = rowk + zhi;
                } else {
                    klo = (uint32_t)ax * g.s[1] + ylo;
                    khi = (uint32_t)ax * g.s[1] + yhi;
                }
#pragma unroll
                for (int seg = 0; seg < Acc::kSegs; seg++) {
                    int64_t s0, s1;
                    acc.run(seg, klo, khi, s0, s1);
                    const bool st = acc.store(seg);
                    for (int64_t sbase = s0; sbase < s1; sbase += 32) {
                        const int64_t sidx = sbase + lane;
                        bool ok = false;
                        int64_t j = 0;
                        if (sidx < s1) {
                            j = acc.cand(sidx);
                            if (j != i) {
                                T xj[3];
                                acc.position(j, xj);
                                T r2 = accept_r2<T, D>(xi, xj);
                                ok = (r2 < g.c2) && (r2 > T(0));
                            }
                        }
                        const unsigned b = __ballot_sync(0xffffffffu, ok);
                        if (st) {
                            if (ok) {
                                int pos = n_st + __popc(b & lt);
                                if (pos < kCap)
                                    sb[pos] = ((unsigned long long)acc.idof(j) << 32) |
                                              (unsigned long long)(uint32_t)j;
                            }
                            n_st += __popc(b);
                        }
                        n_tot += __popc(b);
                    }
                }
            }
        }
        if (n_tot > kCap) {
            if (lane == 0) scnt[p] = -1;
            __syncwarp();
            continue;
        }
        __syncwarp();
        if (n_st <= 32) {
            unsigned long long v = lane < (unsigned)n_st ? sb[lane] : ~0ull;
            v = warp_bitonic_reg(v, lane);
            if (lane < (unsigned)n_st) stage[lane * kStagePitch + p] = (int32_t)(uint32_t)v;
        } else {
            int np = 64;
            while (np < n_st) np <<= 1;
            for (int k = n_st + lane; k < np; k += 32) sb[k] = ~0ull;
            __syncwarp();
            warp_bitonic_smem(sb, np, lane);
            for (int k = lane; k < n_st; k += 32)
                stage[k * kStagePitch + p] = (int32_t)(uint32_t)sb[k];
        }
        if (lane == 0) scnt[p] = n_st;
        __syncwarp();
    }
    __syncthreads();
    int mc = 0;
#pragma unroll 4
    for (int q = 0; q < 32; q++) mc = max(mc, scnt[q]);
    int32_t* dst = lists + (size_t)((slot_first + t0) >> 5) * (kCap * 32);
    for (int idx = threadIdx.x; idx < mc * 32; idx += kNlThreads)
        dst[idx] = stage[(idx >> 5) * kStagePitch + (idx & 31)];
    if (threadIdx.x < 32 && t0 + threadIdx.x < count)
        lcount[slot_first + t0 + threadIdx.x] = scnt[threadIdx.x];
}

template <class T, int D, class Acc>
inline int launch_build_lists(const Acc& acc, const GridP<T>& g, int64_t first, int64_t count,
                              int64_t slot_first, int32_t* lists, int32_t* lcount,
                              cudaStream_t s)
{
    if (count <= 0) return 0;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_build_lists<T, D, Acc>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNlSmem);
        attr_set = true;
    }
    int64_t tiles = (count + 31) / 32;
    note_launch(), k_build_lists<T, D, Acc><<<(unsigned)tiles, kNlThreads, kNlSmem, s>>>(acc, g, first, count,
                                                                          slot_first, lists,
                                                                          lcount);
    return 0;
}

}  // namespace sph
