// sort.cu -- device radix sort and scans (replaces sorting.py:27-70 and the
// count/prefix/scatter phases of neighborhood.py:120-173).
//
// Stable LSD radix sort, 8-bit digits, reduce-then-scan per pass:
//   1. k_radix_hist: per-tile digit histogram, warp-aggregated with
//      match.any so runs of equal digits (cell-sorted input) cost one shared
//      atomic per warp instead of one per key;
//   2. exclusive scan of the digit-major [256][tiles] table -> the global
//      write base of every (digit, tile);
//   3. k_radix_scatter: stable in-tile ranks with match.any + per-warp digit
//      counters, then scatter.
// The result equals np.argsort(keys, kind="stable") (the reference's
// comparison_sort_permutation), which is what the CLL and particle sort need.
#include <atomic>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "internal.cuh"

namespace sph {

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static thread_local char g_err[512];
void set_error(const char* msg)
{
    std::strncpy(g_err, msg, sizeof(g_err) - 1);
    g_err[sizeof(g_err) - 1] = 0;
}

int check_launch(const char* what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        char buf[512];
        std::snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
        set_error(buf);
        return SPH_ERR_CUDA;
    }
    return SPH_OK;
}

// ---------------------------------------------------------------------------
// scans
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

// block-wide exclusive scan of one value per thread; *total = block sum
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t& total)
{
    constexpr int kW = kScanThreads / 32;
    __shared__ uint32_t wt[kW];
    __shared__ uint32_t tot_s;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    if (lane == 31) wt[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (unsigned)kW ? wt[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= (unsigned)o) wi += t;
        }
        if (lane < (unsigned)kW) wt[lane] = wi - w;
        if (lane == (unsigned)kW - 1) tot_s = wi;
    }
    __syncthreads();
    uint32_t r = wt[warp] + incl - v;
    total = tot_s;
    __syncthreads();
    return r;
}

__global__ void k_scan_tile_sums(const uint32_t* __restrict__ in, int64_t n,
                                 uint32_t* __restrict__ sums)
{
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t acc = 0;
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = base + (int64_t)k * kScanThreads + threadIdx.x;
        if (idx < n) acc += in[idx];
    }
    uint32_t tot;
    block_exclusive_scan(acc, tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// single-block exclusive scan over the tile sums (any count)
__global__ void k_scan_sums(uint32_t* sums, int64_t m)
{
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < m; b0 += kScanThreads) {
        int64_t idx = b0 + threadIdx.x;
        uint32_t v = idx < m ? sums[idx] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan(v, tot);
        if (idx < m) sums[idx] = ex + carry;
        carry += tot;
        __syncthreads();
    }
}

__global__ void k_scan_apply(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                             int64_t n, const uint32_t* __restrict__ sums)
{
    // blocked arrangement: thread t owns items [t*16, t*16+16) of the tile
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = base + k;
        v[k] = idx < n ? in[idx] : 0;
        acc += v[k];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan(acc, tot) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = base + k;
        if (idx < n) out[idx] = run;
        run += v[k];
    }
}

size_t scan_scratch_bytes(int64_t n)
{
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    return align_up(sizeof(uint32_t) * (size_t)(tiles > 0 ? tiles : 1));
}

int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, void* scratch,
                       cudaStream_t s)
{
    if (n <= 0) return SPH_OK;
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    uint32_t* sums = static_cast<uint32_t*>(scratch);
    note_launch(), k_scan_tile_sums<<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, sums);
    note_launch(), k_scan_sums<<<1, kScanThreads, 0, s>>>(sums, tiles);
    note_launch(), k_scan_apply<<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, n, sums);
    return check_launch("exclusive_scan_u32");
}

// ---------------------------------------------------------------------------
// radix sort
// ---------------------------------------------------------------------------
template <class K>
__global__ void __launch_bounds__(kRsThreads)
k_radix_hist(const K* __restrict__ keys, int64_t n, int shift, uint32_t* __restrict__ hist,
             int64_t ntiles)
{
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRsTile;
    const unsigned lane = lane_id();
    for (int k = 0; k < kRsItems; k++) {
        int64_t idx = base + (int64_t)k * kRsThreads + threadIdx.x;
        unsigned d = idx < n ? (unsigned)((keys[idx] >> shift) & 255u) : 256u;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d < 256u && lane == (unsigned)(__ffs(peers) - 1))
            atomicAdd(&h[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <class K>
__global__ void __launch_bounds__(kRsThreads)
k_radix_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin, bool vals_identity,
                K* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n, int shift,
                const uint32_t* __restrict__ offs, int64_t ntiles)
{
    constexpr int kWarps = kRsThreads / 32;
    __shared__ uint32_t wcnt[kWarps][256];
    __shared__ uint32_t gbase[256];
    for (int w = 0; w < kWarps; w++) wcnt[w][threadIdx.x] = 0;
    gbase[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles + blockIdx.x];
    __syncthreads();

    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const int64_t wbase = (int64_t)blockIdx.x * kRsTile + (int64_t)warp * (kRsItems * 32);
    const unsigned lt = lanemask_lt();
    K key[kRsItems];
    uint32_t val[kRsItems];
    uint32_t rank[kRsItems];
    unsigned dig[kRsItems];
#pragma unroll
    for (int k = 0; k < kRsItems; k++) {
        int64_t idx = wbase + (int64_t)k * 32 + lane;
        bool valid = idx < n;
        key[k] = valid ? kin[idx] : K(0);
        val[k] = valid ? (vals_identity ? (uint32_t)idx : vin[idx]) : 0u;
        unsigned d = valid ? (unsigned)((key[k] >> shift) & 255u) : 256u;
        dig[k] = d;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = d < 256u ? wcnt[warp][d] : 0u;
        __syncwarp();
        if (d < 256u && lane == (unsigned)(__ffs(peers) - 1))
            wcnt[warp][d] = before + (uint32_t)__popc(peers);
        __syncwarp();
        rank[k] = before + (uint32_t)__popc(peers & lt);
    }
    __syncthreads();
    {   // exclusive prefix over warps, per digit
        uint32_t run = 0;
        for (int w = 0; w < kWarps; w++) {
            uint32_t c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRsItems; k++) {
        unsigned d = dig[k];
        if (d < 256u) {
            uint32_t pos = gbase[d] + wcnt[warp][d] + rank[k];
            kout[pos] = key[k];
            vout[pos] = val[k];
        }
    }
}

size_t radix_hist_bytes(int64_t n)
{
    int64_t tiles = rs_blocks(n);
    if (tiles < 1) tiles = 1;
    size_t table = align_up(sizeof(uint32_t) * 256 * (size_t)tiles);
    return table + scan_scratch_bytes(256 * tiles);
}

template <class K>
static int radix_sort_impl(K* k0, K* k1, uint32_t* v0, uint32_t* v1, int64_t n, int key_bits,
                           bool vals_identity, void* hist, int* which, cudaStream_t s)
{
    *which = 0;
    if (n <= 0) return SPH_OK;
    int passes = (key_bits + 7) / 8;
    if (passes < 1) passes = 1;
    const int64_t tiles = rs_blocks(n);
    uint32_t* table = static_cast<uint32_t*>(hist);
    void* scan_tmp = static_cast<char*>(hist) + align_up(sizeof(uint32_t) * 256 * (size_t)tiles);
    K* kin = k0; K* kout = k1;
    uint32_t* vin = v0; uint32_t* vout = v1;
    bool ident = vals_identity;
    for (int p = 0; p < passes; p++) {
        int shift = p * 8;
        note_launch(), k_radix_hist<K><<<(unsigned)tiles, kRsThreads, 0, s>>>(kin, n, shift, table, tiles);
        int rc = exclusive_scan_u32(table, table, 256 * tiles, scan_tmp, s);
        if (rc) return rc;
        note_launch(), k_radix_scatter<K><<<(unsigned)tiles, kRsThreads, 0, s>>>(
            kin, vin, ident, kout, vout, n, shift, table, tiles);
        if ((rc = check_launch("radix_scatter"))) return rc;
        ident = false;
        K* tk = kin; kin = kout; kout = tk;
        uint32_t* tv = vin; vin = vout; vout = tv;
    }
    *which = (kin == k0) ? 0 : 1;
    return SPH_OK;
}

int radix_sort_u32(uint32_t* k0, uint32_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                   int key_bits, bool vals_identity, void* hist, int* which, cudaStream_t s)
{
    return radix_sort_impl<uint32_t>(k0, k1, v0, v1, n, key_bits, vals_identity, hist, which, s);
}

int radix_sort_u64(uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                   int key_bits, bool vals_identity, void* hist, int* which, cudaStream_t s)
{
    return radix_sort_impl<uint64_t>(k0, k1, v0, v1, n, key_bits, vals_identity, hist, which, s);
}

// ---------------------------------------------------------------------------
// radix_sort_permutation ABI (sorting.py:46-70)
// ---------------------------------------------------------------------------
__global__ void k_minmax_i64(const int64_t* __restrict__ keys, int64_t n,
                             unsigned long long* __restrict__ out /*[2]: min key, max*/)
{
    unsigned long long mn = ~0ull, mx = 0ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        // order-preserving map of int64 to uint64
        unsigned long long u = (unsigned long long)keys[i] ^ 0x8000000000000000ull;
        mn = u < mn ? u : mn;
        mx = u > mx ? u : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o);
        unsigned long long b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if (lane_id() == 0) {
        atomicMin(&out[0], mn);
        atomicMax(&out[1], mx);
    }
}

__global__ void k_u32_to_i64(const uint32_t* __restrict__ in, int64_t* __restrict__ out,
                             int64_t n)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int64_t)in[i];
}

}  // namespace sph

using namespace sph;

extern "C" size_t sph_sort_workspace_bytes(int64_t n)
{
    size_t b = align_up(16);
    b += 2 * align_up(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    b += 2 * align_up(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
    b += radix_hist_bytes(n);
    return b;
}

extern "C" int sph_radix_sort_perm(const int64_t* keys, int64_t n, int64_t* perm, void* ws,
                                   size_t ws_bytes, cudaStream_t s)
{
    if (n <= 0) return SPH_OK;
    if (n >= (int64_t)UINT32_MAX) { set_error("too many keys"); return SPH_ERR_UNSUPPORTED; }
    if (ws_bytes < sph_sort_workspace_bytes(n)) return SPH_ERR_WORKSPACE;
    Bump bump(ws, ws_bytes);
    unsigned long long* mm = bump.take<unsigned long long>(2);
    uint64_t* k0 = bump.take<uint64_t>(n);
    uint64_t* k1 = bump.take<uint64_t>(n);
    uint32_t* v0 = bump.take<uint32_t>(n);
    uint32_t* v1 = bump.take<uint32_t>(n);
    void* hist = bump.take<char>(radix_hist_bytes(n));
    unsigned long long init[2] = {~0ull, 0ull};
    cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s);
    note_launch(), k_minmax_i64<<<grid_for(n, 256, 2048), 256, 0, s>>>(keys, n, mm);
    unsigned long long host[2];
    cudaMemcpyAsync(host, mm, sizeof(host), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("radix minmax");
    int64_t mn = (int64_t)(host[0] ^ 0x8000000000000000ull);
    int64_t mx = (int64_t)(host[1] ^ 0x8000000000000000ull);
    if (mn < 0) { set_error("radix sort keys must be non-negative"); return SPH_ERR_NEGATIVE_KEY; }
    int bits = bit_length((uint64_t)mx);
    cudaMemcpyAsync(k0, keys, sizeof(int64_t) * (size_t)n, cudaMemcpyDeviceToDevice, s);
    int which = 0;
    int rc = radix_sort_u64(k0, k1, v0, v1, n, bits, true, hist, &which, s);
    if (rc) return rc;
    note_launch(), k_u32_to_i64<<<grid_for(n, 256), 256, 0, s>>>(which ? v1 : v0, perm, n);
    return check_launch("radix_sort_perm");
}

extern "C" int sph_abi_version(void) { return SPH_ABI_VERSION; }
extern "C" const char* sph_last_error(void) { return g_err; }
extern "C" long long sph_kernel_launches(void) { return g_launches.load(); }
