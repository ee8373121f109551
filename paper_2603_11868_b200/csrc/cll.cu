// cll.cu -- cell keys, stable cell linked list, permutation gathers.
//
// Replaces neighborhood.py:105-173 (_compute_keys, _count_cells,
// _scatter_cells, build_cell_linked_list) and variables.py:132-145
// (apply_permutation) on the device.  The CLL is the stable sort of the
// particles by row-major cell key (particle_ids == argsort(keys, stable)),
// so it is built as a radix sort of (key, index) followed by a per-cell
// lower-bound search for the offsets.
#include "common.cuh"
#include "internal.cuh"

namespace sph {

// neighborhood.py:105-117: row-major key lin = (c0*s1 + c1)*s2 + c2 with
// clamped coordinates; counts clamped particles.
template <class T, class KeyOut>
__global__ void k_cell_keys(const T* __restrict__ x, int64_t n, int dim, T o0, T o1, T o2,
                            T cs, int s0, int s1, int s2, KeyOut* __restrict__ keys,
                            uint32_t* __restrict__ oob_count)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int clamped = 0;
    if (i < n) {
        int c0 = cell_coord<T>(x[i * dim + 0], o0, cs, s0, clamped);
        int c1 = cell_coord<T>(x[i * dim + 1], o1, cs, s1, clamped);
        int64_t lin = (int64_t)c0 * s1 + c1;
        if (dim == 3) {
            int c2 = cell_coord<T>(x[i * dim + 2], o2, cs, s2, clamped);
            lin = lin * s2 + c2;
        }
        keys[i] = (KeyOut)lin;
    }
    unsigned b = __ballot_sync(0xffffffffu, clamped);
    if (oob_count && lane_id() == 0 && b) atomicAdd(oob_count, (uint32_t)__popc(b));
}

// offsets[c] = lower_bound(sorted_keys, c) for c in [0, ncells]
template <class OffT>
__global__ void k_offsets_lower_bound(const uint32_t* __restrict__ keys, int64_t n,
                                      int64_t ncells, OffT* __restrict__ offsets, OffT add)
{
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncells) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((int64_t)keys[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    offsets[c] = (OffT)lo + add;
}

__global__ void k_u32_to_i64_b(const uint32_t* __restrict__ in, int64_t* __restrict__ out,
                               int64_t n)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int64_t)in[i];
}

template <int B>
struct Blob { unsigned char b[B]; };

template <class E>
__global__ void k_gather(E* __restrict__ dst, const E* __restrict__ src,
                         const int64_t* __restrict__ perm, int64_t n)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

void launch_offsets_u32(const uint32_t* sorted_keys, int64_t n, int64_t ncells,
                        uint32_t* offsets, cudaStream_t s)
{
    note_launch(), k_offsets_lower_bound<uint32_t><<<grid_for(ncells + 1, 256), 256, 0, s>>>(
        sorted_keys, n, ncells, offsets, 0u);
}

}  // namespace sph

using namespace sph;

template <class T>
static int cell_keys_impl(const T* x, int64_t n, int dim, const T* origin, T cs,
                          const int64_t* shape, int64_t* keys, uint32_t* oob, cudaStream_t s)
{
    if (n <= 0) return SPH_OK;
    if (dim != 2 && dim != 3) return SPH_ERR_INVALID;
    note_launch(), k_cell_keys<T, int64_t><<<grid_for(n, 256), 256, 0, s>>>(
        x, n, dim, origin[0], origin[1], dim == 3 ? origin[2] : T(0), cs, (int)shape[0],
        (int)shape[1], dim == 3 ? (int)shape[2] : 1, keys, oob);
    return check_launch("cell_keys");
}

extern "C" int sph_cell_keys_f32(const float* x, int64_t n, int dim, const float* origin,
                                 float cell_size, const int64_t* shape, int64_t* keys,
                                 uint32_t* oob_count, cudaStream_t s)
{
    return cell_keys_impl<float>(x, n, dim, origin, cell_size, shape, keys, oob_count, s);
}

extern "C" int sph_cell_keys_f64(const double* x, int64_t n, int dim, const double* origin,
                                 double cell_size, const int64_t* shape, int64_t* keys,
                                 uint32_t* oob_count, cudaStream_t s)
{
    return cell_keys_impl<double>(x, n, dim, origin, cell_size, shape, keys, oob_count, s);
}

extern "C" size_t sph_cll_workspace_bytes(int64_t n, int64_t ncells)
{
    (void)ncells;
    size_t m = (size_t)(n > 0 ? n : 1);
    return 4 * align_up(sizeof(uint32_t) * m) + radix_hist_bytes(n) + 256;
}

template <class T>
static int cll_build_impl(const T* x, int64_t n, int dim, const T* origin, T cs,
                          const int64_t* shape, int64_t* offsets, int64_t* pids,
                          uint32_t* oob, void* ws, size_t ws_bytes, cudaStream_t s)
{
    if (dim != 2 && dim != 3) return SPH_ERR_INVALID;
    int64_t ncells = shape[0] * shape[1] * (dim == 3 ? shape[2] : 1);
    if (ncells >= (int64_t)UINT32_MAX || n >= (int64_t)UINT32_MAX) {
        set_error("grid or particle count exceeds 32-bit cell keys");
        return SPH_ERR_UNSUPPORTED;
    }
    if (n <= 0) {
        cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (size_t)(ncells + 1), s);
        return check_launch("cll_build(empty)");
    }
    if (ws_bytes < sph_cll_workspace_bytes(n, ncells)) return SPH_ERR_WORKSPACE;
    Bump bump(ws, ws_bytes);
    uint32_t* k0 = bump.take<uint32_t>(n);
    uint32_t* k1 = bump.take<uint32_t>(n);
    uint32_t* v0 = bump.take<uint32_t>(n);
    uint32_t* v1 = bump.take<uint32_t>(n);
    void* hist = bump.take<char>(radix_hist_bytes(n));
    note_launch(), k_cell_keys<T, uint32_t><<<grid_for(n, 256), 256, 0, s>>>(
        x, n, dim, origin[0], origin[1], dim == 3 ? origin[2] : T(0), cs, (int)shape[0],
        (int)shape[1], dim == 3 ? (int)shape[2] : 1, k0, oob);
    int which = 0;
    int rc = radix_sort_u32(k0, k1, v0, v1, n, bit_length((uint64_t)(ncells - 1)), true, hist,
                            &which, s);
    if (rc) return rc;
    const uint32_t* sk = which ? k1 : k0;
    const uint32_t* sv = which ? v1 : v0;
    note_launch(), k_u32_to_i64_b<<<grid_for(n, 256), 256, 0, s>>>(sv, pids, n);
    note_launch(), k_offsets_lower_bound<int64_t><<<grid_for(ncells + 1, 256), 256, 0, s>>>(sk, n, ncells,
                                                                            offsets, 0);
    return check_launch("cll_build");
}

extern "C" int sph_cll_build_f32(const float* x, int64_t n, int dim, const float* origin,
                                 float cell_size, const int64_t* shape, int64_t* offsets,
                                 int64_t* particle_ids, uint32_t* oob_count, void* ws,
                                 size_t ws_bytes, cudaStream_t s)
{
    return cll_build_impl<float>(x, n, dim, origin, cell_size, shape, offsets, particle_ids,
                                 oob_count, ws, ws_bytes, s);
}

extern "C" int sph_cll_build_f64(const double* x, int64_t n, int dim, const double* origin,
                                 double cell_size, const int64_t* shape, int64_t* offsets,
                                 int64_t* particle_ids, uint32_t* oob_count, void* ws,
                                 size_t ws_bytes, cudaStream_t s)
{
    return cll_build_impl<double>(x, n, dim, origin, cell_size, shape, offsets, particle_ids,
                                  oob_count, ws, ws_bytes, s);
}

extern "C" int sph_gather(void* dst, const void* src, const int64_t* perm, int64_t n,
                          int elem_bytes, cudaStream_t s)
{
    if (n <= 0) return SPH_OK;
    int g = grid_for(n, 256);
    switch (elem_bytes) {
    case 4: note_launch(), k_gather<uint32_t><<<g, 256, 0, s>>>((uint32_t*)dst, (const uint32_t*)src, perm, n); break;
    case 8: note_launch(), k_gather<uint2><<<g, 256, 0, s>>>((uint2*)dst, (const uint2*)src, perm, n); break;
    case 12: note_launch(), k_gather<Blob<12>><<<g, 256, 0, s>>>((Blob<12>*)dst, (const Blob<12>*)src, perm, n); break;
    case 16: note_launch(), k_gather<uint4><<<g, 256, 0, s>>>((uint4*)dst, (const uint4*)src, perm, n); break;
    case 24: note_launch(), k_gather<Blob<24>><<<g, 256, 0, s>>>((Blob<24>*)dst, (const Blob<24>*)src, perm, n); break;
    case 32: note_launch(), k_gather<Blob<32>><<<g, 256, 0, s>>>((Blob<32>*)dst, (const Blob<32>*)src, perm, n); break;
    default: set_error("sph_gather: unsupported element size"); return SPH_ERR_INVALID;
    }
    return check_launch("gather");
}

extern "C" int sph_copy(void* dst, const void* src, int64_t nbytes, cudaStream_t s)
{
    if (nbytes <= 0) return SPH_OK;
    cudaMemcpyAsync(dst, src, (size_t)nbytes, cudaMemcpyDeviceToDevice, s);
    return check_launch("copy");
}
