// internal.cuh -- host-side declarations shared between the .cu units.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sph {

// error reporting for sph_last_error()
void set_error(const char* msg);
int check_launch(const char* what);

// ---- radix sort (sort.cu) ----------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsItems = 16;
constexpr int kRsTile = kRsThreads * kRsItems;   // 4096 keys per block

inline int64_t rs_blocks(int64_t n) { return (n + kRsTile - 1) / kRsTile; }
// scratch for sorting n keys of key_bytes with uint32 values, excluding the
// caller-owned ping-pong key/value buffers
size_t radix_hist_bytes(int64_t n);

// Stable LSD radix sort of (key, value) pairs over bits [0, key_bits) with
// 8-bit digits.  keys/vals ping-pong between buffer 0 and 1; on return
// *which says which buffer holds the result.  vals_in may be null (== the
// identity 0..n-1).  hist: radix_hist_bytes(n) of scratch.
int radix_sort_u32(uint32_t* k0, uint32_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                   int key_bits, bool vals_identity, void* hist, int* which,
                   cudaStream_t s);
int radix_sort_u64(uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                   int key_bits, bool vals_identity, void* hist, int* which,
                   cudaStream_t s);

// Device-wide exclusive scan of uint32 (in place allowed).  scratch:
// scan_scratch_bytes(n).
size_t scan_scratch_bytes(int64_t n);
int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, void* scratch,
                       cudaStream_t s);

inline int bit_length(uint64_t v)
{
    int b = 0;
    while (b < 64 && (v >> b) != 0) b++;
    return b;
}

inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// simple bump allocator over a caller workspace
struct Bump {
    char* base; size_t size; size_t used = 0;
    Bump(void* b, size_t s) : base(static_cast<char*>(b)), size(s) {}
    template <class T> T* take(size_t count)
    {
        size_t off = align_up(used);
        size_t bytes = align_up(count * sizeof(T));
        if (off + bytes > size) return nullptr;
        used = off + bytes;
        return reinterpret_cast<T*>(base + off);
    }
};

}  // namespace sph
