// common.cuh -- shared device helpers for the B200 SPH hot path (sm_100a).
//
// Exact-arithmetic contract: the reference's f32 run
// evaluates array/f32-scalar operations in binary32 and anything touching a
// Python float literal in binary64, with no FMA contraction, IEEE division
// and square root.  Every floating-point operation on the hot path goes
// through the explicit round-to-nearest intrinsics below, which nvcc never
// contracts or reorders; the library is also built with --fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sph_b200.h"

namespace sph {

constexpr int kWarp = 32;
constexpr int kCap = SPH_NEIGHBOR_CAPACITY;   // neighborhood.py:30

// ---- exact scalar ops, T = run precision ------------------------------------
template <class T> struct RN;
template <> struct RN<float> {
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
    static __device__ __forceinline__ float from_d(double a) { return __double2float_rn(a); }
    // upward-rounded ops for rigorous displacement bounds
    static __device__ __forceinline__ float add_ru(float a, float b) { return __fadd_ru(a, b); }
    static __device__ __forceinline__ float sub_ru(float a, float b) { return __fsub_ru(a, b); }
    static __device__ __forceinline__ float mul_ru(float a, float b) { return __fmul_ru(a, b); }
    static __device__ __forceinline__ float sqrt_ru(float a) { return __fsqrt_ru(a); }
    static constexpr float kOnePlus2Eps = 1.0000002384185791f;   // 1 + 2^-22
};
template <> struct RN<double> {
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
    static __device__ __forceinline__ double from_d(double a) { return a; }
    static __device__ __forceinline__ double add_ru(double a, double b) { return __dadd_ru(a, b); }
    static __device__ __forceinline__ double sub_ru(double a, double b) { return __dsub_ru(a, b); }
    static __device__ __forceinline__ double mul_ru(double a, double b) { return __dmul_ru(a, b); }
    static __device__ __forceinline__ double sqrt_ru(double a) { return __dsqrt_ru(a); }
    static constexpr double kOnePlus2Eps = 1.0000000000000004;   // 1 + 2^-51
};
// ---- periodic boxes (not in the reference) --------------
// libsphb200_periodic.so is the same sources built with -DSPH_PERIODIC=1.
// Per axis k: L[k] > 0 makes the axis periodic with period L[k] over the
// interval [lo[k], hi[k]) (hi = RN(lo + L)); pair differences take the
// minimum image (dx > L/2: dx - L, dx < -L/2: dx + L, one binary32/64 op)
// and a drift leaving [lo, hi) re-enters by one +-L.  All values are the run
// precision, computed on the host (oracle/sph_oracle_impl.h restates the
// same operations).  The box lives in constant memory of the translation
// unit that launches the engine kernels (engine.cu sets it on the caller's
// stream at every engine entry); the bounded build compiles none of this.
#ifndef SPH_PERIODIC
#define SPH_PERIODIC 0
#endif
#if SPH_PERIODIC
struct PerBox {
    float Lf[3], hLf[3], lof[3], hif[3];
    double Ld[3], hLd[3], lod[3], hid[3];
};
static __constant__ PerBox c_box;
template <class T> struct BoxOf;
template <> struct BoxOf<float> {
    static __device__ __forceinline__ float L(int k) { return c_box.Lf[k]; }
    static __device__ __forceinline__ float hL(int k) { return c_box.hLf[k]; }
    static __device__ __forceinline__ float lo(int k) { return c_box.lof[k]; }
    static __device__ __forceinline__ float hi(int k) { return c_box.hif[k]; }
};
template <> struct BoxOf<double> {
    static __device__ __forceinline__ double L(int k) { return c_box.Ld[k]; }
    static __device__ __forceinline__ double hL(int k) { return c_box.hLd[k]; }
    static __device__ __forceinline__ double lo(int k) { return c_box.lod[k]; }
    static __device__ __forceinline__ double hi(int k) { return c_box.hid[k]; }
};
#endif

// minimum image of a pair difference along axis k (identity when bounded)
template <class T>
__device__ __forceinline__ T min_image(T dx, int k)
{
#if SPH_PERIODIC
    const T L = BoxOf<T>::L(k), hL = BoxOf<T>::hL(k);
    if (L > T(0)) {
        if (dx > hL) dx = RN<T>::sub(dx, L);
        else if (dx < -hL) dx = RN<T>::add(dx, L);
    }
#else
    (void)k;
#endif
    return dx;
}

// a drifted coordinate back into the periodic interval (identity when bounded)
template <class T>
__device__ __forceinline__ T wrap_coord(T x, int k)
{
#if SPH_PERIODIC
    const T L = BoxOf<T>::L(k);
    if (L > T(0)) {
        if (x >= BoxOf<T>::hi(k)) x = RN<T>::sub(x, L);
        else if (x < BoxOf<T>::lo(k)) x = RN<T>::add(x, L);
    }
#else
    (void)k;
#endif
    return x;
}

__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ---- division by a loop-invariant divisor ------------------------------------
// a / b correctly rounded from y = RN(1/b) (computed once per thread) with
// the FMA residual step: q0 = RN(a*y), r = a - b*q0 (exact), q = RN(q0 + r*y)
// (Markstein's theorem: y within half an ulp of 1/b and q0 faithful give the
// correctly rounded quotient).  Valid while a, b, q stay well inside the
// normal range -- ok_b says b is -- else the IEEE division is taken.  This is
// bit-identical to __fdiv_rn / __ddiv_rn; tests/test_gpu_kernels.py checks it
// against them on 10^8 quotients per divisor.
// The IEEE fallbacks are out-of-line calls: inlined, the compiler
// if-converts them and evaluates the full division on every pair.
static __device__ __noinline__ float fdiv_slow(float a, float b) { return __fdiv_rn(a, b); }
static __device__ __noinline__ double ddiv_slow(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float fdiv_rcp(float a, float b, float y, bool ok_b)
{
    const float q0 = __fmul_rn(a, y);
    const float r = __fmaf_rn(-b, q0, a);
    const float q1 = __fmaf_rn(r, y, q0);
    const float aa = fabsf(a);
    if (ok_b && aa > 1e-18f && aa < 1e18f) return q1;
    return fdiv_slow(a, b);
}
__device__ __forceinline__ double ddiv_rcp(double a, double b, double y, bool ok_b)
{
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-b, q0, a);
    const double q1 = __fma_rn(r, y, q0);
    const double aa = fabs(a);
    if (ok_b && aa > 1e-140 && aa < 1e140) return q1;
    return ddiv_slow(a, b);
}
template <class T> __device__ __forceinline__ T div_rcp(T a, T b, T y, bool ok_b);
template <> __device__ __forceinline__ float div_rcp<float>(float a, float b, float y, bool ok)
{
    return fdiv_rcp(a, b, y, ok);
}
template <> __device__ __forceinline__ double div_rcp<double>(double a, double b, double y,
                                                              bool ok)
{
    return ddiv_rcp(a, b, y, ok);
}
template <class T> __device__ __forceinline__ T rcp_rn(T b);
template <> __device__ __forceinline__ float rcp_rn<float>(float b) { return __frcp_rn(b); }
template <> __device__ __forceinline__ double rcp_rn<double>(double b) { return __drcp_rn(b); }
template <class T> __device__ __forceinline__ bool rcp_ok(T b)
{
    const double ab = fabs(double(b));
    return ab > 1e-15 && ab < 1e15;
}

// ---- packed vectors ---------------------------------------------------------
template <class T> struct V4;
template <> struct V4<float> { using type = float4; };
template <> struct V4<double> { using type = double4; };
template <class T> struct V2;
template <> struct V2<float> { using type = float2; };
template <> struct V2<double> { using type = double2; };
template <class T> using vec4 = typename V4<T>::type;
template <class T> using vec2 = typename V2<T>::type;

template <class T> __device__ __forceinline__ T comp(const vec4<T>& v, int k)
{
    return k == 0 ? v.x : (k == 1 ? v.y : v.z);
}

// ---- grid cell coordinate (neighborhood.py:76-84) ----------------------------
// c = int(floor(f(f(x - origin) / cell_size))), clamped to [0, ncells-1].
template <class T>
__device__ __forceinline__ int cell_coord(T x, T origin, T cell_size, int ncells,
                                          int& clamped)
{
    T t = RN<T>::div(RN<T>::sub(x, origin), cell_size);
    T f = floor(t);
    // int(floor(t)) on x86 maps NaN and |t| >= 2^63 to INT64_MIN, which the
    // reference then clamps to cell 0; mirror that.
    if (!(f >= T(0)) || f >= T(9.2233720368547758e18)) { clamped = 1; return 0; }
    if (!(f < T(ncells))) { clamped = 1; return ncells - 1; }
    return int(f);
}

// ---- Wendland C2 factors (physics.py:113-117, 184-186), binary64 ------------
// fac = gw / r with gw = -5.0*alpha_d*q*tq*tq*tq/h, tq = 1.0 - 0.5*q.
template <class T>
__device__ __forceinline__ double grad_fac(T r, T q, T h, T alpha_d)
{
    double tq = dsub(1.0, dmul(0.5, double(q)));
    double gw = dmul(-5.0, double(alpha_d));
    gw = dmul(gw, double(q));
    gw = dmul(gw, tq);
    gw = dmul(gw, tq);
    gw = dmul(gw, tq);
    gw = ddiv(gw, double(h));
    return ddiv(gw, double(r));
}

// the same with 1/h precomputed (rh = RN(1/(double)h), ok = rcp_ok(h))
template <class T>
__device__ __forceinline__ double grad_fac_rh(T r, T q, T h, double m5a, double rh, bool ok)
{
    const double tq = dsub(1.0, dmul(0.5, double(q)));
    double gw = dmul(m5a, double(q));   // m5a = -5.0 * alpha_d
    gw = dmul(gw, tq);
    gw = dmul(gw, tq);
    gw = dmul(gw, tq);
    gw = ddiv_rcp(gw, double(h), rh, ok);
    return ddiv(gw, double(r));
}

// w = alpha_d*tq*tq*tq*tq*(2.0*q + 1.0)
template <class T>
__device__ __forceinline__ double kernel_w(T q, T alpha_d)
{
    double tq = dsub(1.0, dmul(0.5, double(q)));
    double w = dmul(double(alpha_d), tq);
    w = dmul(w, tq);
    w = dmul(w, tq);
    w = dmul(w, tq);
    return dmul(w, dadd(dmul(2.0, double(q)), 1.0));
}

// ---- warp helpers -----------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <class U>
__device__ __forceinline__ U warp_sum(U v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

__device__ __forceinline__ unsigned warp_min_u32(unsigned v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Order-preserving maps so exact max/min reductions can use integer atomics.
// Non-negative doubles order like their bit patterns.
__device__ __forceinline__ unsigned long long dbits(double v)
{
    return (unsigned long long)__double_as_longlong(v);
}
// float -> monotone u32 key (total order, -0 < +0)
__device__ __forceinline__ unsigned fkey(float f)
{
    unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ unsigned long long dkey(double f)
{
    unsigned long long u = (unsigned long long)__double_as_longlong(f);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// process-wide count of kernel launches issued by this library (bench.py
// reports it as gpu_launches); defined in sort.cu
void note_launch();

// Programmatic dependent launch (sm_90+): the sub-step kernels are launched
// with programmaticStreamSerialization, so a kernel's blocks may be
// scheduled while the previous kernel's last wave still runs.  Every kernel
// launched that way calls pdl_begin() first: griddepcontrol.wait blocks
// until the previous grid has completed and its writes are visible (so the
// stream order is unchanged), then launch_dependents lets the next grid
// launch once all of this grid's blocks are resident.  Without PDL both are
// no-ops.  Measured (bench, alternating A/B runs): 2D 1M +0.7% (short
// sub-step kernels, ~10-120 us), 3D 4M -1.1% (ms-long sweeps): the engine
// enables it for 2D only (pdl_for).
#ifndef SPH_PDL
#define SPH_PDL 1
#endif
__device__ __forceinline__ void pdl_begin()
{
#if SPH_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

template <class... KArgs, class... Args>
inline void launch_pdl(bool pdl, void (*kernel)(KArgs...), int grid, int block, cudaStream_t s,
                       Args&&... args)
{
    note_launch();
#if SPH_PDL
    if (!pdl) {
        kernel<<<grid, block, 0, s>>>(static_cast<Args&&>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
#else
    kernel<<<grid, block, 0, s>>>(static_cast<Args&&>(args)...);
#endif
}

inline int grid_for(int64_t n, int threads, int cap = 1 << 30)
{
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return int(g);
}

}  // namespace sph
