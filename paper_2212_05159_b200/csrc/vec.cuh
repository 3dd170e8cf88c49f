// vec.cuh -- 256-bit global vector access (sm_100a LDG.E.ENL2.256 / STG.E.ENL2.256).
//
// A 32-byte vector is 4 doubles or 8 floats; four lanes with consecutive vectors cover one
// 128-byte L1 line per instruction.  Values are widened to double on load (the library
// accumulates in fp64 for both dtypes, A5) and rounded to T on store.
// Pointers must be 32-byte aligned.  Loads use the non-coherent path: the operand must not be
// written by the same kernel.
#pragma once

namespace csrk {

template <typename T> struct V32 { static constexpr int E = 32 / (int)sizeof(T); };

__device__ __forceinline__ void ldv32(const double *p, double *r)
{
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}

__device__ __forceinline__ void ldv32(const float *p, double *r)
{
    float f[8];
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]), "=f"(f[7])
        : "l"(p));
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = (double)f[i];
}

// The same 32 bytes as two 16-byte loads (LDG.128): these allocate in L1, so rows gathered again by
// nearby rows of the same CTA hit L1 (the 256-bit form does not).
__device__ __forceinline__ void ldv32_l1(const double *p, double *r)
{
    asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(r[0]), "=d"(r[1]) : "l"(p));
    asm("ld.global.nc.v2.f64 {%0,%1}, [%2+16];" : "=d"(r[2]), "=d"(r[3]) : "l"(p));
}

__device__ __forceinline__ void ldv32_l1(const float *p, double *r)
{
    float f[8];
    asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]) : "l"(p));
    asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4+16];" : "=f"(f[4]), "=f"(f[5]), "=f"(f[6]), "=f"(f[7]) : "l"(p));
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = (double)f[i];
}

__device__ __forceinline__ void stv32(double *p, const double *r)
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r[0]), "d"(r[1]), "d"(r[2]), "d"(r[3])
                 : "memory");
}

__device__ __forceinline__ void stv32(float *p, const double *r)
{
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"((float)r[0]),
                 "f"((float)r[1]), "f"((float)r[2]), "f"((float)r[3]), "f"((float)r[4]), "f"((float)r[5]),
                 "f"((float)r[6]), "f"((float)r[7])
                 : "memory");
}

// 32 bytes from shared memory as two 16-byte loads.  h (0/1) = which half is loaded first:
// the two 4-lane groups of a quarter-warp phase use opposite orders, so they hit disjoint
// banks even when both rows are 128-byte aligned.
__device__ __forceinline__ void lds32(const double *p, double *r, int h)
{
    const double2 a = reinterpret_cast<const double2 *>(p)[h], b = reinterpret_cast<const double2 *>(p)[h ^ 1];
    const double2 lo = h ? b : a, hi = h ? a : b;
    r[0] = lo.x; r[1] = lo.y; r[2] = hi.x; r[3] = hi.y;
}

__device__ __forceinline__ void lds32(const float *p, double *r, int h)
{
    const float4 a = reinterpret_cast<const float4 *>(p)[h], b = reinterpret_cast<const float4 *>(p)[h ^ 1];
    const float4 lo = h ? b : a, hi = h ? a : b;
    r[0] = lo.x; r[1] = lo.y; r[2] = lo.z; r[3] = lo.w; r[4] = hi.x; r[5] = hi.y; r[6] = hi.z; r[7] = hi.w;
}

// Four lanes (a group of consecutive lanes l = 0..3) each hold partial sums d[0..3] of four
// dot products; after two butterfly steps lane l holds the full sum of product l.  6 SHFL +
// 3 DADD for four dots instead of 16 + 8 for four separate group reductions.  The summation
// order is fixed (deterministic).
__device__ __forceinline__ double transpose_reduce4(const double (&d)[4], int l)
{
    const bool hi = l & 2;
    double s0 = hi ? d[0] : d[2], s1 = hi ? d[1] : d[3];
    double k0 = hi ? d[2] : d[0], k1 = hi ? d[3] : d[1];
    k0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    k1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    const bool odd = l & 1;
    const double s = odd ? k0 : k1;
    double k = odd ? k1 : k0;
    k += __shfl_xor_sync(0xffffffffu, s, 1);
    return k;
}

// G consecutive lanes (G = 4 or 8) each hold partial sums d[0..G) of G dot products; after log2 G
// butterfly steps lane l (of the group) holds the full sum of product l (G - 1 shuffles for G dots;
// fixed summation order, deterministic).
template <int G>
__device__ __forceinline__ double transpose_reduce(const double (&d)[G], int l)
{
    if constexpr (G == 4) {
        return transpose_reduce4(d, l);
    } else {
        static_assert(G == 8, "G = 4 or 8");
        double k[4], k2[2];
        const bool b4 = l & 4, b2 = l & 2, b1 = l & 1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double keep = b4 ? d[4 + i] : d[i], send = b4 ? d[i] : d[4 + i];
            k[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = b2 ? k[2 + i] : k[i], send = b2 ? k[i] : k[2 + i];
            k2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        const double keep = b1 ? k2[1] : k2[0], send = b1 ? k2[0] : k2[1];
        return keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
}

}  // namespace csrk
