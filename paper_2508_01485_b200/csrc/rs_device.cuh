// Device helpers of librs: exact fixed-point accumulation (reading C-12) and
// vertex-group abstractions for degree-binned scheduling.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rs {

// ---------------------------------------------------------------------------
// Exact fixed point. A per-head triad sum is a sum of non-negative fp64 terms;
// each term is rounded once onto the 2^-64 grid (round-half-even, from the
// IEEE bits) and the grid integers are summed exactly in 128 bits, so the sum
// does not depend on the order threads add them (C-12). Terms are
// unnormalised (omega_max is applied once in the epilogue), bounded by
// omega_max <= k log2(k-1) (wide_bound): < 2^11 for the dense k <= 254, about
// 2^17 in the all-communities mode at 10^4 communities, so a term is < 2^18 and
// every per-head sum stays far below 2^128.
// ---------------------------------------------------------------------------
struct U128 {
    unsigned long long lo, hi;
};

__device__ __forceinline__ U128 u128_zero() { return U128{0ull, 0ull}; }

__device__ __forceinline__ U128 u128_add(U128 a, U128 b) {
    U128 r;
    asm("add.cc.u64 %0, %2, %4;\n\taddc.u64 %1, %3, %5;"
        : "=l"(r.lo), "=l"(r.hi)
        : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
    return r;
}

// round-half-even(t * 2^64) for finite t >= 0 (t < 2^64).
__device__ __forceinline__ U128 fx_quantize(double t) {
    unsigned long long bits = (unsigned long long)__double_as_longlong(t);
    int e = (int)((bits >> 52) & 0x7ff);
    if (e == 0) return u128_zero();               // +-0 and subnormals (< 2^-1022)
    unsigned long long m = (bits & 0xFFFFFFFFFFFFFull) | (1ull << 52);
    int s = e - 1011;                             // t * 2^64 = m * 2^s
    if (s >= 0) {
        if (s == 0) return U128{m, 0ull};
        if (s < 64) return U128{m << s, m >> (64 - s)};
        return U128{0ull, m << (s - 64)};         // s < 128 by the bound above
    }
    int r = -s;
    if (r >= 54) return u128_zero();              // m < 2^53 <= half of 2^r
    unsigned long long q = m >> r;
    unsigned long long rem = m & ((1ull << r) - 1ull);
    unsigned long long half = 1ull << (r - 1);
    if (rem > half || (rem == half && (q & 1ull))) q++;
    return U128{q, 0ull};
}

// correctly rounded (round-to-nearest-even) conversion of v * 2^-64 to fp64
__device__ __forceinline__ double fx_to_double(U128 v) {
    if (v.hi == 0ull) return __ull2double_rn(v.lo) * 0x1p-64;
    int lz = __clzll(v.hi);                       // 0..63
    unsigned long long top, rest;
    if (lz == 0) { top = v.hi; rest = v.lo; }
    else { top = (v.hi << lz) | (v.lo >> (64 - lz)); rest = v.lo << lz; }
    if (rest) top |= 1ull;                        // sticky bit below the rounding point
    // v = top * 2^(64 - lz) (up to the sticky bit), times 2^-64
    return __ull2double_rn(top) * __longlong_as_double((long long)(1023 - lz) << 52);   // * 2^-lz, exact
}

// Type-I accumulators are three 64-bit limbs per head updated with
// fire-and-forget RED (no carries between limbs): limb0 += bits[0,32),
// limb1 += bits[32,64), limb2 += bits[64,128). Exact while a head receives
// fewer than 2^32 terms.
__device__ __forceinline__ void fx_red3(unsigned long long *acc3, U128 q) {
    atomicAdd(acc3 + 0, q.lo & 0xFFFFFFFFull);
    atomicAdd(acc3 + 1, q.lo >> 32);
    if (q.hi) atomicAdd(acc3 + 2, q.hi);
}
__device__ __forceinline__ U128 fx_from3(const unsigned long long *acc3) {
    unsigned long long l0 = acc3[0], l1 = acc3[1], l2 = acc3[2];
    U128 a{l0, l2};
    U128 b{l1 << 32, l1 >> 32};
    return u128_add(a, b);
}

// Two-limb variant for the Type-I scatter: limb0 += bits[0,32), limb1 +=
// bits[32,96). Exact while a head receives < 2^32 terms and its unnormalised
// Type-I sum stays below 2^32 (limb1 then never wraps): both hold for any
// graph with d_max < 2^16 since every grouped term is < 2 * 2^11.
__device__ __forceinline__ void fx_red2(unsigned long long *acc2, U128 q) {
    atomicAdd(acc2 + 0, q.lo & 0xFFFFFFFFull);
    atomicAdd(acc2 + 1, (q.lo >> 32) | (q.hi << 32));
}
__device__ __forceinline__ U128 fx_from2(const unsigned long long *acc2) {
    unsigned long long l0 = acc2[0], l1 = acc2[1];
    return u128_add(U128{l0, 0ull}, U128{l1 << 32, l1 >> 32});
}

// w^(1/3) for the weights (finite w > 0, inside fp32's normal range): an fp32
// reciprocal cube root refined by two Newton steps in fp64 (r <- r (4 - w r^3)
// / 3; the relative error goes 2^-22 -> 2^-43 -> below fp64 rounding), then
// w r^2. Within a few ulps of the correctly rounded root and a fixed sequence
// of operations (deterministic: structural ties stay exact); several times
// cheaper than the libm-style cbrt, which was a quarter of Phase A's time.
__device__ __forceinline__ double cube_root(double w) {
#ifdef RS_EXP_LIBCBRT
    return cbrt(w);
#else
    double r = (double)rcbrtf((float)w);
    r = r * fma(-w * r, r * r, 4.0) * (1.0 / 3.0);
    r = r * fma(-w * r, r * r, 4.0) * (1.0 / 3.0);
    return w * r * r;
#endif
}

// B-table grid (BQL): round-to-nearest of a * 2^q as an integer (a >= 0, the
// scaling by a power of two is exact), and back
__device__ __forceinline__ unsigned long long bq_quantize(double a, int q) {
    return __double2ull_rn(a * __longlong_as_double((long long)(1023 + q) << 52));
}
__device__ __forceinline__ double bq_to_double(unsigned long long v, int q) {
    return __ull2double_rn(v) * __longlong_as_double((long long)(1023 - q) << 52);
}

// ---------------------------------------------------------------------------
// Vertex groups. A group of G lanes (G in {4, 8, 16, 32}) owns one vertex and
// walks its adjacency G entries per step; 32/G groups share a warp. Lanes of
// one group always execute the same trip count, so group-masked shuffles are
// well defined even when the groups of a warp diverge.
// ---------------------------------------------------------------------------
template <int G>
struct WarpGroup {
    static constexpr int size = G;
    unsigned lane;   // 0..G-1
    unsigned shift;  // first lane of the group in the warp
    unsigned gmask;  // the group's lanes
    __device__ __forceinline__ WarpGroup() {
        unsigned l = threadIdx.x & 31u;
        lane = l & (G - 1);
        shift = l & ~(unsigned)(G - 1);
        gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << shift);
    }
    __device__ __forceinline__ void sync() const { __syncwarp(gmask); }
    // exclusive rank of this lane among lanes with p set; total in *tot
    __device__ __forceinline__ int rank(bool p, int *tot) const {
        unsigned b = __ballot_sync(gmask, p) & gmask;
        b >>= shift;
        *tot = __popc(b);
        return __popc(b & ((1u << lane) - 1u));
    }
    // number of lanes of the group with p set
    __device__ __forceinline__ int count(bool p) const {
        return __popc(__ballot_sync(gmask, p) & gmask);
    }
    // U independent ranks (one per unrolled slot); warps need no batching
    template <int U>
    __device__ __forceinline__ void rank_u(const bool (&p)[U], int (&r)[U], int (&tot)[U]) {
#pragma unroll
        for (int j = 0; j < U; j++) r[j] = rank(p[j], &tot[j]);
    }
    template <class T>
    __device__ __forceinline__ T sum(T v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o, G);
        return v;
    }
    __device__ __forceinline__ U128 sum(U128 v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            U128 w{__shfl_xor_sync(gmask, v.lo, o, G), __shfl_xor_sync(gmask, v.hi, o, G)};
            v = u128_add(v, w);
        }
        return v;
    }
    template <class T>
    __device__ __forceinline__ T bcast(T v, int src) const {
        return __shfl_sync(gmask, v, src, G);
    }
};

// Lockstep vertex groups: like WarpGroup, but every lane of the warp executes
// every step together (loop bounds are the warp maximum, a group with a shorter
// row or no vertex just has its lanes masked by predicates), so collectives use
// the full warp mask and groups never diverge. Round 1's profile of the 8-lane
// classes: the groups of a warp, at different iterations of their own loops,
// were serialised -- the ballots alone were 22% of the instructions.
template <int G>
struct LockGroup {
    static constexpr int size = G;
    unsigned lane;   // 0..G-1
    unsigned shift;  // first lane of the group in the warp
    __device__ __forceinline__ LockGroup() {
        const unsigned l = threadIdx.x & 31u;
        lane = l & (G - 1);
        shift = l & ~(unsigned)(G - 1);
    }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    // warp-uniform loop bound: the largest v over the warp's groups
    __device__ __forceinline__ int umax(int v) const { return (int)__reduce_max_sync(0xffffffffu, (unsigned)v); }
    __device__ __forceinline__ unsigned bits(bool p) const {
        const unsigned b = __ballot_sync(0xffffffffu, p);
        return G == 32 ? b : (b >> shift) & ((1u << G) - 1u);
    }
    __device__ __forceinline__ int rank(bool p, int *tot) const {
        const unsigned b = bits(p);
        *tot = __popc(b);
        return __popc(b & ((1u << lane) - 1u));
    }
    __device__ __forceinline__ int count(bool p) const { return __popc(bits(p)); }
    template <int U>
    __device__ __forceinline__ void rank_u(const bool (&p)[U], int (&r)[U], int (&tot)[U]) const {
#pragma unroll
        for (int j = 0; j < U; j++) r[j] = rank(p[j], &tot[j]);
    }
    template <class T>
    __device__ __forceinline__ T sum(T v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
        return v;
    }
    __device__ __forceinline__ U128 sum(U128 v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            U128 w{__shfl_xor_sync(0xffffffffu, v.lo, o, G), __shfl_xor_sync(0xffffffffu, v.hi, o, G)};
            v = u128_add(v, w);
        }
        return v;
    }
    // v of the group's lane src (src may differ per lane)
    template <class T>
    __device__ __forceinline__ T from(T v, int src) const { return __shfl_sync(0xffffffffu, v, (int)shift + src); }
};

// A whole CTA (blockDim.x == kCtaThreads) owning one vertex (degree hubs).
constexpr int kCtaThreads = 256;
constexpr int kCtaWarps = kCtaThreads / 32;

struct CtaGroup {
    static constexpr int size = kCtaThreads;
    unsigned lane;
    int *s_i;            // kCtaWarps + 1 ints of shared scratch
    unsigned long long *s_u;  // 2 * kCtaWarps u64 of shared scratch
    __device__ __forceinline__ CtaGroup(int *si, unsigned long long *su) : lane(threadIdx.x), s_i(si), s_u(su) {}
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ int rank(bool p, int *tot) {
        unsigned b = __ballot_sync(0xffffffffu, p);
        int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) s_i[w] = __popc(b);
        __syncthreads();
        int before = 0, all = 0;
#pragma unroll
        for (int i = 0; i < kCtaWarps; i++) { int c = s_i[i]; before += (i < w) ? c : 0; all += c; }
        __syncthreads();
        *tot = all;
        return before + __popc(b & ((1u << l) - 1u));
    }
    __device__ __forceinline__ int count(bool p) {
        int tot;
        rank(p, &tot);
        return tot;
    }
    __device__ __forceinline__ int umax(int v) const { return v; }   // one vertex per CTA: uniform already
    __device__ __forceinline__ double bcast(double v, int src) {
        if ((int)threadIdx.x == src) s_u[0] = (unsigned long long)__double_as_longlong(v);
        __syncthreads();
        const double r = __longlong_as_double((long long)s_u[0]);
        __syncthreads();
        return r;
    }
    // U ranks with ONE pair of barriers (the warp counts of all U slots go to
    // shared memory together): slot j's order is warp-major, as rank()'s
    template <int U>
    __device__ __forceinline__ void rank_u(const bool (&p)[U], int (&r)[U], int (&tot)[U]) {
        static_assert(U * kCtaWarps <= 4 * kCtaWarps, "shared scratch holds 4 slots");
        int *cnt = reinterpret_cast<int *>(s_u);   // 2 * kCtaWarps u64 = U * kCtaWarps ints for U <= 4
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        unsigned b[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            b[j] = __ballot_sync(0xffffffffu, p[j]);
            if (l == 0) cnt[j * kCtaWarps + w] = __popc(b[j]);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < U; j++) {
            int before = 0, all = 0;
#pragma unroll
            for (int i = 0; i < kCtaWarps; i++) { const int c = cnt[j * kCtaWarps + i]; before += (i < w) ? c : 0; all += c; }
            tot[j] = all;
            r[j] = before + __popc(b[j] & ((1u << l) - 1u));
        }
        __syncthreads();
    }
    __device__ __forceinline__ long long sum(long long v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) s_u[w] = (unsigned long long)v;
        __syncthreads();
        long long a = 0;
#pragma unroll
        for (int i = 0; i < kCtaWarps; i++) a += (long long)s_u[i];
        __syncthreads();
        return a;
    }
    __device__ __forceinline__ int sum(int v) { return (int)sum((long long)v); }
    __device__ __forceinline__ double sum(double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) s_u[w] = (unsigned long long)__double_as_longlong(v);
        __syncthreads();
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < kCtaWarps; i++) a += __longlong_as_double((long long)s_u[i]);
        __syncthreads();
        return a;
    }
    __device__ __forceinline__ unsigned long long sum(unsigned long long v) {
        return (unsigned long long)sum((long long)v);
    }
    __device__ __forceinline__ U128 sum(U128 v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            U128 w{__shfl_xor_sync(0xffffffffu, v.lo, o), __shfl_xor_sync(0xffffffffu, v.hi, o)};
            v = u128_add(v, w);
        }
        int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) { s_u[2 * w] = v.lo; s_u[2 * w + 1] = v.hi; }
        __syncthreads();
        U128 a = u128_zero();
#pragma unroll
        for (int i = 0; i < kCtaWarps; i++) a = u128_add(a, U128{s_u[2 * i], s_u[2 * i + 1]});
        __syncthreads();
        return a;
    }
};

__device__ __forceinline__ double atomic_max_nonneg(unsigned long long *addr, double v) {
    // non-negative IEEE doubles order like their bit patterns
    return __longlong_as_double((long long)atomicMax(addr, (unsigned long long)__double_as_longlong(v)));
}

}  // namespace rs
