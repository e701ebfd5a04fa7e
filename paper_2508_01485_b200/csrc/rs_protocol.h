// Multi-GPU host protocol shared by the device code and the exported host
// functions (include/rs.h, "Multi-GPU host protocol"): one definition of the
// range split, so that what the gloo tests exercise is what the GPU runs.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define RS_HD __host__ __device__ __forceinline__
#else
#define RS_HD inline
#endif

namespace rs {

// boundary r (0 < r < world) of the balanced split of an inclusive work prefix:
// the first vertex after the prefix reaches ceil(total * r / world)
RS_HD int64_t split_point(const int64_t *incl, int64_t n, int world, int r) {
    if (r <= 0 || n <= 0) return 0;
    if (r >= world) return n;
    const int64_t total = incl[n - 1];
    const int64_t target = (total * r + world - 1) / world;
    int64_t lo = 0, hi = n;   // first u with incl[u] >= target
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (incl[mid] < target) lo = mid + 1; else hi = mid;
    }
    return lo + 1 < n ? lo + 1 : n;
}

// the Step 4 order key of a non-negative score: its IEEE bits, -0.0 folded to
// +0.0 (monotone as an unsigned integer)
RS_HD uint64_t score_key_bits(uint64_t bits) { return bits == 0x8000000000000000ull ? 0ull : bits; }

// the candidate order of Step 4: key descending, id ascending
RS_HD bool cand_before(uint64_t ka, int32_t ia, uint64_t kb, int32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}

}  // namespace rs
