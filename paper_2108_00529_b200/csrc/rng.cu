// numpy's PCG64 stream on the device, bit-exact (host RNG parity, SURVEY.md
// 7.3 #5).  C/layout.py:78-82 init_positions draws
//   default_rng(seed).uniform(-s/2, s/2, (n, 2))
// i.e. value_i = low + range * next_double(), next_double = (next_u64 >> 11)
// * 2^-53, next_u64 = XSL-RR output of the 128-bit LCG state after one step
// (numpy/random/src/pcg64: pcg_setseq_128_xsl_rr_64_random_r).  The host
// seeds the generator with numpy (SeedSequence) and passes the 128-bit state
// and increment; each thread jumps ahead to its chunk in O(log i) (LCG
// composition) and steps sequentially, so the n*2 draws fill HBM in one
// launch instead of a host loop + copy.
#include "common.cuh"

namespace cvz {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
    return ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
}

__device__ __forceinline__ unsigned long long xsl_rr(u128 s) {
    unsigned long long x = (unsigned long long)(s >> 64) ^ (unsigned long long)s;
    unsigned r = (unsigned)(s >> 122);
    return (x >> r) | (x << ((64u - r) & 63u));
}

// state after k LCG steps
__device__ u128 pcg_advance(u128 s, u128 inc, unsigned long long k) {
    u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
    while (k) {
        if (k & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        k >>= 1;
    }
    return am * s + ap;
}

constexpr int CHUNK = 16;

__global__ void pcg64_uniform_kernel(unsigned long long shi, unsigned long long slo,
                                     unsigned long long ihi, unsigned long long ilo, double low,
                                     double range, long long count, double *__restrict__ out) {
    const u128 inc = ((u128)ihi << 64) | ilo;
    const u128 M = pcg_mult();
    for (long long c0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * CHUNK; c0 < count;
         c0 += (long long)gridDim.x * blockDim.x * CHUNK) {
        u128 s = pcg_advance(((u128)shi << 64) | slo, inc, (unsigned long long)c0);
        const long long end = min(count, c0 + CHUNK);
        for (long long i = c0; i < end; ++i) {
            s = s * M + inc;
            double u = (double)(xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
            out[i] = __dadd_rn(low, __dmul_rn(range, u));
        }
    }
}

}  // namespace
}  // namespace cvz

using namespace cvz;

extern "C" int cvz_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                 uint64_t inc_lo, double low, double range, int64_t count,
                                 double *out, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(count >= 0, CVZ_ERR_VALUE, "count must be non-negative");
        if (count == 0) return;
        cudaStream_t s = as_stream(stream);
        CVZ_LAUNCH(pcg64_uniform_kernel, grid_for((count + CHUNK - 1) / CHUNK, 256, 1, 8), 256, 0,
                   s, (unsigned long long)state_hi, (unsigned long long)state_lo,
                   (unsigned long long)inc_hi, (unsigned long long)inc_lo, low, range,
                   (long long)count, out);
    });
}
