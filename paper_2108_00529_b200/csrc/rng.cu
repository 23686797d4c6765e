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

namespace cvz {
namespace {

// Counter-based R-MAT (BASELINE config C5: scale 26, edge factor 16,
// (a, b, c, d) = (0.57, 0.19, 0.19, 0.05)).  Draw l of edge k
// is a function of (seed, k, l) only -- splitmix64 of seed * phi + k * 64 +
// l, top 53 bits as a uniform double -- so every rank generates its own
// slice of the stream, bit-identical for any number of ranks, and
// synth.rmat_counter (numpy) reproduces it on the host for the tests.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void rmat_kernel(int scale, double a, double ab, double abc,
                            unsigned long long seed, long long start, long long count,
                            int2 *__restrict__ out) {
    const unsigned long long base = seed * 0x9E3779B97F4A7C15ull;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < count;
         j += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = (unsigned long long)(start + j);
        unsigned u = 0, v = 0;
        for (int l = 0; l < scale; ++l) {
            double r = (double)(splitmix64(base + k * 64ull + (unsigned long long)l) >> 11) *
                       0x1.0p-53;
            unsigned ub = r >= ab;
            unsigned vb = (r >= a && r < ab) || r >= abc;
            u = (u << 1) | ub;
            v = (v << 1) | vb;
        }
        out[j] = make_int2((int)u, (int)v);
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

extern "C" int cvz_rmat_edges(int scale, double a, double b, double c, uint64_t seed,
                              int64_t start, int64_t count, int32_t *edges_out, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(scale >= 1 && scale <= 30, CVZ_ERR_VALUE, "R-MAT scale must be in [1, 30]");
        CVZ_REQUIRE(start >= 0 && count >= 0, CVZ_ERR_VALUE, "bad edge range");
        if (count == 0) return;
        CVZ_LAUNCH(rmat_kernel, grid_for(count, 256, 1, 16), 256, 0, as_stream(stream), scale, a,
                   a + b, a + b + c, (unsigned long long)seed, (long long)start, (long long)count,
                   reinterpret_cast<int2 *>(edges_out));
    });
}
