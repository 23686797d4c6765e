// Device peak probes for bench.py's roofline denominators that
// MEASURED_PEAKS.json does not carry (it has HBM copy bandwidth and bf16
// tensor throughput only).  Measurement only: nothing on the hot path calls
// these.  No reference counterpart.
//
// FP64: the Barnes-Hut walk is a per-thread fp64 chain, so its compute
// roofline is the FP64 FMA pipe.  The probe runs 8 independent DFMA chains per
// thread on every SM (full occupancy) and times them with CUDA events.
#include "common.cuh"

namespace cvz {
namespace {

constexpr int CHAINS = 8;

__global__ void __launch_bounds__(256) dfma_probe_kernel(double seed, int iters,
                                                        double *__restrict__ sink) {
    double a[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
    const double m = 0.999999999, b = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) a[c] = fma(a[c], m, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += a[c];
    if (s == 12345.678) sink[threadIdx.x] = s;  // never true; keeps the chains live
}

}  // namespace
}  // namespace cvz

using namespace cvz;

extern "C" int cvz_probe_fp64(double *gflops, void *stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        double *sink = sc.alloc<double>(256);
        int per_sm = 0;
        CVZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dfma_probe_kernel, 256, 0));
        const unsigned grid = (unsigned)(num_sms() * (per_sm > 0 ? per_sm : 1));
        const int iters = 4096;
        cudaEvent_t a, b;
        CVZ_CUDA(cudaEventCreate(&a));
        CVZ_CUDA(cudaEventCreate(&b));
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {  // rep 0 warms up
            CVZ_CUDA(cudaEventRecord(a, s));
            CVZ_LAUNCH(dfma_probe_kernel, grid, 256, 0, s, 1.0, iters, sink);
            CVZ_CUDA(cudaEventRecord(b, s));
            CVZ_CUDA(cudaEventSynchronize(b));
            float ms = 0;
            CVZ_CUDA(cudaEventElapsedTime(&ms, a, b));
            if (rep > 0 && ms < best) best = ms;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        const double flops = 2.0 * CHAINS * (double)iters * grid * 256.0;
        *gflops = flops / (best * 1e-3) / 1e9;
    });
}
