// Graph ingestion: stable self-loop compaction, degree histogram, degree stats.
// Reference: C/graph.py:114-136 (from_edge_array, degree_stats).
//
// HBM-bound streaming kernels.  Edges are read as 128-bit vectors (one int64
// pair or two int32 pairs per load), each CTA owns a contiguous tile so the
// compaction stays stable, and the tile offset comes from a single-pass
// decoupled look-back (no second pass over the edges).
#include <cub/cub.cuh>

#include <map>
#include <mutex>
#include <sstream>

#include <cstring>

#include "common.cuh"

namespace cvz {

std::atomic<long long> g_launches{0};
static thread_local std::string t_last_error;
void set_last_error(const std::string &m) { t_last_error = m; }

// ---- kernel profiler ---------------------------------------------------------
namespace {
struct ProfRec {
    const char *name;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof{false};
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;
std::string g_prof_report;
}  // namespace

bool prof_on() { return g_prof.load(std::memory_order_relaxed); }

cudaEvent_t prof_event() {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t e;
    if (!g_prof_pool.empty()) {
        e = g_prof_pool.back();
        g_prof_pool.pop_back();
    } else {
        cudaEventCreate(&e);
    }
    return e;
}

void prof_record(const char *name, cudaEvent_t a, cudaEvent_t b) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_recs.push_back(ProfRec{name, a, b});
}

void init_pool_once() {  // per device: the release threshold is a pool attribute
    static DeviceCache done;
    done.get([] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, current_device()) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        return 1;
    });
}

namespace {
__global__ void read_small_kernel(const unsigned char *__restrict__ src,
                                  volatile unsigned char *__restrict__ dst, int bytes) {
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

void read_small(void *host, const void *dev, size_t bytes, cudaStream_t s) {
    constexpr size_t kSlot = 256;
    CVZ_REQUIRE(bytes <= kSlot, CVZ_ERR_VALUE, "read_small: at most 256 bytes");
    // one mapped pinned slot per host thread (portable: any device can
    // write it through UVA); the synchronise below serialises its reuse
    static thread_local unsigned char *slot = nullptr;
    if (!slot) {
        void *p = nullptr;
        CVZ_CUDA(cudaHostAlloc(&p, kSlot, cudaHostAllocMapped | cudaHostAllocPortable));
        slot = static_cast<unsigned char *>(p);
    }
    if (bytes == 0) return;
    CVZ_LAUNCH(read_small_kernel, 1, 32, 0, s, static_cast<const unsigned char *>(dev), slot,
               (int)bytes);
    CVZ_CUDA(cudaStreamSynchronize(s));
    std::memcpy(host, slot, bytes);
}

namespace {

constexpr int CBLOCK = 256;
constexpr int CITEMS = 8;  // edges per thread
constexpr int CTILE = CBLOCK * CITEMS;

template <bool IN32>
__global__ void __launch_bounds__(CBLOCK) compact_edges_kernel(
    const void *__restrict__ in, long long m, int2 *__restrict__ out, LookbackState st,
    unsigned long long *__restrict__ d_count, long long *__restrict__ d_max,
    int *__restrict__ d_bad, unsigned num_tiles) {
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_prefix;
    __shared__ int s_warp[CBLOCK / 32];
    __shared__ long long s_max[CBLOCK / 32];
    const unsigned tile = acquire_tile(st, &s_tile);
    const long long base = (long long)tile * CTILE;

    int2 e[CITEMS];
    bool keep[CITEMS];
    int cnt = 0;
    long long mx = -1;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < CITEMS; ++j) {
        long long i = base + (long long)j * CBLOCK + threadIdx.x;  // coalesced
        keep[j] = false;
        if (i < m) {
            long long u, v;
            if (IN32) {
                int2 p = __ldg(reinterpret_cast<const int2 *>(in) + i);
                u = p.x;
                v = p.y;
            } else {
                longlong2 p = __ldg(reinterpret_cast<const longlong2 *>(in) + i);  // 128-bit
                u = p.x;
                v = p.y;
            }
            bad |= (u < 0) | (v < 0) | (u > 0x7fffffffLL) | (v > 0x7fffffffLL);
            e[j] = make_int2((int)u, (int)v);
            keep[j] = (u != v);
            if (keep[j]) {
                cnt++;
                mx = max(mx, max(u, v));
            }
        }
    }
    // warp ballots -> per (item, warp) counts -> one scan by warp 0: two
    // block barriers per tile instead of one block scan per item slot
    constexpr int NW = CBLOCK / 32;
    __shared__ unsigned s_cnt[CITEMS * NW];
    __shared__ unsigned s_total;
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned bal[CITEMS];
#pragma unroll
    for (int j = 0; j < CITEMS; ++j) {
        bal[j] = __ballot_sync(0xffffffffu, keep[j]);
        if (lane == 0) s_cnt[j * NW + wid] = __popc(bal[j]);
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the CITEMS * NW counts, PER per lane
        constexpr int PER = CITEMS * NW / 32;
        static_assert(PER * 32 == CITEMS * NW, "scan layout");
        unsigned a[PER], v = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            a[q] = s_cnt[PER * lane + q];
            v += a[q];
        }
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        unsigned r = x - v;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            s_cnt[PER * lane + q] = r;
            r += a[q];
        }
        if (lane == 31) s_total = x;
    }
    __syncthreads();
    const unsigned total = s_total;
    (void)cnt;
    (void)s_warp;
    unsigned long long prefix = tile_prefix(st, tile, (unsigned long long)total, &s_prefix);
    const unsigned lt = (1u << lane) - 1;
#pragma unroll
    for (int j = 0; j < CITEMS; ++j)
        if (keep[j]) out[prefix + s_cnt[j * NW + wid] + __popc(bal[j] & lt)] = e[j];
    // max + range flag
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane_id() == 0) s_max[threadIdx.x >> 5] = mx;
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        long long b = -1;
        for (int w = 0; w < CBLOCK / 32; ++w) b = max(b, s_max[w]);
        if (b >= 0) atomicMax(reinterpret_cast<unsigned long long *>(d_max), (unsigned long long)b);
        if (bad) atomicExch(d_bad, 1);
        if (tile == num_tiles - 1) *d_count = prefix + total;
    }
}

// degree[x] += endpoint count.  64-bit RED into an L2-resident n-array.
__global__ void degree_kernel(const int4 *__restrict__ e2, long long npairs2,
                              const int2 *__restrict__ e, long long m,
                              unsigned long long *__restrict__ deg) {
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < npairs2;
         i += stride) {
        int4 p = __ldg(e2 + i);  // two edges per 128-bit load
        atomicAdd(deg + p.x, 1ull);
        atomicAdd(deg + p.y, 1ull);
        atomicAdd(deg + p.z, 1ull);
        atomicAdd(deg + p.w, 1ull);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (m & 1)) {
        int2 p = e[m - 1];
        atomicAdd(deg + p.x, 1ull);
        atomicAdd(deg + p.y, 1ull);
    }
}

// Single pass with the lowest HOT node ids counted in shared memory first
// (R-MAT and most generators put the hubs at low ids; same-address L2
// atomics on a hub serialise): CVZ_DEGREE_HOT experiment.
constexpr int HOT = 2048;
template <class C>  // counter type: u64 (the output) or u32 scratch
__global__ void degree_hot_kernel(const int4 *__restrict__ e2, long long npairs2,
                                  const int2 *__restrict__ e, long long m, C *__restrict__ deg) {
    __shared__ unsigned sh[HOT];
    for (int i = threadIdx.x; i < HOT; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    long long stride = (long long)gridDim.x * blockDim.x;
    auto add = [&](int x) {
        if (x < HOT)
            atomicAdd(sh + x, 1u);
        else
            atomicAdd(deg + x, (C)1);
    };
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < npairs2;
         i += stride) {
        const int4 p = __ldcs(e2 + i);
        add(p.x);
        add(p.y);
        add(p.z);
        add(p.w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (m & 1)) {
        const int2 p = e[m - 1];
        add(p.x);
        add(p.y);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HOT; i += blockDim.x)
        if (sh[i]) atomicAdd(deg + i, (C)sh[i]);
}

__global__ void widen_counts_kernel(const unsigned *__restrict__ cnt, long long n,
                                    long long *__restrict__ deg) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        deg[i] = cnt[i];
}

// sum / max / histogram of nonzero degrees (mode).
__global__ void degree_summary_kernel(const long long *__restrict__ deg, long long n,
                                      unsigned long long *__restrict__ sum,
                                      unsigned long long *__restrict__ mx) {
    unsigned long long s = 0, m = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned long long d = (unsigned long long)deg[i];
        s += d;
        m = max(m, d);
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if (lane_id() == 0) {
        atomicAdd(sum, s);
        atomicMax(mx, m);
    }
}

constexpr int SMEM_BINS = 4096;
__global__ void degree_hist_kernel(const long long *__restrict__ deg, long long n,
                                   unsigned int *__restrict__ hist, long long nbins) {
    __shared__ unsigned int sh[SMEM_BINS];
    for (int i = threadIdx.x; i < SMEM_BINS; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        long long d = deg[i];
        if (d > 0) {
            if (d < SMEM_BINS)
                atomicAdd(&sh[d], 1u);
            else
                atomicAdd(&hist[d], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SMEM_BINS && i < nbins; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// argmax over the histogram, ties -> smallest degree (np.argmax semantics).
__global__ void hist_argmax_kernel(const unsigned int *__restrict__ hist, long long nbins,
                                   unsigned long long *__restrict__ best) {
    unsigned long long b = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nbins;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned long long key = ((unsigned long long)hist[i] << 32) |
                                 (0xffffffffull - (unsigned long long)i);
        b = max(b, key);
    }
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (lane_id() == 0) atomicMax(best, b);
}

__global__ void stats_finalize_kernel(const unsigned long long *__restrict__ sum,
                                      const unsigned long long *__restrict__ mx,
                                      const unsigned long long *__restrict__ best,
                                      long long *__restrict__ out3) {
    unsigned long long b = *best;
    long long mode = (b >> 32) ? (long long)(0xffffffffull - (b & 0xffffffffull)) : 0;
    out3[0] = mode;
    out3[1] = (long long)*sum;
    out3[2] = (long long)*mx;
}

}  // namespace

void edges_compact(const void *edges, bool in32, int64_t m, int32_t *out, int64_t *d_m_out,
                   int64_t *d_max, int *d_bad, cudaStream_t s) {
    Scratch sc(s);
    unsigned tiles = (unsigned)((m + CTILE - 1) / CTILE);
    if (tiles == 0) tiles = 1;
    auto *status = sc.alloc<unsigned long long>(tiles);
    auto *ctr = sc.alloc<unsigned>(1);
    CVZ_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * tiles, s));
    CVZ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
    CVZ_CUDA(cudaMemsetAsync(d_m_out, 0, sizeof(int64_t), s));
    // max id starts at 0; callers treat *d_m_out == 0 as "no edges, n = 0"
    CVZ_CUDA(cudaMemsetAsync(d_max, 0, sizeof(int64_t), s));
    LookbackState st{status, ctr};
    if (in32)
        CVZ_LAUNCH(compact_edges_kernel<true>, tiles, CBLOCK, 0, s, edges, (long long)m,
                   reinterpret_cast<int2 *>(out), st,
                   reinterpret_cast<unsigned long long *>(d_m_out),
                   reinterpret_cast<long long *>(d_max), d_bad, tiles);
    else
        CVZ_LAUNCH(compact_edges_kernel<false>, tiles, CBLOCK, 0, s, edges, (long long)m,
                   reinterpret_cast<int2 *>(out), st,
                   reinterpret_cast<unsigned long long *>(d_m_out),
                   reinterpret_cast<long long *>(d_max), d_bad, tiles);
}

void degree_count(const int32_t *edges, int64_t m, int64_t n, int64_t *degree,
                  cudaStream_t s) {
    CVZ_CUDA(cudaMemsetAsync(degree, 0, sizeof(int64_t) * (n ? n : 1), s));
    if (m == 0) return;
    long long pairs2 = m / 2;
    static const bool plain = getenv("CVZ_DEGREE_PLAIN") != nullptr;  // A/B knob
    const unsigned hg = grid_for(pairs2 > 0 ? pairs2 : 1, 256, 1, 16);
    // arrays beyond L2 (> 8M nodes): u32 counters (a degree is < 2m < 2^32)
    // halve the DRAM read-modify-write traffic of the missing atomics,
    // widened afterwards (R-MAT-26: 23.1 -> 18.6 ms + 0.5 ms widen)
    if (!plain && n > (8LL << 20) && m < (1LL << 31)) {
        Scratch sc(s);
        unsigned *cnt = sc.alloc<unsigned>(n);
        CVZ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * n, s));
        CVZ_LAUNCH(degree_hot_kernel<unsigned>, hg, 256, 0, s,
                   reinterpret_cast<const int4 *>(edges), pairs2,
                   reinterpret_cast<const int2 *>(edges), (long long)m, cnt);
        CVZ_LAUNCH(widen_counts_kernel, grid_for(n, 256, 1, 8), 256, 0, s, cnt, (long long)n,
                   reinterpret_cast<long long *>(degree));
        return;
    }
    if (!plain) {
        CVZ_LAUNCH(degree_hot_kernel<unsigned long long>, hg, 256, 0, s,
                   reinterpret_cast<const int4 *>(edges), pairs2,
                   reinterpret_cast<const int2 *>(edges), (long long)m,
                   reinterpret_cast<unsigned long long *>(degree));
        return;
    }
    unsigned grid = grid_for(pairs2 > 0 ? pairs2 : 1, 256, 1, 16);
    CVZ_LAUNCH(degree_kernel, grid, 256, 0, s, reinterpret_cast<const int4 *>(edges), pairs2,
               reinterpret_cast<const int2 *>(edges), (long long)m,
               reinterpret_cast<unsigned long long *>(degree));
}

void degree_stats(const int64_t *degree, int64_t n, int64_t *out3, cudaStream_t s) {
    Scratch sc(s);
    auto *acc = sc.alloc<unsigned long long>(3);  // sum, max, best
    CVZ_CUDA(cudaMemsetAsync(acc, 0, 3 * sizeof(unsigned long long), s));
    unsigned grid = grid_for(n, 256, 4, 4);
    CVZ_LAUNCH(degree_summary_kernel, grid, 256, 0, s, reinterpret_cast<const long long *>(degree),
               (long long)n, acc, acc + 1);
    // bins sized by the max degree: read it back (tiny sync, host API is sync)
    unsigned long long mx = 0;
    read_small(&mx, acc + 1, sizeof(mx), s);
    long long nbins = (long long)mx + 1;
    auto *hist = sc.alloc<unsigned int>(nbins > SMEM_BINS ? nbins : SMEM_BINS);
    CVZ_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned) * (nbins > SMEM_BINS ? nbins : SMEM_BINS), s));
    CVZ_LAUNCH(degree_hist_kernel, grid, 256, 0, s, reinterpret_cast<const long long *>(degree),
               (long long)n, hist, nbins);
    CVZ_LAUNCH(hist_argmax_kernel, grid_for(nbins, 256, 4, 2), 256, 0, s, hist, nbins, acc + 2);
    CVZ_LAUNCH(stats_finalize_kernel, 1, 1, 0, s, acc, acc + 1, acc + 2,
               reinterpret_cast<long long *>(out3));
}

}  // namespace cvz

using namespace cvz;

extern "C" {

int cvz_version(void) { return 1; }
const char *cvz_last_error(void) { return t_last_error.c_str(); }
long long cvz_launch_count(void) { return g_launches.load(); }

int cvz_read_small(void *host, const void *dev, int64_t bytes, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(bytes >= 0 && bytes <= 256, CVZ_ERR_VALUE, "read_small: 0..256 bytes");
        CVZ_REQUIRE(host && (dev || bytes == 0), CVZ_ERR_VALUE, "null pointer");
        read_small(host, dev, (size_t)bytes, as_stream(stream));
    });
}

int cvz_profile_begin(void) {
    return guard([&] {
        {
            std::lock_guard<std::mutex> lk(g_prof_mu);
            for (auto &r : g_prof_recs) {
                g_prof_pool.push_back(r.a);
                g_prof_pool.push_back(r.b);
            }
            g_prof_recs.clear();
        }
        g_prof.store(true);
    });
}

int cvz_profile_end(void) {
    return guard([&] {
        g_prof.store(false);
        CVZ_CUDA(cudaDeviceSynchronize());
        std::lock_guard<std::mutex> lk(g_prof_mu);
        std::map<std::string, std::pair<long long, double>> agg;
        for (auto &r : g_prof_recs) {
            float ms = 0.f;
            CVZ_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            auto &v = agg[r.name];
            v.first += 1;
            v.second += ms;
            g_prof_pool.push_back(r.a);
            g_prof_pool.push_back(r.b);
        }
        g_prof_recs.clear();
        std::ostringstream os;
        os.precision(9);
        for (auto &kv : agg) os << kv.first << "\t" << kv.second.first << "\t" << kv.second.second << "\n";
        g_prof_report = os.str();
    });
}

const char *cvz_profile_report(void) { return g_prof_report.c_str(); }

int cvz_edges_compact(const void *edges, int in_is_int32, int64_t m, int32_t *edges_out,
                      int64_t *d_m_out, int64_t *d_max_id, int check_range, void *stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        int *bad = sc.alloc<int>(1);
        CVZ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
        edges_compact(edges, in_is_int32 != 0, m, edges_out, d_m_out, d_max_id, bad, s);
        if (check_range) {
            int hbad = 0;
            read_small(&hbad, bad, sizeof(int), s);
            CVZ_REQUIRE(!hbad, CVZ_ERR_RANGE, "node ids must lie in [0, 2^31)");
        }
    });
}

int cvz_degree_count(const int32_t *edges, int64_t m, int64_t n, int64_t *degree,
                     void *stream) {
    return guard([&] { degree_count(edges, m, n, degree, as_stream(stream)); });
}

int cvz_degree_stats(const int64_t *degree, int64_t n, int64_t *out3, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n > 0, CVZ_ERR_VALUE, "degree stats need n > 0");
        degree_stats(degree, n, out3, as_stream(stream));
    });
}

}  // extern "C"
