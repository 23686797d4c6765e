// Host edge list -> HBM (the drop-in from_edge_array's host input path).
// Reference: C/graph.py:114-122 takes an (m, 2) numpy array -- int64 and in
// ordinary pageable memory for any caller of the reference API.
//
// A pageable cudaMemcpy is staged by the driver at a fraction of the link
// rate, and int64 ids double the bytes on the link.  Instead the ids are
// narrowed to int32 on the host (range-checked: [0, 2^31)) by a persistent
// pool of worker threads straight into page-locked staging buffers, and each
// buffer goes to the device with cudaMemcpyAsync as soon as it is full:
// the conversion of chunk i+1 overlaps the DMA of chunk i (NB buffers in
// flight, reused once their copy event completed).  The link then carries
// 8 B per edge at full rate.  No reference counterpart beyond the call.
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <immintrin.h>
#include <mutex>
#include <thread>

#include "common.cuh"

namespace cvz {
namespace {

// ---- a minimal persistent fork-join pool --------------------------------
class Pool {
   public:
    static Pool &get() {
        static Pool p;
        return p;
    }
    int size() const { return (int)workers_.size() + 1; }
    // fn(t, T) on T = size() threads (the caller is thread 0); blocks
    void run(const std::function<void(int, int)> &fn) {
        const int T = size();
        {
            std::unique_lock<std::mutex> lk(mu_);
            fn_ = &fn;
            pending_ = T - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0, T);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

   private:
    Pool() {
        unsigned hc = std::thread::hardware_concurrency();
        int T = (int)std::max(1u, std::min(hc ? hc : 1u, 32u));
        for (int t = 1; t < T; ++t) workers_.emplace_back([this, t] { loop(t); });
    }
    ~Pool() {
        {
            std::unique_lock<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &w : workers_) w.join();
    }
    void loop(int t) {
        unsigned long long seen = 0;
        while (true) {
            const std::function<void(int, int)> *fn;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                fn = fn_;
            }
            (*fn)(t, size());
            std::unique_lock<std::mutex> lk(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int, int)> *fn_ = nullptr;
    int pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

constexpr int NB = 3;                             // staging buffers in flight
constexpr long long CHUNK_PAIRS = 4LL << 20;      // 4M edges = 32 MB of int32 pairs

struct Staging {
    int32_t *buf[NB] = {};
    cudaEvent_t ev[NB] = {};
    bool ready = false;
};
std::mutex g_stage_mu;
Staging g_stage[DeviceCache::kMax];

Staging &staging() {
    const int d = current_device();
    CVZ_REQUIRE(d >= 0 && d < DeviceCache::kMax, CVZ_ERR_VALUE, "device id out of range");
    Staging &st = g_stage[d];
    if (!st.ready) {
        for (int b = 0; b < NB; ++b) {
            CVZ_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&st.buf[b]),
                                   CHUNK_PAIRS * 2 * sizeof(int32_t), cudaHostAllocPortable));
            CVZ_CUDA(cudaEventCreateWithFlags(&st.ev[b], cudaEventDisableTiming));
        }
        st.ready = true;
    }
    return st;
}

// int64 ids -> int32 with non-temporal 16-byte stores (no read-for-
// ownership of the staging lines: the copy is host-memory-bound); returns
// true if any id lies outside [0, 2^31).  dst is 16-byte aligned.
bool narrow64(const int64_t *src, int32_t *dst, long long k) {
    __m128i acc = _mm_setzero_si128();
    long long i = 0;
    for (; i + 4 <= k; i += 4) {
        const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i));
        const __m128i y = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i + 2));
        acc = _mm_or_si128(acc, _mm_or_si128(x, y));
        const __m128 lo = _mm_shuffle_ps(_mm_castsi128_ps(x), _mm_castsi128_ps(y),
                                         _MM_SHUFFLE(2, 0, 2, 0));
        _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i), _mm_castps_si128(lo));
    }
    alignas(16) uint64_t w[2];
    _mm_store_si128(reinterpret_cast<__m128i *>(w), acc);
    uint64_t orr = w[0] | w[1];
    for (; i < k; ++i) {
        orr |= (uint64_t)src[i];
        dst[i] = (int32_t)src[i];
    }
    _mm_sfence();
    return (orr >> 31) != 0;
}

// int32 ids: streaming copy + sign check
bool narrow32(const int32_t *src, int32_t *dst, long long k) {
    __m128i acc = _mm_setzero_si128();
    long long i = 0;
    for (; i + 4 <= k; i += 4) {
        const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i));
        acc = _mm_or_si128(acc, x);
        _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i), x);
    }
    int orr = _mm_movemask_ps(_mm_castsi128_ps(acc));  // sign bits
    for (; i < k; ++i) {
        orr |= src[i] < 0;
        dst[i] = src[i];
    }
    _mm_sfence();
    return orr != 0;
}

}  // namespace
}  // namespace cvz

using namespace cvz;

extern "C" int cvz_edges_upload(const void *host_edges, int in_is_int32, int64_t m,
                                int32_t *dev_out, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(m >= 0, CVZ_ERR_VALUE, "negative edge count");
        if (m == 0) return;
        cudaStream_t s = as_stream(stream);
        std::lock_guard<std::mutex> lk(g_stage_mu);  // the staging ring is per device, shared
        Staging &st = staging();
        Pool &pool = Pool::get();
        const long long vals = 2 * m;
        const long long chunk_vals = 2 * CHUNK_PAIRS;
        const long long chunks = (vals + chunk_vals - 1) / chunk_vals;
        std::atomic<int> bad{0};
        for (long long c = 0; c < chunks; ++c) {
            const int b = (int)(c % NB);
            const long long lo = c * chunk_vals;
            const long long cnt = std::min(chunk_vals, vals - lo);
            CVZ_CUDA(cudaEventSynchronize(st.ev[b]));  // buffer b's previous copy is done
            int32_t *dst = st.buf[b];
            pool.run([&](int t, int T) {
                // slices of whole 16-byte groups (4 ids) so streaming stores align
                const long long g = (cnt + 3) / 4;
                const long long a = lo + 4 * (g * t / T), e = std::min(lo + 4 * (g * (t + 1) / T),
                                                                       lo + cnt);
                if (e <= a) return;
                bool b = in_is_int32 ? narrow32(static_cast<const int32_t *>(host_edges) + a,
                                                dst + (a - lo), e - a)
                                     : narrow64(static_cast<const int64_t *>(host_edges) + a,
                                                dst + (a - lo), e - a);
                if (b) bad.store(1, std::memory_order_relaxed);
            });
            CVZ_CUDA(cudaMemcpyAsync(dev_out + lo, dst, (size_t)cnt * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, s));
            CVZ_CUDA(cudaEventRecord(st.ev[b], s));
        }
        // the staging buffers are reused by the next call: it waits on their
        // events; the caller's stream orders the data for the kernels
        CVZ_REQUIRE(!bad.load(), CVZ_ERR_RANGE, "node ids must lie in [0, 2^31)");
    });
}
