// Shared infrastructure for the commviz-b200 CUDA library (sm_100a).
//
// * status/error plumbing for the C-ABI (cvz_status codes, thread-local msg)
// * stream-ordered scratch allocation (cudaMallocAsync on the caller's stream,
//   pool release threshold raised once so steady-state calls never hit the OS)
// * a single-pass decoupled look-back tile prefix (used by every stable
//   stream compaction on the hot path: self-loop drop, round contraction)
// * launch accounting (cvz_launch_count) for bench.py's gpu_launches claim
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <climits>
#include <cstdlib>
#include <tuple>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cvz_b200.h"

namespace cvz {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &m);
extern std::atomic<long long> g_launches;

#define CVZ_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t _e = (call);                                                    \
        if (_e != cudaSuccess)                                                      \
            throw ::cvz::Error(_e == cudaErrorMemoryAllocation ? CVZ_ERR_OOM        \
                                                               : CVZ_ERR_CUDA,      \
                               std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define CVZ_REQUIRE(cond, code, msg)                 \
    do {                                             \
        if (!(cond)) throw ::cvz::Error(code, msg);  \
    } while (0)

// ---- per-kernel device timing (cvz_profile_begin/end/report) --------------
// While enabled, every CVZ_LAUNCH / CVZ_REGION on a stream that is not being
// captured is bracketed by a pair of CUDA events recorded on the launching
// stream; the report sums the elapsed times per kernel name.  Layout runs
// skip CUDA-graph capture while profiling so their kernels are seen too.
bool prof_on();
void prof_record(const char *name, cudaEvent_t a, cudaEvent_t b);
cudaEvent_t prof_event();

struct ProfScope {
    const char *name;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    ProfScope(const char *n, cudaStream_t st) : name(n), s(st) {
        if (!prof_on()) return;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        if (cs != cudaStreamCaptureStatusNone) return;
        a = prof_event();
        cudaEventRecord(a, s);
    }
    ~ProfScope() {
        if (!a) return;
        cudaEvent_t b = prof_event();
        cudaEventRecord(b, s);
        prof_record(name, a, b);
    }
};

// Launch with accounting + immediate launch-error check.
#define CVZ_LAUNCH(kernel, grid, block, smem, stream, ...)              \
    do {                                                                \
        ::cvz::ProfScope _cvz_ps(#kernel, (stream));                    \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);     \
        ::cvz::g_launches.fetch_add(1, std::memory_order_relaxed);      \
        CVZ_CUDA(cudaGetLastError());                                   \
    } while (0)

// Programmatic dependent launch (PDL): the kernel may be scheduled while its
// stream predecessor drains; it must call griddep_wait() before touching
// anything the predecessor produces (a no-op when launched without PDL).
// Used for the chains of small kernels in a layout iteration, where launch
// gaps are a visible share of each ~10-20 us kernel.  CVZ_NO_PDL disables.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = getenv("CVZ_NO_PDL") == nullptr;
    return on;
}

template <class... KArgs, class... Args>
void pdl_launch(const char *name, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                cudaStream_t s, Args... args) {
    ProfScope ps(name, s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    CVZ_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
#define CVZ_LAUNCH_PDL(kernel, grid, block, smem, stream, ...) \
    ::cvz::pdl_launch(#kernel, kernel, dim3(grid), dim3(block), (smem), (stream), __VA_ARGS__)

// Cooperative launch (grid-wide barriers inside the kernel): the grid is the
// number of CTAs that can be co-resident on all SMs.
// `max_grid` > 0 caps the grid (kernels whose work is a known number of CTAs).
template <class... KArgs, class... Args>
void coop_launch_n(const char *name, void (*kernel)(KArgs...), unsigned max_grid, int block,
                   cudaStream_t s, Args... args) {
    int per_sm = 0;
    CVZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0));
    int dev = 0, sms = 0;
    CVZ_CUDA(cudaGetDevice(&dev));
    CVZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    dim3 grid((unsigned)(per_sm > 0 ? per_sm : 1) * (unsigned)sms);
    if (max_grid > 0 && max_grid < grid.x) grid.x = max_grid;
    // arguments converted to the kernel's exact parameter types first
    std::tuple<typename std::decay<KArgs>::type...> typed(args...);
    void *argv[sizeof...(KArgs) > 0 ? sizeof...(KArgs) : 1];
    std::apply([&](auto &...a) {
        int i = 0;
        ((argv[i++] = static_cast<void *>(&a)), ...);
    }, typed);
    ProfScope ps(name, s);
    CVZ_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(kernel), grid, dim3(block),
                                         argv, 0, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}
template <class... KArgs, class... Args>
void coop_launch(const char *name, void (*kernel)(KArgs...), int block, cudaStream_t s,
                 Args... args) {
    coop_launch_n(name, kernel, 0u, block, s, args...);
}
#define CVZ_COOP(kernel, block, stream, ...) \
    ::cvz::coop_launch(#kernel, kernel, (block), (stream), __VA_ARGS__)
#define CVZ_COOP_N(kernel, max_grid, block, stream, ...) \
    ::cvz::coop_launch_n(#kernel, kernel, (max_grid), (block), (stream), __VA_ARGS__)

// Time a library primitive (CUB) under `name` (same rules as CVZ_LAUNCH).
#define CVZ_REGION(name, stream) ::cvz::ProfScope _cvz_region(name, (stream))

// Count a library (CUB) primitive's kernels in the launch tally.
inline void count_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// C-ABI boundary: run body, map exceptions to status codes.
template <class F>
int guard(F &&f) {
    try {
        f();
        return CVZ_OK;
    } catch (const Error &e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        set_last_error(e.what());
        return CVZ_ERR_CUDA;
    }
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// A lazily computed per-device int (SM counts, occupancy, one-time function
// attributes): one slot per device id, so a process that switches devices
// never reuses another device's value.  Racing first calls compute the same
// value, so a relaxed publish is enough.
struct DeviceCache {
    static constexpr int kMax = 64;
    std::atomic<int> v[kMax];
    DeviceCache() {
        for (auto &x : v) x.store(INT_MIN, std::memory_order_relaxed);
    }
    template <class F>
    int get(F &&compute) {
        const int d = current_device();
        if (d < 0 || d >= kMax) return compute();
        int x = v[d].load(std::memory_order_acquire);
        if (x == INT_MIN) {
            x = compute();
            v[d].store(x, std::memory_order_release);
        }
        return x;
    }
};

void init_pool_once();

// Small device -> host readback (counts, flags) that bypasses the copy
// engines: a one-CTA kernel stores the bytes into mapped pinned memory and
// the stream is synchronised.  A cudaMemcpyAsync of four bytes queues behind
// any bulk copy in flight on the same engine (the label prefetch: ~0.5 ms of
// D2H at C4) and would stall the caller that long.  bytes <= 256.
void read_small(void *host, const void *dev, size_t bytes, cudaStream_t s);

// Stream-ordered scratch arena: every allocation is released (stream-ordered)
// when the arena goes out of scope, so kernels queued before the free still
// see valid memory.
class Scratch {
   public:
    explicit Scratch(cudaStream_t s) : s_(s) { init_pool_once(); }
    ~Scratch() {
        for (void *p : ptrs_) cudaFreeAsync(p, s_);
    }
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    template <class T>
    T *alloc(size_t n) {
        void *p = nullptr;
        size_t bytes = n * sizeof(T);
        if (bytes == 0) bytes = 16;
        CVZ_CUDA(cudaMallocAsync(&p, bytes, s_));
        ptrs_.push_back(p);
        return static_cast<T *>(p);
    }
    // Detach an allocation so it outlives the arena (ownership -> caller).
    void release(void *p) {
        for (auto &q : ptrs_)
            if (q == p) q = nullptr;
        std::vector<void *> keep;
        for (void *q : ptrs_)
            if (q) keep.push_back(q);
        ptrs_.swap(keep);
    }
    cudaStream_t stream() const { return s_; }

   private:
    cudaStream_t s_;
    std::vector<void *> ptrs_;
};

template <class T>
T *device_alloc(size_t n, cudaStream_t s) {
    init_pool_once();
    void *p = nullptr;
    CVZ_CUDA(cudaMallocAsync(&p, (n ? n : 1) * sizeof(T), s));
    return static_cast<T *>(p);
}

inline int num_sms() {
    static DeviceCache cache;
    return cache.get([] {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device());
        return sms > 0 ? sms : 148;
    });
}

inline unsigned grid_for(long long work, int block, int per_thread = 1, int waves = 8) {
    long long need = (work + (long long)block * per_thread - 1) / ((long long)block * per_thread);
    long long cap = (long long)num_sms() * waves;
    if (need < 1) need = 1;
    return (unsigned)(need < cap ? need : cap);
}

inline unsigned blocks_for(long long work, int block) {
    long long b = (work + block - 1) / block;
    return (unsigned)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------- device
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Decoupled look-back (single pass) exclusive prefix over tiles.
// status[t] packs (flag << 62) | value; flag 1 = aggregate, 2 = inclusive.
// The caller zeroes status[] and *tile_counter before the launch.
struct LookbackState {
    unsigned long long *status;
    unsigned int *tile_counter;
};

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    return *reinterpret_cast<const volatile unsigned long long *>(p);
}

constexpr unsigned long long LB_AGG = 1ull << 62;
constexpr unsigned long long LB_INC = 2ull << 62;
constexpr unsigned long long LB_VAL = (1ull << 62) - 1;

// Dynamic, monotonically ordered tile id (guarantees forward progress of
// the look-back regardless of CTA scheduling order).  Call from all threads.
__device__ __forceinline__ unsigned acquire_tile(LookbackState st, unsigned *smem_slot) {
    if (threadIdx.x == 0) *smem_slot = atomicAdd(st.tile_counter, 1u);
    __syncthreads();
    return *smem_slot;
}

// Returns the exclusive prefix of this tile (valid in all threads).
// `local` must be valid in thread 0.  smem_slot: one shared u64.
__device__ __forceinline__ unsigned long long tile_prefix(LookbackState st, unsigned tile,
                                                          unsigned long long local,
                                                          unsigned long long *smem_slot) {
    if (threadIdx.x < 32) {
        unsigned long long excl = 0;
        if (tile == 0) {
            if (threadIdx.x == 0) {
                __threadfence();
                atomicExch(&st.status[0], LB_INC | local);
            }
        } else {
            if (threadIdx.x == 0) {
                __threadfence();
                atomicExch(&st.status[tile], LB_AGG | local);
            }
            // warp-parallel look-back over 32 predecessors at a time
            long long base = (long long)tile - 1;
            while (true) {
                long long idx = base - threadIdx.x;
                unsigned long long v = 0;
                if (idx >= 0) {
                    do {
                        v = ld_volatile(&st.status[idx]);
                    } while ((v >> 62) == 0);
                } else {
                    v = LB_INC;  // virtual inclusive zero before tile 0
                }
                unsigned inc_mask = __ballot_sync(0xffffffffu, (v >> 62) == 2);
                // lanes up to (and including) the first inclusive one contribute
                int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
                unsigned long long contrib = (threadIdx.x <= (unsigned)first_inc) ? (v & LB_VAL) : 0;
                for (int o = 16; o > 0; o >>= 1) contrib += __shfl_down_sync(0xffffffffu, contrib, o);
                excl += __shfl_sync(0xffffffffu, contrib, 0);
                if (inc_mask) break;
                base -= 32;
            }
            if (threadIdx.x == 0) {
                __threadfence();
                atomicExch(&st.status[tile], LB_INC | (excl + local));
            }
        }
        if (threadIdx.x == 0) *smem_slot = excl;
    }
    __syncthreads();
    return *smem_slot;
}

// Block-wide exclusive scan of one int per thread (BLOCK threads).
template <int BLOCK>
__device__ __forceinline__ int block_exclusive_scan(int v, int *warp_sums, int &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = (lane < BLOCK / 32) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < BLOCK / 32) warp_sums[lane] = w;
    }
    __syncthreads();
    int before = (wid ? warp_sums[wid - 1] : 0);
    total = warp_sums[BLOCK / 32 - 1];
    __syncthreads();
    return before + x - v;
}

}  // namespace cvz
