// Count-min sketch: Carter-Wegman hashing over the Mersenne prime, weighted
// saturating adds, row-wise-min estimates.  Reference: C/sketch.py:39-98 and
// C/supergraph.py:42-46 (accumulate_sizes).
//
// Adds are integer additions mod 2^64, so any interleaving of atomics gives
// the same table as numpy's sequential np.add.at; the wrap -> INT64_MAX
// saturation runs once afterwards exactly like C/sketch.py:80-86.
//
// Two add paths:
//  * staged: the whole rows x cols table lives in shared memory as u64
//    (default 4 x 6500 = 208 KB fits one CTA per SM); each CTA accumulates
//    its contiguous slice of keys there with plain 64-bit shared atomics
//    (collisions inside a warp are rare over 6,500+ columns) and stores its
//    partial table with coalesced plain stores; one pass sums the partials;
//  * direct: warp-aggregated 64-bit global atomics into the L2-resident table
//    for tables too big for shared memory (e.g. 4 x 107,375 at 2^30 edges).
#include "common.cuh"

namespace cvz {
namespace {

constexpr unsigned long long P31 = 0x7fffffffull;  // 2^31 - 1

__device__ __forceinline__ unsigned long long key_mod_p(long long x) {
    // numpy: x % p with a non-negative result for negative x
    if (x >= 0 && x < (long long)P31) return (unsigned long long)x;
    long long r = x % (long long)P31;
    if (r < 0) r += (long long)P31;
    return (unsigned long long)r;
}

// y mod cols for y < 2^32 without a hardware divide: Lemire's fastmod with
// M = floor((2^64 - 1) / cols) + 1 (exact for 32-bit y and cols).
__device__ __forceinline__ unsigned fast_mod(unsigned y, unsigned cols) {
    const unsigned long long M = 0xFFFFFFFFFFFFFFFFull / cols + 1;  // hoisted: cols is uniform
    return (unsigned)__umul64hi(M * (unsigned long long)y, (unsigned long long)cols);
}

// ((a*x + b) mod p) mod cols with a, x < 2^31, b < 2^31: y < 2^62 + 2^31.
__device__ __forceinline__ unsigned hash_col(unsigned long long a, unsigned long long b,
                                             unsigned long long xm, unsigned cols) {
    unsigned long long y = a * xm + b;
    y = (y & P31) + (y >> 31);  // < 2^31 + 2^32
    y = (y & P31) + (y >> 31);  // < 2^31 + 2
    if (y >= P31) y -= P31;
    return fast_mod((unsigned)y, cols);
}

__global__ void indices_kernel(const long long *__restrict__ ha, const long long *__restrict__ hb,
                               int rows, unsigned cols, const long long *__restrict__ keys,
                               long long k, long long *__restrict__ idx) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < k;
         j += (long long)gridDim.x * blockDim.x) {
        unsigned long long xm = key_mod_p(keys[j]);
        for (int r = 0; r < rows; ++r)
            idx[(long long)r * k + j] = hash_col(ha[r], hb[r], xm, cols);
    }
}

__global__ void negative_check_kernel(const long long *__restrict__ a, long long k,
                                      int *__restrict__ flag) {
    bool neg = false;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < k;
         j += (long long)gridDim.x * blockDim.x)
        neg |= a[j] < 0;
    if (__any_sync(0xffffffffu, neg) && lane_id() == 0) atomicExch(flag, 1);
}

// Warp-level aggregation: lanes hitting the same cell combine their amounts
// (match_any on the cell index) and only the leader issues the atomic.
template <bool SHARED>
__device__ __forceinline__ void agg_add(unsigned long long *base, unsigned cell,
                                        unsigned long long amt, bool valid) {
    unsigned active = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    unsigned peers = __match_any_sync(active, cell);
    int leader = __ffs(peers) - 1;
    // reduce amounts over peers (sum mod 2^64)
    unsigned long long sum = 0;
    unsigned rest = peers;
    while (rest) {
        int l = __ffs(rest) - 1;
        unsigned long long v = __shfl_sync(peers, amt, l);
        sum += v;
        rest &= rest - 1;
    }
    if (lane_id() == leader) atomicAdd(base + cell, sum);
}

template <class Src>
__global__ void add_direct_kernel(unsigned long long *__restrict__ table,
                                  const long long *__restrict__ ha,
                                  const long long *__restrict__ hb, int rows, unsigned cols,
                                  Src src, long long k) {
    long long stride = (long long)gridDim.x * blockDim.x;
    long long kk = (k + 31) / 32 * 32;  // whole warps iterate together
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < kk; j += stride) {
        bool valid = j < k;
        long long key = 0;
        unsigned long long amt = 0;
        if (valid) src.get(j, key, amt);
        unsigned long long xm = valid ? key_mod_p(key) : 0;
        for (int r = 0; r < rows; ++r) {
            unsigned c = valid ? hash_col(ha[r], hb[r], xm, cols) : 0;
            agg_add<false>(table + (size_t)r * cols, c, amt, valid && amt != 0);
        }
    }
}

// Key sources for the staged add: explicit (key, amount) arrays
// (sketch_add_many) or the endpoint slots of an edge list, key = label of the
// endpoint, amount 1 (the edge-based form of accumulate_sizes, SURVEY.md a17:
// identical counters to the node-based form because it is integer addition).
struct KeyAmounts {
    const long long *keys, *amounts;
    long long astride;  // 1, or 0 to broadcast amounts[0] (np.add.at broadcasting)
    __device__ __forceinline__ void get(long long j, long long &key,
                                        unsigned long long &amt) const {
        key = keys[j];
        amt = (unsigned long long)amounts[j * astride];
    }
};
struct EdgeLabels {
    const int *ep;  // int32 endpoints, 2 per edge
    const long long *labels;
    __device__ __forceinline__ void get(long long j, long long &key,
                                        unsigned long long &amt) const {
        key = labels[ep[j]];
        amt = 1;
    }
};

template <class Src>
__global__ void add_staged_kernel(unsigned long long *__restrict__ partial,
                                  const long long *__restrict__ ha,
                                  const long long *__restrict__ hb, int rows, unsigned cols,
                                  Src src, long long k) {
    extern __shared__ unsigned long long sh[];
    const unsigned cells = rows * cols;
    for (unsigned i = threadIdx.x; i < cells; i += blockDim.x) sh[i] = 0;
    __shared__ long long s_a[8], s_b[8];
    if (threadIdx.x < rows) {
        s_a[threadIdx.x] = ha[threadIdx.x];
        s_b[threadIdx.x] = hb[threadIdx.x];
    }
    __syncthreads();
    // contiguous slice per CTA
    long long per = (k + gridDim.x - 1) / gridDim.x;
    long long lo = (long long)blockIdx.x * per, hi = min(k, lo + per);
    for (long long j0 = lo; j0 < hi; j0 += blockDim.x) {
        long long j = j0 + threadIdx.x;
        bool valid = j < hi;
        long long key = 0;
        unsigned long long amt = 0;
        if (valid) src.get(j, key, amt);
        unsigned long long xm = valid ? key_mod_p(key) : 0;
        // shared-memory atomics are cheap and collisions inside a warp are
        // rare (6,500+ columns): no match_any aggregation on this path
        if (valid && amt != 0)
            for (int r = 0; r < rows; ++r)
                atomicAdd(sh + (size_t)r * cols + hash_col(s_a[r], s_b[r], xm, cols), amt);
    }
    __syncthreads();
    // plain coalesced store of this CTA's partial table; reduce_partials sums
    // them (no global atomics on a 26K-cell table from every CTA)
    unsigned long long *mine = partial + (size_t)blockIdx.x * cells;
    for (unsigned i = threadIdx.x; i < cells; i += blockDim.x) mine[i] = sh[i];
}

__global__ void reduce_partials_kernel(unsigned long long *__restrict__ table,
                                       const unsigned long long *__restrict__ partial,
                                       unsigned nparts, unsigned cells) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cells;
         i += gridDim.x * blockDim.x) {
        unsigned long long acc = table[i];  // u64 wrap-around == numpy int64 add.at
        for (unsigned p = 0; p < nparts; ++p) acc += partial[(size_t)p * cells + i];
        table[i] = acc;
    }
}

__global__ void merge_kernel(unsigned long long *__restrict__ table,
                             const unsigned long long *__restrict__ delta, long long cells) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cells;
         i += (long long)gridDim.x * blockDim.x)
        table[i] += delta[i];  // u64 wrap-around == numpy int64 add.at
}

__global__ void saturate_kernel(long long *__restrict__ table, long long cells,
                                int *__restrict__ flag) {
    bool wrapped = false;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cells;
         i += (long long)gridDim.x * blockDim.x) {
        if (table[i] < 0) {
            table[i] = 0x7fffffffffffffffLL;
            wrapped = true;
        }
    }
    if (__any_sync(0xffffffffu, wrapped) && lane_id() == 0) atomicExch(flag, 1);
}

__global__ void estimate_kernel(const long long *__restrict__ table, int rows, unsigned cols,
                                const long long *__restrict__ ha,
                                const long long *__restrict__ hb,
                                const long long *__restrict__ keys, long long k,
                                long long *__restrict__ out) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < k;
         j += (long long)gridDim.x * blockDim.x) {
        unsigned long long xm = key_mod_p(keys[j]);
        long long best = 0x7fffffffffffffffLL;
        for (int r = 0; r < rows; ++r)
            best = min(best, table[(size_t)r * cols + hash_col(ha[r], hb[r], xm, cols)]);
        out[j] = best;
    }
}

constexpr size_t STAGED_MAX_BYTES = 220 * 1024;

}  // namespace

template <class Src>
void sketch_accumulate(int64_t *table, int rows, int64_t cols, const int64_t *ha,
                       const int64_t *hb, Src src, int64_t k, cudaStream_t s) {
    if (k <= 0) return;
    size_t bytes = (size_t)rows * cols * sizeof(unsigned long long);
    bool staged = rows <= 8 && bytes <= STAGED_MAX_BYTES && k >= 4 * (long long)rows * cols;
    auto *t = reinterpret_cast<unsigned long long *>(table);
    auto *pa = reinterpret_cast<const long long *>(ha);
    auto *pb = reinterpret_cast<const long long *>(hb);
    if (staged) {
        static DeviceCache attr;  // the attribute is per device
        attr.get([] {
            CVZ_CUDA(cudaFuncSetAttribute(add_staged_kernel<Src>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)STAGED_MAX_BYTES));
            return 1;
        });
        // one CTA per SM (the table fills its shared memory), on every SM
        // once there are >= 16K keys per CTA; each CTA writes a partial
        // table, one pass sums them into the sketch
        unsigned grid = (unsigned)std::max<long long>(
            1, std::min<long long>((k + 16383) / 16384, num_sms()));
        Scratch sc(s);
        auto *partial = sc.alloc<unsigned long long>((size_t)grid * rows * cols);
        CVZ_LAUNCH(add_staged_kernel<Src>, grid, 1024, bytes, s, partial, pa, pb, rows,
                   (unsigned)cols, src, (long long)k);
        CVZ_LAUNCH(reduce_partials_kernel, grid_for((long long)rows * cols, 256, 1, 4), 256, 0,
                   s, t, partial, grid, (unsigned)(rows * cols));
    } else {
        CVZ_LAUNCH(add_direct_kernel<Src>, grid_for(k, 256, 1, 8), 256, 0, s, t, pa, pb, rows,
                   (unsigned)cols, src, (long long)k);
    }
}

void sketch_saturate(int64_t *table, int rows, int64_t cols, int32_t *d_sat, cudaStream_t s) {
    long long cells = (long long)rows * cols;
    CVZ_LAUNCH(saturate_kernel, grid_for(cells, 256, 4, 2), 256, 0, s,
               reinterpret_cast<long long *>(table), cells, d_sat);
}

void sketch_add(int64_t *table, int rows, int64_t cols, const int64_t *ha, const int64_t *hb,
                const int64_t *keys, const int64_t *amounts, int64_t k, int64_t n_amounts,
                int32_t *d_sat, cudaStream_t s) {
    sketch_accumulate(table, rows, cols, ha, hb,
                      KeyAmounts{reinterpret_cast<const long long *>(keys),
                                 reinterpret_cast<const long long *>(amounts),
                                 n_amounts == k ? 1LL : 0LL},
                      k, s);
    sketch_saturate(table, rows, cols, d_sat, s);
}

void sketch_estimate(const int64_t *table, int rows, int64_t cols, const int64_t *ha,
                     const int64_t *hb, const int64_t *keys, int64_t k, int64_t *out,
                     cudaStream_t s) {
    if (k <= 0) return;
    CVZ_LAUNCH(estimate_kernel, grid_for(k, 256, 1, 8), 256, 0, s,
               reinterpret_cast<const long long *>(table), rows, (unsigned)cols,
               reinterpret_cast<const long long *>(ha), reinterpret_cast<const long long *>(hb),
               reinterpret_cast<const long long *>(keys), (long long)k,
               reinterpret_cast<long long *>(out));
}

}  // namespace cvz

using namespace cvz;

extern "C" {

int cvz_sketch_indices(const int64_t *hash_a, const int64_t *hash_b, int rows, int64_t cols,
                       const int64_t *keys, int64_t k, int64_t *idx, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(rows >= 1 && cols >= 1 && cols < (1LL << 31), CVZ_ERR_VALUE,
                    "sketch needs 1 <= cols < 2^31 and rows >= 1");
        if (k <= 0) return;
        CVZ_LAUNCH(indices_kernel, grid_for(k, 256, 1, 8), 256, 0, as_stream(stream),
                   reinterpret_cast<const long long *>(hash_a),
                   reinterpret_cast<const long long *>(hash_b), rows, (unsigned)cols,
                   reinterpret_cast<const long long *>(keys), (long long)k,
                   reinterpret_cast<long long *>(idx));
    });
}

int cvz_sketch_add(int64_t *table, int rows, int64_t cols, const int64_t *hash_a,
                   const int64_t *hash_b, const int64_t *keys, const int64_t *amounts,
                   int64_t k, int64_t n_amounts, int validate, int32_t *d_saturated,
                   void *stream) {
    return guard([&] {
        CVZ_REQUIRE(rows >= 1 && cols >= 1 && cols < (1LL << 31), CVZ_ERR_VALUE,
                    "sketch needs 1 <= cols < 2^31 and rows >= 1");
        CVZ_REQUIRE(k >= 0 && (n_amounts == k || n_amounts == 1), CVZ_ERR_VALUE,
                    "array is not broadcastable to correct shape");
        cudaStream_t s = as_stream(stream);
        if (validate && k > 0) {
            Scratch sc(s);
            int *flag = sc.alloc<int>(1);
            CVZ_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
            CVZ_LAUNCH(negative_check_kernel, grid_for(n_amounts, 256, 4, 4), 256, 0, s,
                       reinterpret_cast<const long long *>(amounts), (long long)n_amounts, flag);
            int h = 0;
            read_small(&h, flag, sizeof(int), s);
            CVZ_REQUIRE(!h, CVZ_ERR_VALUE, "amounts must be non-negative");
        }
        sketch_add(table, rows, cols, hash_a, hash_b, keys, amounts, k, n_amounts, d_saturated, s);
    });
}

int cvz_sketch_accumulate(int64_t *delta, int rows, int64_t cols, const int64_t *hash_a,
                          const int64_t *hash_b, const int64_t *keys, const int64_t *amounts,
                          int64_t k, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(rows >= 1 && cols >= 1 && cols < (1LL << 31), CVZ_ERR_VALUE,
                    "sketch needs 1 <= cols < 2^31 and rows >= 1");
        sketch_accumulate(delta, rows, cols, hash_a, hash_b,
                          KeyAmounts{reinterpret_cast<const long long *>(keys),
                                     reinterpret_cast<const long long *>(amounts), 1LL},
                          k, as_stream(stream));
    });
}

int cvz_sketch_accumulate_edges(int64_t *delta, int rows, int64_t cols, const int64_t *hash_a,
                                const int64_t *hash_b, const int32_t *edges, int64_t m,
                                const int64_t *labels, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(rows >= 1 && cols >= 1 && cols < (1LL << 31), CVZ_ERR_VALUE,
                    "sketch needs 1 <= cols < 2^31 and rows >= 1");
        CVZ_REQUIRE(m >= 0, CVZ_ERR_VALUE, "negative edge count");
        sketch_accumulate(delta, rows, cols, hash_a, hash_b,
                          EdgeLabels{reinterpret_cast<const int *>(edges),
                                     reinterpret_cast<const long long *>(labels)},
                          2 * m, as_stream(stream));
    });
}

int cvz_sketch_merge(int64_t *table, const int64_t *delta, int rows, int64_t cols,
                     int32_t *d_saturated, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(rows >= 1 && cols >= 1, CVZ_ERR_VALUE, "bad sketch shape");
        cudaStream_t s = as_stream(stream);
        long long cells = (long long)rows * cols;
        CVZ_LAUNCH(merge_kernel, grid_for(cells, 256, 4, 2), 256, 0, s,
                   reinterpret_cast<unsigned long long *>(table),
                   reinterpret_cast<const unsigned long long *>(delta), cells);
        sketch_saturate(table, rows, cols, d_saturated, s);
    });
}

int cvz_sketch_estimate(const int64_t *table, int rows, int64_t cols, const int64_t *hash_a,
                        const int64_t *hash_b, const int64_t *keys, int64_t k, int64_t *out,
                        void *stream) {
    return guard([&] {
        CVZ_REQUIRE(rows >= 1 && cols >= 1 && cols < (1LL << 31), CVZ_ERR_VALUE,
                    "sketch needs 1 <= cols < 2^31 and rows >= 1");
        sketch_estimate(table, rows, cols, hash_a, hash_b, keys, k, out, as_stream(stream));
    });
}

}  // extern "C"
