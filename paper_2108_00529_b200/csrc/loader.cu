// First-seen id remap of a parsed edge list on the GPU: the device half of
// C/graph.py:80-81 (`remap.setdefault(x, len(remap))` for u then v, line by
// line).  SURVEY.md 8f row 1.
//
// Sequentially, an external id's dense id is the number of distinct ids whose
// first occurrence precedes its own.  Order-free form, bit-exact:
//   1. stable radix sort of the 2m slots by external id (only the bits the
//      id range needs), slot index as the value -> each id's run starts at
//      its FIRST occurrence;
//   2. flag[first occurrence slot] = 1; exclusive scan over slot order gives
//      every first occurrence its rank among first occurrences = dense id;
//   3. every slot takes the dense id of its run head (max-scan of head index).
// No hash table, no second sort.  n = number of runs.
#include <cub/cub.cuh>

#include "common.cuh"

namespace cvz {
namespace {

constexpr int RB = 256;

__global__ void minmax_i64_kernel(const long long *__restrict__ x, long long k,
                                  unsigned long long *__restrict__ mm) {
    // mm[0] = min, mm[1] = max in the order-preserving u64 encoding x ^ 2^63
    unsigned long long lo = ~0ull, hi = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned long long v = (unsigned long long)x[i] ^ (1ull << 63);
        lo = min(lo, v);
        hi = max(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane_id() == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

__global__ void remap_keys_kernel(const long long *__restrict__ x, long long k,
                                  const unsigned long long *__restrict__ mm,
                                  unsigned long long *__restrict__ key,
                                  unsigned *__restrict__ val) {
    const unsigned long long base = mm[0];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (long long)gridDim.x * blockDim.x) {
        key[i] = ((unsigned long long)x[i] ^ (1ull << 63)) - base;
        val[i] = (unsigned)i;
    }
}

__global__ void run_heads_kernel(const unsigned long long *__restrict__ skey,
                                 const unsigned *__restrict__ sval, long long k,
                                 unsigned *__restrict__ hidx, unsigned *__restrict__ first) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (long long)gridDim.x * blockDim.x) {
        bool head = i == 0 || skey[i] != skey[i - 1];
        hidx[i] = head ? (unsigned)i : 0u;
        if (head) first[sval[i]] = 1u;  // stable sort: the run head is the first slot
    }
}

__global__ void dense_ids_kernel(const unsigned *__restrict__ sval,
                                 const unsigned *__restrict__ hidx,
                                 const unsigned *__restrict__ rank, long long k,
                                 int *__restrict__ dense) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (long long)gridDim.x * blockDim.x)
        dense[sval[i]] = (int)rank[sval[hidx[i]]];
}

struct MaxOp {
    __device__ __forceinline__ unsigned operator()(unsigned a, unsigned b) const {
        return a > b ? a : b;
    }
};

}  // namespace
}  // namespace cvz

using namespace cvz;

extern "C" {

int cvz_first_seen_remap(const int64_t *ext, int64_t count, int32_t *dense, int64_t *n_out,
                         void *stream) {
    return guard([&] {
        // CUB's num_items is a signed int here: < 2^31 slots (C5 would shard)
        CVZ_REQUIRE(count >= 0 && count < (1LL << 31), CVZ_ERR_VALUE,
                    "remap supports < 2^31 endpoint slots");
        *n_out = 0;
        if (count == 0) return;
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        auto *x = reinterpret_cast<const long long *>(ext);
        auto *mm = sc.alloc<unsigned long long>(2);
        unsigned long long init[2] = {~0ull, 0ull};
        CVZ_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
        CVZ_LAUNCH(minmax_i64_kernel, grid_for(count, RB, 4, 4), RB, 0, s, x, (long long)count,
                   mm);
        unsigned long long hm[2];
        read_small(hm, mm, sizeof(hm), s);
        unsigned long long range = hm[1] - hm[0];
        int bits = 1;
        while (bits < 64 && (range >> bits) != 0) ++bits;
        auto *key = sc.alloc<unsigned long long>(count), *skey = sc.alloc<unsigned long long>(count);
        auto *val = sc.alloc<unsigned>(count), *sval = sc.alloc<unsigned>(count);
        CVZ_LAUNCH(remap_keys_kernel, grid_for(count, RB, 1, 8), RB, 0, s, x, (long long)count, mm,
                   key, val);
        // scratch in / out: sort over DoubleBuffers (no copy pass)
        cub::DoubleBuffer<unsigned long long> dk(key, skey);
        cub::DoubleBuffer<unsigned> dv(val, sval);
        size_t tb = 0;
        CVZ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)count, 0, bits, s));
        void *tmp = sc.alloc<char>(tb);
        {
            CVZ_REGION("cub_sort:remap", s);
            CVZ_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)count, 0, bits, s));
            count_launches(1 + (bits + 7) / 8);
        }
        skey = dk.Current();
        sval = dv.Current();
        auto *hidx = sc.alloc<unsigned>(count), *first = sc.alloc<unsigned>(count);
        auto *rank = sc.alloc<unsigned>(count);
        CVZ_CUDA(cudaMemsetAsync(first, 0, sizeof(unsigned) * count, s));
        CVZ_LAUNCH(run_heads_kernel, grid_for(count, RB, 1, 8), RB, 0, s, skey, sval,
                   (long long)count, hidx, first);
        size_t t1 = 0, t2 = 0;
        CVZ_CUDA(cub::DeviceScan::InclusiveScan(nullptr, t1, hidx, hidx, MaxOp(), (int)count, s));
        CVZ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, first, rank, (int)count, s));
        void *tmp2 = sc.alloc<char>(std::max(t1, t2));
        {
            CVZ_REGION("cub_scan:remap", s);
            CVZ_CUDA(cub::DeviceScan::InclusiveScan(tmp2, t1, hidx, hidx, MaxOp(), (int)count, s));
            CVZ_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, t2, first, rank, (int)count, s));
            count_launches(4);
        }
        CVZ_LAUNCH(dense_ids_kernel, grid_for(count, RB, 1, 8), RB, 0, s, sval, hidx, rank,
                   (long long)count, reinterpret_cast<int *>(dense));
        unsigned tail[2];
        read_small(&tail[0], rank + count - 1, 4, s);
        read_small(&tail[1], first + count - 1, 4, s);
        *n_out = (int64_t)tail[0] + tail[1];
    });
}

}  // extern "C"
