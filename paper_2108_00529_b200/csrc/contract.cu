// Supergraph contraction: dense community ids, sketch weights, superedge
// aggregation by radix sort + run-length encode.  Reference:
// C/supergraph.py:49-76 (np.unique(labels), sketch_estimate_many,
// np.unique(pairs, axis=0, return_counts=True)).  Also the modularity
// ingredients of C/metrics.py:34-46.
//
// Dense ids: when labels are node ids (the detect output) a presence bitmap
// + exclusive scan gives rank-of-label in O(n + range) with no sort; arbitrary
// int64 labels fall back to a (label, node) radix sort.  Superedges: each
// crossing edge becomes one packed key (lo << B) | hi with B = bits(k-1) --
// 32-bit keys whenever k <= 65536 -- so the sort runs only 2B bits and the
// lexicographic (lo, hi) order of np.unique(axis=0) falls out directly.
#include <cub/cub.cuh>

#include "common.cuh"

namespace cvz {

void sketch_estimate(const int64_t *table, int rows, int64_t cols, const int64_t *ha,
                     const int64_t *hb, const int64_t *keys, int64_t k, int64_t *out,
                     cudaStream_t s);

namespace {

__global__ void minmax_kernel(const long long *__restrict__ v, long long n,
                              long long *__restrict__ mn, long long *__restrict__ mx) {
    long long a = LLONG_MAX, b = LLONG_MIN;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        long long x = v[i];
        a = min(a, x);
        b = max(b, x);
    }
    for (int o = 16; o > 0; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane_id() == 0) {
        atomicMin(mn, a);
        atomicMax(mx, b);
    }
}

__global__ void mark_present_kernel(const long long *__restrict__ lab, long long n,
                                    int *__restrict__ present) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        present[lab[i]] = 1;
}

__global__ void comm_from_present_kernel(const int *__restrict__ present,
                                         const int *__restrict__ rank, long long range,
                                         long long *__restrict__ comm) {
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < range;
         v += (long long)gridDim.x * blockDim.x)
        if (present[v]) comm[rank[v]] = v;
}

__global__ void dense_from_rank_kernel(const long long *__restrict__ lab, long long n,
                                       const int *__restrict__ rank, int *__restrict__ dense) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dense[i] = rank[lab[i]];
}

__global__ void head_flags_kernel(const long long *__restrict__ sorted, long long n,
                                  int *__restrict__ flags) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        flags[i] = (i == 0 || sorted[i] != sorted[i - 1]) ? 1 : 0;
}

// incl = inclusive scan of head flags -> dense id = incl - 1
__global__ void dense_from_sorted_kernel(const long long *__restrict__ sorted,
                                         const int *__restrict__ node,
                                         const int *__restrict__ incl, long long n,
                                         int *__restrict__ dense, long long *__restrict__ comm) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int id = incl[i] - 1;
        dense[node[i]] = id;
        if (i == 0 || sorted[i] != sorted[i - 1]) comm[id] = sorted[i];
    }
}

__global__ void iota_kernel(int *__restrict__ v, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] = (int)i;
}

// crossing edges -> packed keys, warp-aggregated append (order is irrelevant:
// the keys are sorted next).
template <class K>
__global__ void cross_keys_kernel(const int2 *__restrict__ e, long long m,
                                  const int *__restrict__ dense, int B, K *__restrict__ out,
                                  unsigned long long *__restrict__ count) {
    // ITEMS edges per thread per step and one append atomic per block and
    // step (per-warp atomics on the single counter serialised ~700K warps
    // at C4)
    constexpr int ITEMS = 4;
    __shared__ unsigned s_w[32];
    __shared__ unsigned long long s_base;
    const long long stride = (long long)gridDim.x * blockDim.x * ITEMS;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    for (long long i0 = (long long)blockIdx.x * blockDim.x * ITEMS; i0 < m; i0 += stride) {
        bool cross[ITEMS];
        K key[ITEMS];
        unsigned mask[ITEMS], mine = 0;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            long long i = i0 + (long long)j * blockDim.x + threadIdx.x;
            cross[j] = false;
            key[j] = 0;
            if (i < m) {
                int2 p = __ldg(e + i);
                int a = __ldg(dense + p.x), b = __ldg(dense + p.y);
                cross[j] = a != b;
                int lo = min(a, b), hi = max(a, b);
                key[j] = ((K)lo << B) | (K)hi;
            }
            mask[j] = __ballot_sync(0xffffffffu, cross[j]);
            mine += __popc(mask[j]);
        }
        if (lane == 0) s_w[wid] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                unsigned c = s_w[w];
                s_w[w] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(count, (unsigned long long)tot) : 0;
        }
        __syncthreads();
        unsigned long long base = s_base + s_w[wid];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (cross[j]) out[base + __popc(mask[j] & ((1u << lane) - 1))] = key[j];
            base += __popc(mask[j]);
        }
        __syncthreads();
    }
}

template <class K>
__global__ void decode_kernel(const K *__restrict__ keys, const int *__restrict__ counts,
                              const long long *__restrict__ nruns, int B,
                              long long *__restrict__ se, long long *__restrict__ mult) {
    long long r = *nruns;
    K maskhi = ((K)1 << B) - 1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < r;
         i += (long long)gridDim.x * blockDim.x) {
        K k = keys[i];
        se[2 * i] = (long long)(k >> B);
        se[2 * i + 1] = (long long)(k & maskhi);
        mult[i] = counts[i];
    }
}

__global__ void modularity_parts_kernel(const int2 *__restrict__ e, long long m,
                                        const int *__restrict__ dense,
                                        unsigned long long *__restrict__ intra) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x) {
        int2 p = __ldg(e + i);
        int a = __ldg(dense + p.x);
        if (a == __ldg(dense + p.y)) atomicAdd(intra + a, 1ull);
    }
}

__global__ void degsum_kernel(const int *__restrict__ dense, const long long *__restrict__ deg,
                              long long n, unsigned long long *__restrict__ degsum) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        atomicAdd(degsum + dense[i], (unsigned long long)deg[i]);
}

// C/metrics.py:70-75 community sizes (bincount of dense ids) and the size
// histogram {size: number of communities}; hist has n + 1 bins.
__global__ void sizes_kernel(const int *__restrict__ dense, long long n,
                             unsigned long long *__restrict__ sizes) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int c = dense[i];
        // warp-aggregate runs of equal ids (labels are clustered)
        unsigned peers = __match_any_sync(__activemask(), c);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(sizes + c, (unsigned long long)__popc(peers));
    }
}

__global__ void size_hist2_kernel(const long long *__restrict__ sizes, long long k,
                                  unsigned long long *__restrict__ hist) {
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < k;
         c += (long long)gridDim.x * blockDim.x)
        atomicAdd(hist + sizes[c], 1ull);
}

// C/metrics.py:34-46 final sum: Q = sum_c intra_c/m - (degsum_c/2m)^2 in fp64
// (block tree + last-block reduction; numpy's pairwise order differs only in
// rounding, the tests gate 1e-9 like T/test_acceptance.py:51-75).
__global__ void modularity_sum_kernel(const long long *__restrict__ intra,
                                      const long long *__restrict__ degsum, long long k,
                                      double m, double *__restrict__ part,
                                      unsigned *__restrict__ ctr, double *__restrict__ q) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < k;
         c += (long long)gridDim.x * blockDim.x) {
        double d = (double)degsum[c] / (2.0 * m);
        acc += (double)intra[c] / m - d * d;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    __shared__ bool last;
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sh[0];
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    double v = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 256) v += ((volatile double *)part)[b];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *q = sh[0];
}

int bits_for(long long k) {  // bits to hold values 0..k-1 (>= 1)
    int b = 1;
    while (b < 62 && (1LL << b) < k) ++b;
    return b;
}

template <class K>
void superedges(const int2 *e, long long m, const int *dense, long long k, int B, Scratch &sc,
                cudaStream_t s, cvz_contract_result *res) {
    K *keys = sc.alloc<K>(m);
    auto *cnt = sc.alloc<unsigned long long>(1);
    CVZ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    if (m > 0)
        CVZ_LAUNCH(cross_keys_kernel<K>, grid_for(m, 256, 1, 16), 256, 0, s, e, m, dense, B, keys,
                   cnt);
    unsigned long long hc = 0;
    read_small(&hc, cnt, sizeof(hc), s);
    long long c = (long long)hc;
    res->se = 0;
    if (c == 0) {
        res->se_edges = device_alloc<int64_t>(0, s);
        res->mult = device_alloc<int64_t>(0, s);
        return;
    }
    // keys are scratch: sort in place over a DoubleBuffer (no copy pass)
    cub::DoubleBuffer<K> dk(keys, sc.alloc<K>(c));
    size_t tb = 0;
    CVZ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, dk, (int)c, 0, 2 * B, s));
    void *tmp = sc.alloc<char>(tb);
    {
        CVZ_REGION("cub_sort:contract_pairs", s);
        CVZ_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, dk, (int)c, 0, 2 * B, s));
    }
    count_launches(1 + (2 * B + 7) / 8);
    K *sorted = dk.Current();
    K *uniq = sc.alloc<K>(c);
    int *counts = sc.alloc<int>(c);
    auto *nruns = sc.alloc<long long>(1);
    size_t tb2 = 0;
    CVZ_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb2, sorted, uniq, counts, nruns, (int)c, s));
    void *tmp2 = sc.alloc<char>(tb2);
    {
        CVZ_REGION("cub_rle:contract_pairs", s);
        CVZ_CUDA(cub::DeviceRunLengthEncode::Encode(tmp2, tb2, sorted, uniq, counts, nruns, (int)c, s));
    }
    count_launches(2);
    long long hr = 0;
    read_small(&hr, nruns, sizeof(hr), s);
    res->se = hr;
    res->se_edges = device_alloc<int64_t>(2 * hr, s);
    res->mult = device_alloc<int64_t>(hr, s);
    CVZ_LAUNCH(decode_kernel<K>, grid_for(hr, 256, 1, 8), 256, 0, s, uniq, counts, nruns, B,
               reinterpret_cast<long long *>(res->se_edges),
               reinterpret_cast<long long *>(res->mult));
}

}  // namespace

// labels -> dense int32 ids + ascending community ids (device, k returned).
long long dense_ids(const int64_t *labels, int64_t n, int *dense, int64_t **comm_out,
                    Scratch &sc, cudaStream_t s) {
    auto *mm = sc.alloc<long long>(2);
    long long init[2] = {LLONG_MAX, LLONG_MIN};
    CVZ_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
    auto *lab = reinterpret_cast<const long long *>(labels);
    CVZ_LAUNCH(minmax_kernel, grid_for(n, 256, 4, 4), 256, 0, s, lab, (long long)n, mm, mm + 1);
    long long h[2];
    read_small(h, mm, sizeof(h), s);
    long long k;
    long long range = h[1] + 1;
    if (h[0] >= 0 && h[1] < (1LL << 31) && range <= std::max<long long>(4 * n, 1 << 20)) {
        int *present = sc.alloc<int>(range);
        int *rank = sc.alloc<int>(range);
        CVZ_CUDA(cudaMemsetAsync(present, 0, sizeof(int) * range, s));
        CVZ_LAUNCH(mark_present_kernel, grid_for(n, 256, 1, 8), 256, 0, s, lab, (long long)n,
                   present);
        size_t tb = 0;
        CVZ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, present, rank, (int)range, s));
        void *tmp = sc.alloc<char>(tb);
        {
            CVZ_REGION("cub_scan:contract_dense", s);
            CVZ_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, present, rank, (int)range, s));
        }
        count_launches(2);
        int last[2];
        read_small(&last[0], rank + range - 1, sizeof(int), s);
        read_small(&last[1], present + range - 1, sizeof(int), s);
        k = (long long)last[0] + last[1];
        int64_t *comm = device_alloc<int64_t>(k, s);
        CVZ_LAUNCH(comm_from_present_kernel, grid_for(range, 256, 1, 8), 256, 0, s, present, rank,
                   range, reinterpret_cast<long long *>(comm));
        CVZ_LAUNCH(dense_from_rank_kernel, grid_for(n, 256, 1, 8), 256, 0, s, lab, (long long)n,
                   rank, dense);
        *comm_out = comm;
    } else {
        long long *sorted = sc.alloc<long long>(n);
        int *iota = sc.alloc<int>(n), *node = sc.alloc<int>(n);
        CVZ_LAUNCH(iota_kernel, grid_for(n, 256, 1, 8), 256, 0, s, iota, (long long)n);
        size_t tb = 0;
        CVZ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, lab, sorted, iota, node, (int)n, 0, 64, s));
        void *tmp = sc.alloc<char>(tb);
        {
            CVZ_REGION("cub_sort:contract_labels", s);
            CVZ_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, lab, sorted, iota, node, (int)n, 0,
                                                     64, s));
        }
        count_launches(9);
        int *flags = sc.alloc<int>(n), *incl = sc.alloc<int>(n);
        CVZ_LAUNCH(head_flags_kernel, grid_for(n, 256, 1, 8), 256, 0, s, sorted, (long long)n, flags);
        size_t tb2 = 0;
        CVZ_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb2, flags, incl, (int)n, s));
        void *tmp2 = sc.alloc<char>(tb2);
        CVZ_CUDA(cub::DeviceScan::InclusiveSum(tmp2, tb2, flags, incl, (int)n, s));
        count_launches(2);
        int hk = 0;
        read_small(&hk, incl + n - 1, sizeof(int), s);
        k = hk;
        int64_t *comm = device_alloc<int64_t>(k, s);
        CVZ_LAUNCH(dense_from_sorted_kernel, grid_for(n, 256, 1, 8), 256, 0, s, sorted, node, incl,
                   (long long)n, dense, reinterpret_cast<long long *>(comm));
        *comm_out = comm;
    }
    return k;
}

}  // namespace cvz

using namespace cvz;

extern "C" {

int cvz_contract(const int32_t *edges, int64_t m, const int64_t *labels, int64_t n,
                 const int64_t *table, int rows, int64_t cols, const int64_t *hash_a,
                 const int64_t *hash_b, cvz_contract_result *res, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n >= 1, CVZ_ERR_VALUE, "contract needs at least one node");
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        *res = cvz_contract_result{0, 0, nullptr, nullptr, nullptr, nullptr};
        try {
            int *dense = sc.alloc<int>(n);
            long long k = dense_ids(labels, n, dense, &res->comm_id, sc, s);
            res->k = k;
            res->weight = device_alloc<int64_t>(k, s);
            sketch_estimate(table, rows, cols, hash_a, hash_b, res->comm_id, k, res->weight, s);
            int B = bits_for(k);
            auto *e = reinterpret_cast<const int2 *>(edges);
            if (2 * B <= 32)
                superedges<unsigned>(e, m, dense, k, B, sc, s, res);
            else
                superedges<unsigned long long>(e, m, dense, k, B, sc, s, res);
        } catch (...) {
            // the result buffers live outside the arena: release them here,
            // the caller never sees a half-filled result
            for (void *p : {(void *)res->comm_id, (void *)res->weight, (void *)res->se_edges,
                            (void *)res->mult})
                if (p) cudaFreeAsync(p, s);
            *res = cvz_contract_result{0, 0, nullptr, nullptr, nullptr, nullptr};
            throw;
        }
    });
}

int cvz_contract_release(cvz_contract_result *res, void *stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        for (void *p : {(void *)res->comm_id, (void *)res->weight, (void *)res->se_edges,
                        (void *)res->mult})
            if (p) CVZ_CUDA(cudaFreeAsync(p, s));
        *res = cvz_contract_result{0, 0, nullptr, nullptr, nullptr, nullptr};
    });
}

int cvz_dense_labels(const int64_t *labels, int64_t n, int32_t *dense, int64_t *k_out,
                     void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n >= 1, CVZ_ERR_VALUE, "need at least one label");
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        int64_t *comm = nullptr;
        *k_out = dense_ids(labels, n, dense, &comm, sc, s);
        if (comm) CVZ_CUDA(cudaFreeAsync(comm, s));
    });
}

int cvz_community_sizes(const int32_t *dense, int64_t n, int64_t k, int64_t *sizes,
                        int64_t *hist, void *stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        CVZ_CUDA(cudaMemsetAsync(sizes, 0, sizeof(int64_t) * (k ? k : 1), s));
        if (n > 0)
            CVZ_LAUNCH(sizes_kernel, grid_for(n, 256, 1, 8), 256, 0, s, dense, (long long)n,
                       reinterpret_cast<unsigned long long *>(sizes));
        if (hist) {
            CVZ_CUDA(cudaMemsetAsync(hist, 0, sizeof(int64_t) * (n + 1), s));
            if (k > 0)
                CVZ_LAUNCH(size_hist2_kernel, grid_for(k, 256, 1, 8), 256, 0, s,
                           reinterpret_cast<const long long *>(sizes), (long long)k,
                           reinterpret_cast<unsigned long long *>(hist));
        }
    });
}

int cvz_modularity(const int32_t *edges, int64_t m, const int32_t *dense, const int64_t *degree,
                   int64_t n, int64_t k, double *q, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(m > 0, CVZ_ERR_VALUE, "modularity undefined for a graph with no edges");
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        auto *intra = sc.alloc<int64_t>(k ? k : 1), *degsum = sc.alloc<int64_t>(k ? k : 1);
        CVZ_CUDA(cudaMemsetAsync(intra, 0, sizeof(int64_t) * (k ? k : 1), s));
        CVZ_CUDA(cudaMemsetAsync(degsum, 0, sizeof(int64_t) * (k ? k : 1), s));
        CVZ_LAUNCH(modularity_parts_kernel, grid_for(m, 256, 1, 16), 256, 0, s,
                   reinterpret_cast<const int2 *>(edges), (long long)m, dense,
                   reinterpret_cast<unsigned long long *>(intra));
        if (n > 0)
            CVZ_LAUNCH(degsum_kernel, grid_for(n, 256, 1, 8), 256, 0, s, dense,
                       reinterpret_cast<const long long *>(degree), (long long)n,
                       reinterpret_cast<unsigned long long *>(degsum));
        unsigned g = grid_for(k, 256, 4, 2);
        auto *part = sc.alloc<double>(g);
        auto *ctr = sc.alloc<unsigned>(1);
        CVZ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
        CVZ_LAUNCH(modularity_sum_kernel, g, 256, 0, s, reinterpret_cast<const long long *>(intra),
                   reinterpret_cast<const long long *>(degsum), (long long)k, (double)m, part, ctr,
                   q);
    });
}

int cvz_modularity_parts(const int32_t *edges, int64_t m, const int32_t *dense,
                         const int64_t *degree, int64_t n, int64_t k, int64_t *intra,
                         int64_t *degsum, void *stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        CVZ_CUDA(cudaMemsetAsync(intra, 0, sizeof(int64_t) * (k ? k : 1), s));
        CVZ_CUDA(cudaMemsetAsync(degsum, 0, sizeof(int64_t) * (k ? k : 1), s));
        if (m > 0)
            CVZ_LAUNCH(modularity_parts_kernel, grid_for(m, 256, 1, 16), 256, 0, s,
                       reinterpret_cast<const int2 *>(edges), (long long)m, dense,
                       reinterpret_cast<unsigned long long *>(intra));
        if (n > 0)
            CVZ_LAUNCH(degsum_kernel, grid_for(n, 256, 1, 8), 256, 0, s, dense,
                       reinterpret_cast<const long long *>(degree), (long long)n,
                       reinterpret_cast<unsigned long long *>(degsum));
    });
}

}  // extern "C"
