// Streaming community detection (SCoDA rounds) on B200.
// Reference: C/community.py:98-120 (_scoda_pass), :123-161 (_resolve_labels),
// :220-281 (detect_communities).
//
// DETERMINISTIC mode -- an order-free restatement of the sequential pass that
// is bit-exact with it:
//   1. every endpoint slot s = 2k+side gets key = node (sentinel n for the
//      second slot of a self-loop and for nodes whose counter already
//      exceeds T -- they can neither change nor merge);
//   2. one stable radix sort of the 2m slots by node puts each node's slots
//      in stream order, so the post-increment counter of a slot is
//      min(d0 + rank, T+1) with rank = position - segment start + 1;
//   3. per edge: active iff both counters <= T; the smaller counter adopts
//      (tie rule) -> the event k writes lab[target] := lab[source];
//   4. in the same sorted order a segmented max-scan of "k if this slot is a
//      write" gives, for every read slot, the last earlier write to that
//      node = the event's parent; values then resolve by pointer jumping;
//   5. final counter = min(d0 + count, T+1), final label = value of the last
//      write (segment tail) or the initial label.
// FAST mode -- the literal streaming pass, one thread per edge: counters via
// 32-bit atomics (skipped once a node is saturated), racy label stores.
//
// Label resolution: functional graph x -> lab[x]; representative = min id on
// the reached cycle.  Pointer doubling with a shrinking worklist until every
// node sees a fixed point; nodes that never do sit on/above a >=2-cycle and
// get a min-doubling pass over the (closed) set of such nodes.
#include <algorithm>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"

namespace cvz {
namespace {

constexpr int TB = 256;
// fast mode: edges in flight <= m / FAST_WINDOW_DIV
constexpr long long FAST_WINDOW_DIV = 128;

struct MaxOp {
    __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};

__global__ void gather_edges_kernel(const int2 *__restrict__ e, const long long *__restrict__ order,
                                    long long m, int2 *__restrict__ out) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x)
        out[k] = __ldg(e + order[k]);
}

// ---- deterministic pass --------------------------------------------------

__global__ void slot_keys_kernel(const int2 *__restrict__ E, long long m,
                                 const long long *__restrict__ d0, long long T, unsigned n,
                                 uint2 *__restrict__ keys, uint2 *__restrict__ vals) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        int2 p = __ldg(E + k);
        unsigned ku = (unsigned)p.x, kv = (unsigned)p.y;
        if (p.x == p.y) kv = n;  // a self-loop bumps its counter once
        if (d0) {
            if (__ldg(d0 + p.x) > T) ku = n;
            if (__ldg(d0 + p.y) > T) kv = n;
        }
        keys[k] = make_uint2(ku, kv);
        vals[k] = make_uint2((unsigned)(2 * k), (unsigned)(2 * k + 1));
    }
}

__global__ void seg_bounds_kernel(const unsigned *__restrict__ key, long long ns, unsigned n,
                                  int *__restrict__ seg_start, int *__restrict__ seg_end) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ns;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned x = key[i];
        if (x >= n) continue;
        if (i == 0 || key[i - 1] != x) seg_start[x] = (int)i;
        if (i == ns - 1 || key[i + 1] != x) seg_end[x] = (int)(i + 1);
    }
}

template <class CT>
__global__ void slot_counter_kernel(const unsigned *__restrict__ key,
                                    const unsigned *__restrict__ val, long long ns, unsigned n,
                                    const int *__restrict__ seg_start,
                                    const long long *__restrict__ d0, long long T,
                                    CT *__restrict__ cval) {
    const CT big = (CT)(T + 1);  // > T: marks sentinel slots inactive
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ns;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned x = key[i], s = val[i];
        if (x >= n) {
            cval[s] = big;
            continue;
        }
        long long r = i - seg_start[x] + 1;
        long long d = d0 ? d0[x] : 0;
        long long c = d > T ? d : min(d + r, T + 1);
        cval[s] = (CT)c;
    }
}

template <class CT>
__global__ void edge_role_kernel(const int2 *__restrict__ E, long long m,
                                 const CT *__restrict__ cval, long long T, int tie,
                                 signed char *__restrict__ role) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        int2 p = __ldg(E + k);
        long long du = cval[2 * k], dv = cval[2 * k + 1];
        signed char r = -1;
        if (p.x != p.y && du <= T && dv <= T) {
            if (du < dv)
                r = 0;  // u adopts v's label  (C/community.py:112-113)
            else if (dv < du)
                r = 1;  // v adopts u's label  (:114-115)
            else
                r = tie == 0 ? 0 : (tie == 1 ? 1 : -1);  // (:116-120)
        }
        role[k] = r;
    }
}

// write-slot indicator: k if slot i (sorted) is the TARGET of event k
struct WriteVal {
    const unsigned *key, *val;
    const signed char *role;
    unsigned n;
    __device__ __forceinline__ int operator()(int i) const {
        unsigned x = key[i];
        if (x >= n) return -1;
        unsigned s = val[i];
        int k = (int)(s >> 1);
        return role[k] == (signed char)(s & 1) ? k : -1;
    }
};

__global__ void parents_kernel(const unsigned *__restrict__ key, const unsigned *__restrict__ val,
                               long long ns, unsigned n, const signed char *__restrict__ role,
                               const int *__restrict__ lastw, int *__restrict__ parent,
                               int *__restrict__ finalw) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ns;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned x = key[i];
        if (x >= n) continue;
        unsigned s = val[i];
        int k = (int)(s >> 1);
        signed char r = role[k];
        if (r >= 0 && r != (signed char)(s & 1)) parent[k] = lastw[i];  // source slot
        if (i == ns - 1 || key[i + 1] != x) finalw[x] = lastw[i];
    }
}

// events: origin[k] = node whose initial label event k carries (-1 pending)
__global__ void events_init_kernel(const int2 *__restrict__ E, long long m,
                                   const signed char *__restrict__ role,
                                   const int *__restrict__ parent, int *__restrict__ origin,
                                   int *__restrict__ ptr, int *__restrict__ work,
                                   unsigned *__restrict__ nwork) {
    long long mm = (m + 31) / 32 * 32;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < mm;
         k += (long long)gridDim.x * blockDim.x) {
        bool pend = false;
        if (k < m) {
            signed char r = role[k];
            if (r >= 0) {
                int2 p = __ldg(E + k);
                int src = r == 0 ? p.y : p.x;
                int par = parent[k];
                if (par < 0) {
                    origin[k] = src;
                } else {
                    origin[k] = -1;
                    ptr[k] = par;
                    pend = true;
                }
            }
        }
        unsigned mask = __ballot_sync(0xffffffffu, pend);
        unsigned base = 0;
        if (lane_id() == 0 && mask) base = atomicAdd(nwork, (unsigned)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (pend) work[base + __popc(mask & ((1u << lane_id()) - 1))] = (int)k;
    }
}

// one pointer-jumping sweep; racy reads of origin/ptr are safe (monotone)
__global__ void events_jump_kernel(const int *__restrict__ work, const unsigned *__restrict__ nin,
                                   volatile int *origin, volatile int *ptr,
                                   int *__restrict__ work_out, unsigned *__restrict__ nout) {
    unsigned cnt = *nin;
    unsigned cc = (cnt + 31) / 32 * 32;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cc; t += gridDim.x * blockDim.x) {
        bool keep = false;
        int k = -1;
        if (t < cnt) {
            k = work[t];
            int p = ptr[k];
            int op = origin[p];
            if (op >= 0) {
                origin[k] = op;
            } else {
                ptr[k] = ptr[p];
                keep = true;
            }
        }
        unsigned mask = __ballot_sync(0xffffffffu, keep);
        unsigned base = 0;
        if (lane_id() == 0 && mask) base = atomicAdd(nout, (unsigned)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) work_out[base + __popc(mask & ((1u << lane_id()) - 1))] = k;
    }
}

__global__ void det_finalize_kernel(long long n, const int *__restrict__ seg_start,
                                    const int *__restrict__ seg_end,
                                    const int *__restrict__ finalw, const int *__restrict__ origin,
                                    const long long *__restrict__ d0,
                                    const long long *__restrict__ lab0, long long T,
                                    long long *__restrict__ deg_out,
                                    long long *__restrict__ lab_out) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        int st = seg_start[x];
        long long cnt = st >= 0 ? (long long)(seg_end[x] - st) : 0;
        long long d = d0 ? d0[x] : 0;
        deg_out[x] = d > T ? d : min(d + cnt, T + 1);
        int fw = st >= 0 ? finalw[x] : -1;
        long long src = fw >= 0 ? (long long)origin[fw] : x;
        lab_out[x] = lab0 ? lab0[src] : src;
    }
}

// ---- fast (racy) pass ------------------------------------------------------

__device__ __forceinline__ long long bump(unsigned *cnt, int x, long long d, long long T) {
    if (d > T) return d;
    long long room = T + 1 - d;  // increments that still matter
    unsigned cur = *(volatile unsigned *)(cnt + x);
    if ((long long)cur >= room) return T + 1;  // saturated: skip the atomic
    unsigned old = atomicAdd(cnt + x, 1u);
    return min(d + (long long)old + 1, T + 1);
}

__global__ void fast_pass_kernel(const int2 *__restrict__ E, long long m,
                                 const long long *__restrict__ d0, long long T, int tie,
                                 unsigned *__restrict__ cnt, volatile long long *lab) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        int2 p = __ldg(E + k);
        long long du0 = d0 ? d0[p.x] : 0, dv0 = d0 ? d0[p.y] : 0;
        if (p.x == p.y) {
            bump(cnt, p.x, du0, T);
            continue;
        }
        long long du = bump(cnt, p.x, du0, T);
        long long dv = bump(cnt, p.y, dv0, T);
        if (du > T || dv > T) continue;
        if (du < dv || (du == dv && tie == 0))
            lab[p.x] = lab[p.y];
        else if (dv < du || (du == dv && tie == 1))
            lab[p.y] = lab[p.x];
    }
}

__global__ void fast_finalize_kernel(long long n, const unsigned *__restrict__ cnt,
                                     const long long *__restrict__ d0, long long T,
                                     long long *__restrict__ deg_out) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        long long d = d0 ? d0[x] : 0;
        deg_out[x] = d > T ? d : min(d + (long long)cnt[x], T + 1);
    }
}

__global__ void init_labels_kernel(long long n, const long long *__restrict__ lab0,
                                   long long *__restrict__ lab) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x)
        lab[x] = lab0 ? lab0[x] : x;
}

// ---- resolve ---------------------------------------------------------------

__global__ void resolve_init_kernel(const long long *__restrict__ lab, long long n,
                                    int *__restrict__ f, int *__restrict__ p,
                                    long long *__restrict__ rep, int *__restrict__ work,
                                    unsigned *__restrict__ nwork, int *__restrict__ bad) {
    long long nn = (n + 31) / 32 * 32;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < nn;
         x += (long long)gridDim.x * blockDim.x) {
        bool pend = false;
        if (x < n) {
            long long y = lab[x];
            if (y < 0 || y >= n) {
                atomicExch(bad, 1);
                y = x;
            }
            f[x] = (int)y;
            p[x] = (int)y;
            if (y == x)
                rep[x] = x;
            else
                pend = true;
        }
        unsigned mask = __ballot_sync(0xffffffffu, pend);
        unsigned base = 0;
        if (lane_id() == 0 && mask) base = atomicAdd(nwork, (unsigned)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (pend) work[base + __popc(mask & ((1u << lane_id()) - 1))] = (int)x;
    }
}

__global__ void resolve_jump_kernel(const int *__restrict__ work, const unsigned *__restrict__ nin,
                                    const int *__restrict__ f, volatile int *p,
                                    long long *__restrict__ rep, int *__restrict__ work_out,
                                    unsigned *__restrict__ nout) {
    unsigned cnt = *nin;
    unsigned cc = (cnt + 31) / 32 * 32;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cc; t += gridDim.x * blockDim.x) {
        bool keep = false;
        int x = -1;
        if (t < cnt) {
            x = work[t];
            int y = p[x];
            if (f[y] == y) {
                rep[x] = y;  // reached a fixed point
            } else {
                p[x] = p[y];
                keep = true;
            }
        }
        unsigned mask = __ballot_sync(0xffffffffu, keep);
        unsigned base = 0;
        if (lane_id() == 0 && mask) base = atomicAdd(nout, (unsigned)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) work_out[base + __popc(mask & ((1u << lane_id()) - 1))] = x;
    }
}

__global__ void cycle_min_init_kernel(const int *__restrict__ work, unsigned cnt,
                                      const int *__restrict__ f, int *__restrict__ mn,
                                      int *__restrict__ q) {
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        int x = work[t];
        mn[x] = min(x, f[x]);
        q[x] = f[f[x]];
    }
}

__global__ void cycle_min_step_kernel(const int *__restrict__ work, unsigned cnt,
                                      const int *__restrict__ mn_in, const int *__restrict__ q_in,
                                      int *__restrict__ mn_out, int *__restrict__ q_out) {
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        int x = work[t];
        int y = q_in[x];
        mn_out[x] = min(mn_in[x], mn_in[y]);
        q_out[x] = q_in[y];
    }
}

__global__ void cycle_rep_kernel(const int *__restrict__ work, unsigned cnt,
                                 const int *__restrict__ p, const int *__restrict__ mn,
                                 long long *__restrict__ rep) {
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        int x = work[t];
        rep[x] = mn[p[x]];
    }
}

// ---- round driver helpers --------------------------------------------------

__global__ void size_hist_kernel(const long long *__restrict__ node_lab, long long n,
                                 unsigned *__restrict__ size) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        int l = (int)node_lab[x];
        unsigned peers = __match_any_sync(__activemask(), l);  // warp-aggregated
        if (lane_id() == __ffs(peers) - 1) atomicAdd(size + l, (unsigned)__popc(peers));
    }
}

__global__ void seed_counters_kernel(const unsigned *__restrict__ size, long long n, long long T,
                                     long long *__restrict__ d0) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        long long s = (long long)size[x] - 1;  // C/community.py:258-261
        d0[x] = max(0LL, min(s, T + 1));
    }
}

__global__ void compose_kernel(long long n, const long long *__restrict__ rep,
                               long long *__restrict__ node_lab, long long *__restrict__ prev,
                               long long *__restrict__ hist, int check, int *__restrict__ changed) {
    bool diff = false;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        long long v = rep[node_lab[x]];
        node_lab[x] = v;
        if (hist) hist[x] = v;
        if (check) diff |= prev[x] != v;
        prev[x] = v;
    }
    if (__any_sync(__activemask(), diff) && lane_id() == 0) atomicExch(changed, 1);
}

// stable relabel + drop-intra compaction (single pass, decoupled look-back)
constexpr int RITEMS = 8;
constexpr int RTILE = TB * RITEMS;

__global__ void __launch_bounds__(TB) relabel_compact_kernel(
    const int2 *__restrict__ in, long long m, const long long *__restrict__ map,
    int2 *__restrict__ out, LookbackState st, unsigned long long *__restrict__ d_count,
    unsigned num_tiles) {
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_prefix;
    __shared__ int s_warp[TB / 32];
    const unsigned tile = acquire_tile(st, &s_tile);
    const long long base = (long long)tile * RTILE;
    int2 e[RITEMS];
    bool keep[RITEMS];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < RITEMS; ++j) {
        long long i = base + (long long)j * TB + threadIdx.x;
        keep[j] = false;
        if (i < m) {
            int2 p = __ldg(in + i);
            int a = (int)__ldg(map + p.x), b = (int)__ldg(map + p.y);
            e[j] = make_int2(a, b);
            keep[j] = a != b;
            cnt += keep[j];
        }
    }
    int total;
    block_exclusive_scan<TB>(cnt, s_warp, total);
    unsigned long long prefix = tile_prefix(st, tile, (unsigned long long)total, &s_prefix);
    long long run = 0;
#pragma unroll
    for (int j = 0; j < RITEMS; ++j) {
        int tot_j;
        int o = block_exclusive_scan<TB>(keep[j] ? 1 : 0, s_warp, tot_j);
        if (keep[j]) out[prefix + run + o] = e[j];
        run += tot_j;
    }
    if (threadIdx.x == 0 && tile == num_tiles - 1) *d_count = prefix + total;
}

template <class T>
void cub_sort_pairs(const unsigned *kin, unsigned *kout, const T *vin, T *vout, long long ns,
                    int end_bit, Scratch &sc, cudaStream_t s) {
    size_t tb = 0;
    CVZ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, (int)ns, 0,
                                             end_bit, s));
    void *tmp = sc.alloc<char>(tb);
    CVZ_REGION("cub_sort:scoda_slots", s);
    CVZ_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, (int)ns, 0, end_bit,
                                             s));
    count_launches(1 + (end_bit + 7) / 8);
}

int bits_for_value(unsigned long long v) {  // bits to hold 0..v
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

}  // namespace

// Deterministic pass.  E: stream-ordered edges.  lab0/d0 nullable.
template <class CT>
static void det_pass_t(const int2 *E, long long m, long long n, long long T, int tie,
                       const int64_t *d0, const int64_t *lab0, int64_t *deg_out,
                       int64_t *lab_out, Scratch &sc, cudaStream_t s) {
    const long long ns = 2 * m;
    auto *d0p = reinterpret_cast<const long long *>(d0);
    auto *keys = sc.alloc<unsigned>(ns), *vals = sc.alloc<unsigned>(ns);
    auto *skeys = sc.alloc<unsigned>(ns), *svals = sc.alloc<unsigned>(ns);
    int *seg_start = sc.alloc<int>(n), *seg_end = sc.alloc<int>(n), *finalw = sc.alloc<int>(n);
    CVZ_CUDA(cudaMemsetAsync(seg_start, 0xff, sizeof(int) * n, s));
    CVZ_CUDA(cudaMemsetAsync(finalw, 0xff, sizeof(int) * n, s));
    int *origin = nullptr;
    if (m > 0) {
        CVZ_LAUNCH(slot_keys_kernel, grid_for(m, TB, 1, 16), TB, 0, s, E, m, d0p, T, (unsigned)n,
                   reinterpret_cast<uint2 *>(keys), reinterpret_cast<uint2 *>(vals));
        cub_sort_pairs(keys, skeys, vals, svals, ns, bits_for_value((unsigned long long)n), sc, s);
        CVZ_LAUNCH(seg_bounds_kernel, grid_for(ns, TB, 1, 16), TB, 0, s, skeys, ns, (unsigned)n,
                   seg_start, seg_end);
        CT *cval = sc.alloc<CT>(ns);
        CVZ_LAUNCH(slot_counter_kernel<CT>, grid_for(ns, TB, 1, 16), TB, 0, s, skeys, svals, ns,
                   (unsigned)n, seg_start, d0p, T, cval);
        auto *role = sc.alloc<signed char>(m);
        CVZ_LAUNCH(edge_role_kernel<CT>, grid_for(m, TB, 1, 16), TB, 0, s, E, m, cval, T, tie,
                   role);
        // segmented "last write so far" over the node-sorted slots
        int *lastw = sc.alloc<int>(ns);
        WriteVal wv{skeys, svals, role, (unsigned)n};
        auto vin = thrust::make_transform_iterator(thrust::counting_iterator<int>(0), wv);
        size_t tb = 0;
        CVZ_CUDA(cub::DeviceScan::InclusiveScanByKey(nullptr, tb, skeys, vin, lastw, MaxOp(),
                                                     (int)ns, cub::Equality(), s));
        void *tmp = sc.alloc<char>(tb);
        {
            CVZ_REGION("cub_scan_by_key:scoda_lastw", s);
            CVZ_CUDA(cub::DeviceScan::InclusiveScanByKey(tmp, tb, skeys, vin, lastw, MaxOp(),
                                                         (int)ns, cub::Equality(), s));
        }
        count_launches(2);
        int *parent = sc.alloc<int>(m);
        CVZ_LAUNCH(parents_kernel, grid_for(ns, TB, 1, 16), TB, 0, s, skeys, svals, ns,
                   (unsigned)n, role, lastw, parent, finalw);
        origin = sc.alloc<int>(m);
        int *ptr = sc.alloc<int>(m);
        int *wa = sc.alloc<int>(m), *wb = sc.alloc<int>(m);
        unsigned *cnt = sc.alloc<unsigned>(2);
        CVZ_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned), s));
        CVZ_LAUNCH(events_init_kernel, grid_for(m, TB, 1, 16), TB, 0, s, E, m, role, parent,
                   origin, ptr, wa, cnt);
        unsigned hc = 0;
        CVZ_CUDA(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
        CVZ_CUDA(cudaStreamSynchronize(s));
        int cur = 0;
        while (hc > 0) {
            unsigned *cin = cnt + cur, *cout = cnt + (1 - cur);
            CVZ_CUDA(cudaMemsetAsync(cout, 0, sizeof(unsigned), s));
            CVZ_LAUNCH(events_jump_kernel, grid_for(hc, TB, 1, 16), TB, 0, s, cur ? wb : wa, cin,
                       origin, ptr, cur ? wa : wb, cout);
            CVZ_CUDA(cudaMemcpyAsync(&hc, cout, sizeof(hc), cudaMemcpyDeviceToHost, s));
            CVZ_CUDA(cudaStreamSynchronize(s));
            cur = 1 - cur;
        }
    }
    if (!origin) origin = sc.alloc<int>(1);
    CVZ_LAUNCH(det_finalize_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n, seg_start, seg_end,
               finalw, origin, d0p, reinterpret_cast<const long long *>(lab0), T,
               reinterpret_cast<long long *>(deg_out), reinterpret_cast<long long *>(lab_out));
}

void scoda_pass_dev(const int2 *E, long long m, long long n, long long T, int tie, int mode,
                    const int64_t *d0, const int64_t *lab0, int64_t *deg_out, int64_t *lab_out,
                    Scratch &sc, cudaStream_t s) {
    CVZ_REQUIRE(2 * m < (1LL << 31) - 1, CVZ_ERR_VALUE,
                "edge stream too long for one pass (2m must be < 2^31)");
    if (mode == CVZ_SCODA_DETERMINISTIC) {
        if (T < (1LL << 30))
            det_pass_t<int>(E, m, n, T, tie, d0, lab0, deg_out, lab_out, sc, s);
        else
            det_pass_t<long long>(E, m, n, T, tie, d0, lab0, deg_out, lab_out, sc, s);
        return;
    }
    unsigned *cnt = sc.alloc<unsigned>(n);
    CVZ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * n, s));
    CVZ_LAUNCH(init_labels_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n,
               reinterpret_cast<const long long *>(lab0), reinterpret_cast<long long *>(lab_out));
    if (m > 0) {
        // Bounded in-flight window: the racy pass stays close to the
        // reference's own parallel schedules (C/community.py:164-195) only
        // while the edges in flight are a small fraction of the stream
        // (DESIGN.md "fast mode"); at C4 scale this is full occupancy anyway.
        long long window = std::max(256LL, std::min(m / FAST_WINDOW_DIV, 2048LL * num_sms()));
        unsigned blocks = (unsigned)((window + TB - 1) / TB);
        CVZ_LAUNCH(fast_pass_kernel, blocks, TB, 0, s, E, m,
                   reinterpret_cast<const long long *>(d0), T, tie, cnt,
                   reinterpret_cast<volatile long long *>(lab_out));
    }
    CVZ_LAUNCH(fast_finalize_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n, cnt,
               reinterpret_cast<const long long *>(d0), T, reinterpret_cast<long long *>(deg_out));
}

// rep[x] = min id on the cycle reached from lab[x].  Returns false on range error
// (only checked when check != 0; that synchronises).
void resolve_dev(const int64_t *lab, long long n, int64_t *rep_out, bool check, Scratch &sc,
                 cudaStream_t s) {
    if (n <= 0) return;
    int *f = sc.alloc<int>(n), *p = sc.alloc<int>(n);
    int *wa = sc.alloc<int>(n), *wb = sc.alloc<int>(n);
    unsigned *cnt = sc.alloc<unsigned>(2);
    int *bad = sc.alloc<int>(1);
    CVZ_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned), s));
    CVZ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    auto *rep = reinterpret_cast<long long *>(rep_out);
    CVZ_LAUNCH(resolve_init_kernel, grid_for(n, TB, 1, 8), TB, 0, s,
               reinterpret_cast<const long long *>(lab), n, f, p, rep, wa, cnt, bad);
    unsigned hc[2] = {0, 0};
    int hbad = 0;
    CVZ_CUDA(cudaMemcpyAsync(&hc[0], cnt, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    if (check) CVZ_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CVZ_CUDA(cudaStreamSynchronize(s));
    CVZ_REQUIRE(!hbad, CVZ_ERR_RANGE, "labels must lie in [0, n)");
    unsigned c = hc[0];
    int cur = 0;
    int rounds = 0;
    const int max_rounds = bits_for_value((unsigned long long)n) + 2;  // 2^rounds >= n
    while (c > 0 && rounds < max_rounds) {
        unsigned *cin = cnt + cur, *cout = cnt + (1 - cur);
        CVZ_CUDA(cudaMemsetAsync(cout, 0, sizeof(unsigned), s));
        CVZ_LAUNCH(resolve_jump_kernel, grid_for(c, TB, 1, 16), TB, 0, s, cur ? wb : wa, cin, f,
                   p, rep, cur ? wa : wb, cout);
        CVZ_CUDA(cudaMemcpyAsync(&c, cout, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        CVZ_CUDA(cudaStreamSynchronize(s));
        cur = 1 - cur;
        ++rounds;
    }
    if (c > 0) {
        // remaining nodes never reach a fixed point: p[x] is on a >=2 cycle and
        // the remaining set is closed under f.  Min over each cycle by doubling.
        int *work = cur ? wb : wa;
        int *mn_a = sc.alloc<int>(n), *q_a = sc.alloc<int>(n);
        int *mn_b = sc.alloc<int>(n), *q_b = sc.alloc<int>(n);
        unsigned g = grid_for(c, TB, 1, 16);
        CVZ_LAUNCH(cycle_min_init_kernel, g, TB, 0, s, work, c, f, mn_a, q_a);
        // after init the window covers 2 nodes; double until >= n
        for (int r = 1; r < max_rounds; ++r) {
            CVZ_LAUNCH(cycle_min_step_kernel, g, TB, 0, s, work, c, mn_a, q_a, mn_b, q_b);
            std::swap(mn_a, mn_b);
            std::swap(q_a, q_b);
        }
        CVZ_LAUNCH(cycle_rep_kernel, g, TB, 0, s, work, c, p, mn_a, rep);
    }
}

}  // namespace cvz

using namespace cvz;

extern "C" {

int cvz_scoda_pass(const int32_t *edges, int64_t m, const int64_t *order, int64_t n,
                   int64_t threshold, int tie_code, int mode, int64_t *deg, int64_t *lab,
                   int64_t *lab_raw, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n >= 1, CVZ_ERR_VALUE, "pass needs n >= 1");
        CVZ_REQUIRE(tie_code >= 0 && tie_code <= 2, CVZ_ERR_VALUE, "unknown tie rule");
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        const int2 *E = reinterpret_cast<const int2 *>(edges);
        if (order && m > 0) {
            int2 *g = sc.alloc<int2>(m);
            CVZ_LAUNCH(gather_edges_kernel, grid_for(m, TB, 1, 16), TB, 0, s, E,
                       reinterpret_cast<const long long *>(order), (long long)m, g);
            E = g;
        }
        int64_t *d0 = sc.alloc<int64_t>(n), *l0 = sc.alloc<int64_t>(n);
        CVZ_CUDA(cudaMemcpyAsync(d0, deg, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, s));
        CVZ_CUDA(cudaMemcpyAsync(l0, lab, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, s));
        int64_t *raw = lab_raw ? lab_raw : sc.alloc<int64_t>(n);
        scoda_pass_dev(E, m, n, threshold, tie_code, mode, d0, l0, deg, raw, sc, s);
        resolve_dev(raw, n, lab, true, sc, s);
    });
}

int cvz_resolve_labels(const int64_t *lab, int64_t n, int64_t *out, void *stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        resolve_dev(lab, n, out, true, sc, s);
    });
}

int cvz_detect_round(const int32_t *cur_edges, int64_t m_cur, const int64_t *order,
                     const int32_t *orig_edges, int64_t m_orig, int64_t n, int64_t threshold,
                     int tie_code, int mode, int round_index, int round_stream,
                     int64_t *node_lab, int64_t *prev_lab, int64_t *deg_out,
                     int64_t *history_out, int32_t *next_edges, int64_t *next_m, int *changed,
                     void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n >= 1, CVZ_ERR_VALUE, "detect needs n >= 1");
        CVZ_REQUIRE(tie_code >= 0 && tie_code <= 2, CVZ_ERR_VALUE, "unknown tie rule");
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        const long long T = threshold;
        // 1. size-seeded counters (C/community.py:257-261)
        int64_t *d0 = nullptr;
        if (round_index > 1) {
            unsigned *size = sc.alloc<unsigned>(n);
            CVZ_CUDA(cudaMemsetAsync(size, 0, sizeof(unsigned) * n, s));
            CVZ_LAUNCH(size_hist_kernel, grid_for(n, TB, 1, 8), TB, 0, s,
                       reinterpret_cast<const long long *>(node_lab), (long long)n, size);
            d0 = sc.alloc<int64_t>(n);
            CVZ_LAUNCH(seed_counters_kernel, grid_for(n, TB, 1, 8), TB, 0, s, size, (long long)n,
                       T, reinterpret_cast<long long *>(d0));
        }
        // 2. processing order (C/community.py:263)
        const int2 *cur = reinterpret_cast<const int2 *>(cur_edges);
        const int2 *E = cur;
        if (order && m_cur > 0) {
            int2 *g = sc.alloc<int2>(m_cur);
            CVZ_LAUNCH(gather_edges_kernel, grid_for(m_cur, TB, 1, 16), TB, 0, s, cur,
                       reinterpret_cast<const long long *>(order), (long long)m_cur, g);
            E = g;
        }
        // 3. pass + resolve (labels restart at arange(n), :262-265)
        int64_t *raw = sc.alloc<int64_t>(n), *rep = sc.alloc<int64_t>(n);
        scoda_pass_dev(E, m_cur, n, T, tie_code, mode, d0, nullptr, deg_out, raw, sc, s);
        resolve_dev(raw, n, rep, false, sc, s);
        // 4. compose + history + early-stop test (:266-269)
        int *dchg = sc.alloc<int>(1);
        CVZ_CUDA(cudaMemsetAsync(dchg, 0, sizeof(int), s));
        CVZ_LAUNCH(compose_kernel, grid_for(n, TB, 1, 8), TB, 0, s, (long long)n,
                   reinterpret_cast<const long long *>(rep), reinterpret_cast<long long *>(node_lab),
                   reinterpret_cast<long long *>(prev_lab),
                   reinterpret_cast<long long *>(history_out), round_index > 1 ? 1 : 0, dchg);
        int hchg = 1;
        if (round_index > 1) {
            CVZ_CUDA(cudaMemcpyAsync(&hchg, dchg, sizeof(int), cudaMemcpyDeviceToHost, s));
            CVZ_CUDA(cudaStreamSynchronize(s));
        }
        *changed = hchg;
        *next_m = 0;
        if (!hchg) return;
        // 5. next stream: contract (:272-278) or restream (:274-276)
        const int2 *src = round_stream == 0 ? cur : reinterpret_cast<const int2 *>(orig_edges);
        long long msrc = round_stream == 0 ? m_cur : m_orig;
        const long long *map = reinterpret_cast<const long long *>(round_stream == 0 ? rep : node_lab);
        unsigned tiles = (unsigned)((msrc + RTILE - 1) / RTILE);
        if (tiles == 0) tiles = 1;
        auto *status = sc.alloc<unsigned long long>(tiles);
        auto *ctr = sc.alloc<unsigned>(1);
        auto *dcount = sc.alloc<unsigned long long>(1);
        CVZ_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * tiles, s));
        CVZ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
        CVZ_CUDA(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), s));
        CVZ_LAUNCH(relabel_compact_kernel, tiles, TB, 0, s, src, msrc, map,
                   reinterpret_cast<int2 *>(next_edges), LookbackState{status, ctr}, dcount, tiles);
        unsigned long long hm = 0;
        CVZ_CUDA(cudaMemcpyAsync(&hm, dcount, sizeof(hm), cudaMemcpyDeviceToHost, s));
        CVZ_CUDA(cudaStreamSynchronize(s));
        *next_m = (int64_t)hm;
    });
}

}  // extern "C"
