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
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"

namespace cvz {
namespace cg = cooperative_groups;
namespace {

constexpr int TB = 256;
// fast mode: edges in flight <= m / FAST_WINDOW_DIV (m / FAST_WINDOW_DIV_SMALL
// below 2^20 edges: at C1 (99K edges) a 774-edge window spread the top-10
// community share over 0.35-0.56 across runs, past the reference's own
// 0.34-0.51 envelope; the 256-edge floor keeps it at 0.34-0.46.  Large
// streams keep full occupancy -- 0.8 % of m in flight stays within the
// envelope there and the window does not change their time)
constexpr long long FAST_WINDOW_DIV = 128;
constexpr long long FAST_WINDOW_DIV_SMALL = 512;


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

// Slot keys in stream order, with the slots that can never matter dropped
// on the fly (stable, single pass, decoupled look-back): the second slot of a
// self-loop (its counter is bumped once) and slots of nodes whose seeded
// counter already exceeds T (they can neither change nor merge).  Every
// dropped slot keeps counter T+1 (inactive).
constexpr int SITEMS = 4;
constexpr int STILE = TB * SITEMS;

__global__ void __launch_bounds__(TB) slot_keys_kernel(
    const int2 *__restrict__ E, long long m, const long long *__restrict__ d0, long long T,
    unsigned *__restrict__ keys, unsigned *__restrict__ vals, LookbackState st,
    unsigned long long *__restrict__ d_count, unsigned num_tiles) {
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_prefix;
    const unsigned tile = acquire_tile(st, &s_tile);
    const long long base = (long long)tile * STILE;
    int2 e[SITEMS];
    bool ku[SITEMS], kv[SITEMS];
#pragma unroll
    for (int j = 0; j < SITEMS; ++j) {
        long long k = base + (long long)j * TB + threadIdx.x;
        ku[j] = kv[j] = false;
        if (k < m) {
            int2 p = __ldg(E + k);
            e[j] = p;
            ku[j] = !d0 || __ldg(d0 + p.x) <= T;
            kv[j] = p.x != p.y && (!d0 || __ldg(d0 + p.y) <= T);
        }
    }
    constexpr int NW = TB / 32;
    __shared__ unsigned s_cnt[SITEMS * NW];
    __shared__ unsigned s_total;
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned woff[SITEMS];
#pragma unroll
    for (int j = 0; j < SITEMS; ++j) {  // warp-inclusive scan of the 0..2 live slots
        unsigned c = ku[j] + kv[j], x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        woff[j] = x - c;
        if (lane == 31) s_cnt[j * NW + wid] = x;
    }
    __syncthreads();
    if (wid == 0) {
        static_assert(SITEMS * NW == 32, "scan below covers 32 entries");
        unsigned v = s_cnt[lane], x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        s_cnt[lane] = x - v;
        if (lane == 31) s_total = x;
    }
    __syncthreads();
    const unsigned total = s_total;
    unsigned long long prefix = tile_prefix(st, tile, (unsigned long long)total, &s_prefix);
#pragma unroll
    for (int j = 0; j < SITEMS; ++j) {
        long long k = base + (long long)j * TB + threadIdx.x;
        long long w = (long long)prefix + s_cnt[j * NW + wid] + woff[j];
        if (ku[j]) {
            keys[w] = (unsigned)e[j].x;
            vals[w] = (unsigned)(2 * k);
            ++w;
        }
        if (kv[j]) {
            keys[w] = (unsigned)e[j].y;
            vals[w] = (unsigned)(2 * k + 1);
        }
    }
    if (threadIdx.x == 0 && tile == num_tiles - 1) *d_count = prefix + total;
}

// First-round slot keys: slot 2k = u, 2k+1 = v (sentinel n for the second
// slot of a self-loop: it is bumped once, C/community.py:104-109), values =
// slot ids.  Two edges per 128-bit load, two 128-bit stores per array.
__global__ void slot_keys_direct_kernel(const int4 *__restrict__ E2, const int2 *__restrict__ E,
                                        long long m, unsigned n, unsigned *__restrict__ keys,
                                        unsigned *__restrict__ vals) {
    const long long pairs = m / 2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < pairs;
         i += (long long)gridDim.x * blockDim.x) {
        const int4 p = __ldcs(E2 + i);  // edges 2i, 2i+1
        const unsigned s0 = (unsigned)(4 * i);
        reinterpret_cast<uint4 *>(keys)[i] =
            make_uint4((unsigned)p.x, p.x == p.y ? n : (unsigned)p.y, (unsigned)p.z,
                       p.z == p.w ? n : (unsigned)p.w);
        reinterpret_cast<uint4 *>(vals)[i] = make_uint4(s0, s0 + 1, s0 + 2, s0 + 3);
    }
    if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int2 p = E[m - 1];
        keys[2 * (m - 1)] = (unsigned)p.x;
        keys[2 * (m - 1) + 1] = p.x == p.y ? n : (unsigned)p.y;
        vals[2 * (m - 1)] = (unsigned)(2 * (m - 1));
        vals[2 * (m - 1) + 1] = (unsigned)(2 * (m - 1) + 1);
    }
}

template <class CT>
__global__ void fill_kernel(CT *__restrict__ a, long long len, CT v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len;
         i += (long long)gridDim.x * blockDim.x)
        a[i] = v;
}

// four sorted keys per thread (one 16-byte load; the neighbours across the
// group edges come from two scalar loads that hit L1/L2)
__global__ void seg_bounds_kernel(const unsigned *__restrict__ key, long long ns, unsigned n,
                                  int *__restrict__ seg_start, int *__restrict__ seg_end) {
    const long long groups = (ns + 3) / 4;
    for (long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x; gi < groups;
         gi += (long long)gridDim.x * blockDim.x) {
        const long long i0 = 4 * gi;
        unsigned k[6];  // k[0] = key[i0 - 1], k[1..4] = key[i0..i0+3], k[5] = key[i0 + 4]
        if (i0 + 4 <= ns) {
            const uint4 v = reinterpret_cast<const uint4 *>(key)[gi];
            k[1] = v.x;
            k[2] = v.y;
            k[3] = v.z;
            k[4] = v.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) k[1 + q] = i0 + q < ns ? key[i0 + q] : 0xffffffffu;
        }
        k[0] = i0 > 0 ? key[i0 - 1] : 0xffffffffu;
        k[5] = i0 + 4 < ns ? key[i0 + 4] : 0xffffffffu;
#pragma unroll
        for (int q = 1; q <= 4; ++q) {
            const long long i = i0 + q - 1;
            const unsigned x = k[q];
            if (i >= ns || x >= n) continue;
            if (i == 0 || k[q - 1] != x) seg_start[x] = (int)i;
            if (i == ns - 1 || k[q + 1] != x) seg_end[x] = (int)(i + 1);
        }
    }
}

// 4 slots per thread with the seg_start / d0 gathers issued together: the
// per-slot chain (key -> seg_start[key] -> store) is gather-latency-bound
constexpr int SCITEMS = 4;
template <class CT>
__global__ void slot_counter_kernel(const unsigned *__restrict__ key,
                                    const unsigned *__restrict__ val, long long ns, unsigned n,
                                    const int *__restrict__ seg_start,
                                    const long long *__restrict__ d0, long long T,
                                    CT *__restrict__ cval) {
    const long long stride = (long long)gridDim.x * blockDim.x * SCITEMS;
    for (long long i0 = (long long)blockIdx.x * blockDim.x * SCITEMS + threadIdx.x; i0 < ns;
         i0 += stride) {
        unsigned x[SCITEMS], sv[SCITEMS];
        int st[SCITEMS];
        long long d[SCITEMS];
#pragma unroll
        for (int j = 0; j < SCITEMS; ++j) {
            long long i = i0 + (long long)j * blockDim.x;
            x[j] = i < ns ? key[i] : n;
            sv[j] = i < ns ? val[i] : 0u;
        }
#pragma unroll
        for (int j = 0; j < SCITEMS; ++j) {
            st[j] = x[j] < n ? seg_start[x[j]] : 0;
            d[j] = (d0 && x[j] < n) ? d0[x[j]] : 0;
        }
#pragma unroll
        for (int j = 0; j < SCITEMS; ++j) {
            long long i = i0 + (long long)j * blockDim.x;
            if (i >= ns) continue;
            if (x[j] >= n) continue;  // sentinel slot: T + 1 prefill
            long long r = i - st[j] + 1;
            long long c = d[j] + r;  // d <= T here (larger seeds were dropped)
            if (c <= T) cval[sv[j]] = (CT)c;  // saturated slots keep the T + 1 prefill
        }
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
    // 4 slots per thread, role[] gathers issued together (latency-bound)
    const long long stride = (long long)gridDim.x * blockDim.x * SCITEMS;
    for (long long i0 = (long long)blockIdx.x * blockDim.x * SCITEMS + threadIdx.x; i0 < ns;
         i0 += stride) {
        unsigned x[SCITEMS], sv[SCITEMS], nx[SCITEMS];
        signed char r[SCITEMS];
#pragma unroll
        for (int j = 0; j < SCITEMS; ++j) {
            long long i = i0 + (long long)j * blockDim.x;
            x[j] = i < ns ? key[i] : n;
            sv[j] = i < ns ? val[i] : 0u;
            nx[j] = (i + 1 < ns) ? key[i + 1] : n;
        }
#pragma unroll
        for (int j = 0; j < SCITEMS; ++j) r[j] = x[j] < n ? role[sv[j] >> 1] : (signed char)-1;
#pragma unroll
        for (int j = 0; j < SCITEMS; ++j) {
            long long i = i0 + (long long)j * blockDim.x;
            if (i >= ns || x[j] >= n) continue;
            const int k = (int)(sv[j] >> 1);
            if (r[j] >= 0 && r[j] != (signed char)(sv[j] & 1)) parent[k] = lastw[i];  // source
            if (i == ns - 1 || nx[j] != x[j]) finalw[x[j]] = lastw[i];
        }
    }
}

constexpr long long DIRECT_PARENTS_MAX_T = 64;

// Parents without a segmented scan.  Writes to node x happen only at its
// active slots -- the first b = T - d0(x) of its segment (a later slot's
// post-increment counter exceeds T) -- and the sorted segment lists them in
// stream order.  So the last write before an active source slot i is found
// by scanning back at most b - 1 slots, and x's final write among its (at
// most b) active slots; every other slot does nothing.  Same results as the
// inclusive "last write so far" scan over all slots it replaces.
__global__ void direct_parents_kernel(const unsigned *__restrict__ key,
                                      const unsigned *__restrict__ val, long long ns, unsigned n,
                                      const int *__restrict__ seg_start,
                                      const int *__restrict__ seg_end,
                                      const long long *__restrict__ d0, long long T,
                                      const signed char *__restrict__ role,
                                      int *__restrict__ parent, int *__restrict__ finalw) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ns;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned x = key[i];
        if (x >= n) continue;
        const int st = seg_start[x];
        const long long b = T - (d0 ? d0[x] : 0);  // active slots of x
        if (i - st >= b) continue;
        const unsigned s = val[i];
        const int k = (int)(s >> 1);
        const signed char ro = role[k];
        if (ro >= 0 && ro != (signed char)(s & 1)) {  // event k reads x's label here
            int p = -1;
            for (long long j = i - 1; j >= st; --j) {
                const unsigned sj = val[j];
                if (role[sj >> 1] == (signed char)(sj & 1)) {
                    p = (int)(sj >> 1);
                    break;
                }
            }
            parent[k] = p;
        }
        const long long last_active = min((long long)seg_end[x], (long long)st + b) - 1;
        if (i == last_active) {  // x's final label comes from its last write
            int fw = -1;
            for (long long j = i; j >= st; --j) {
                const unsigned sj = val[j];
                if (role[sj >> 1] == (signed char)(sj & 1)) {
                    fw = (int)(sj >> 1);
                    break;
                }
            }
            finalw[x] = fw;
        }
    }
}

// Same results, one pass per node: the thread holding a segment's first
// slot walks x's (<= b <= T) active slots forward, carrying the last write,
// so each active slot's role is read once (the per-slot kernel above
// rescans up to b - 1 predecessors for every reading slot).
constexpr int DP_BATCH = 8;
// One thread per node: seg_start[x] is only written for nodes that have
// slots this round, so it is validated against the sorted keys (in range,
// key[st] == x, key[st - 1] != x) before use.
__global__ void node_parents_kernel(const unsigned *__restrict__ key,
                                    const unsigned *__restrict__ val, long long ns, unsigned n,
                                    const int *__restrict__ seg_start,
                                    const int *__restrict__ seg_end,
                                    const long long *__restrict__ d0, long long T,
                                    const signed char *__restrict__ role,
                                    int *__restrict__ parent, int *__restrict__ finalw) {
    for (unsigned x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        const long long i = seg_start[x];
        if (i < 0 || i >= ns || key[i] != x || (i > 0 && key[i - 1] == x)) continue;
        const long long b = T - (d0 ? d0[x] : 0);
        const long long end = min((long long)seg_end[x], i + b);
        if (end <= i) continue;
        int last = -1;
        for (long long j0 = i; j0 < end; j0 += DP_BATCH) {
            unsigned sv[DP_BATCH];
            signed char ro[DP_BATCH];
#pragma unroll
            for (int q = 0; q < DP_BATCH; ++q) sv[q] = j0 + q < end ? val[j0 + q] : 0u;
#pragma unroll
            for (int q = 0; q < DP_BATCH; ++q) ro[q] = j0 + q < end ? role[sv[q] >> 1] : -1;
#pragma unroll
            for (int q = 0; q < DP_BATCH; ++q) {
                const signed char e = (signed char)(sv[q] & 1);
                if (ro[q] >= 0 && ro[q] != e) parent[sv[q] >> 1] = last;  // event reads x
                if (ro[q] == e) last = (int)(sv[q] >> 1);                 // event writes x
            }
        }
        finalw[x] = last;
    }
}

// events: origin[k] = node whose initial label event k carries (-1 pending)
// EI_ITEMS events per thread per sweep (block-uniform trip count): the
// worklist append costs one block scan + one atomic per EI_ITEMS * TB
// events, and each thread's role / edge / parent loads are issued together
constexpr int EI_ITEMS = 8;
__global__ void events_init_kernel(const int2 *__restrict__ E, long long m,
                                   const signed char *__restrict__ role,
                                   const int *__restrict__ parent, int *__restrict__ origin,
                                   int *__restrict__ ptr, int *__restrict__ work,
                                   unsigned *__restrict__ nwork) {
    const long long stride = (long long)gridDim.x * blockDim.x * EI_ITEMS;
    __shared__ unsigned s_wcnt[TB / 32], s_base;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    for (long long k0 = (long long)blockIdx.x * blockDim.x * EI_ITEMS; k0 < m; k0 += stride) {
        signed char r[EI_ITEMS];
#pragma unroll
        for (int j = 0; j < EI_ITEMS; ++j) {
            const long long k = k0 + (long long)j * blockDim.x + threadIdx.x;  // coalesced
            r[j] = k < m ? role[k] : (signed char)-1;
        }
        int2 p[EI_ITEMS];
        int par[EI_ITEMS];
#pragma unroll
        for (int j = 0; j < EI_ITEMS; ++j) {
            const long long k = k0 + (long long)j * blockDim.x + threadIdx.x;
            if (r[j] >= 0) {
                p[j] = __ldg(E + k);
                par[j] = parent[k];
            }
        }
        unsigned pmask = 0;
#pragma unroll
        for (int j = 0; j < EI_ITEMS; ++j) {
            const long long k = k0 + (long long)j * blockDim.x + threadIdx.x;
            if (r[j] < 0) continue;
            const int src = r[j] == 0 ? p[j].y : p[j].x;
            if (par[j] < 0) {
                origin[k] = src;
            } else {
                origin[k] = -1;
                ptr[k] = par[j];
                pmask |= 1u << j;
            }
        }
        // one worklist atomic per block and sweep (a per-warp atomic on the
        // single counter serialised ~1M warps in round 1 at C4)
        unsigned bal[EI_ITEMS], mine = 0;
#pragma unroll
        for (int j = 0; j < EI_ITEMS; ++j) {
            bal[j] = __ballot_sync(0xffffffffu, (pmask >> j) & 1u);
            mine += __popc(bal[j]);
        }
        if (lane == 0) s_wcnt[wid] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned tot = 0;
            for (int w = 0; w < TB / 32; ++w) {
                unsigned c = s_wcnt[w];
                s_wcnt[w] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(nwork, tot) : 0;
        }
        __syncthreads();
        unsigned base = s_base + s_wcnt[wid];
#pragma unroll
        for (int j = 0; j < EI_ITEMS; ++j) {
            const long long k = k0 + (long long)j * blockDim.x + threadIdx.x;
            if ((pmask >> j) & 1u) work[base + __popc(bal[j] & ((1u << lane) - 1))] = (int)k;
            base += __popc(bal[j]);
        }
        __syncthreads();
    }
}

// Pointer jumping runs as ONE cooperative launch instead of a launch + host
// round trip per sweep: grid-wide sweeps separated by grid barriers while
// the worklist is large, then block 0 alone (block barriers, ~100x cheaper
// than a grid barrier) once it is at most SMALL_LIST long.  counts[r] =
// worklist length before sweep r (counts[0] set by the init step, the rest
// zeroed by the caller; R + 1 entries).
constexpr unsigned SMALL_LIST = 2048;
constexpr int CB = 512;  // cooperative-kernel block size

// Worklist length after a barrier: one plain L2 load per warp (an atomic
// read here would serialise every thread of the grid on one address).
__device__ __forceinline__ unsigned ld_count(const unsigned *c) {
    return *reinterpret_cast<const volatile unsigned *>(c);
}

// Worklist compaction with one atomic per block: every thread of the block
// must call it (block-uniform trip counts).  Per-warp atomics would put
// ~n/32 serialised updates on one counter for a multi-million worklist.
__device__ __forceinline__ void push_compact_block(bool keep, int v, unsigned *counter,
                                                   int *out) {
    __shared__ unsigned s_w[32];
    __shared__ unsigned s_base;
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    const int wid = threadIdx.x >> 5;
    if (lane_id() == 0) s_w[wid] = __popc(mask);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            unsigned c = s_w[w];
            s_w[w] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(counter, tot) : 0;
    }
    __syncthreads();
    if (keep) out[s_base + s_w[wid] + __popc(mask & ((1u << lane_id()) - 1))] = v;
    __syncthreads();
}

// event values: origin[k] = node whose initial label event k carries; a
// pending event follows its parent chain (parents are earlier events, so
// chains end and there are no cycles).
__global__ void events_coop_kernel(int *__restrict__ wa, int *__restrict__ wb,
                                   unsigned *__restrict__ counts, int R, int *origin, int *ptr) {
    cg::grid_group grid = cg::this_grid();
    int *cur = wa, *nxt = wb;
    bool single = false;
    for (int r = 0; r < R; ++r) {
        const unsigned cnt = ld_count(counts + r);
        if (cnt == 0) return;
        if (!single && cnt <= SMALL_LIST) {
            single = true;
            if (blockIdx.x != 0) return;
        }
        const unsigned start = single ? threadIdx.x : blockIdx.x * blockDim.x + threadIdx.x;
        const unsigned stride = single ? blockDim.x : gridDim.x * blockDim.x;
        const unsigned cc = (cnt + blockDim.x - 1) / blockDim.x * blockDim.x;
        for (unsigned t = start; t < cc; t += stride) {
            bool keep = false;
            int k = -1;
            if (t < cnt) {
                k = cur[t];
                int p = __ldcg(ptr + k);
                int op = __ldcg(origin + p);
                if (op >= 0) {
                    origin[k] = op;
                } else {
                    ptr[k] = __ldcg(ptr + p);
                    keep = true;
                }
            }
            push_compact_block(keep, k, counts + r + 1, nxt);
        }
        if (single)
            __syncthreads();
        else
            grid.sync();
        int *tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
}

// _resolve_labels (C/community.py:123-161): rep[x] = min id on the cycle
// reached from x.  Terminals -- fixed points (rep = x) and 2-cycle members
// (rep = min(x, f[x]); mutual adoptions make these common) -- are resolved
// at init.  Every other node pointer-doubles (p[x] = p[p[x]]) until p[x]
// lands on a node whose rep is already known (a terminal, or a node that
// retired earlier: retiring publishes rep[x]).  While tree nodes remain,
// every sweep retires at least one (the last remaining node on each path
// points at a published node), so a sweep that retires nobody, once 2^r >=
// remaining (every tail is shorter than that), leaves exactly the nodes that
// lead into >= 3-cycles with p[x] on their cycle; min-doubling over that
// f-closed set gives each cycle's minimum.  rep must start at -1.
__global__ void resolve_coop_kernel(const long long *__restrict__ lab, long long n,
                                    int *__restrict__ f, int *p, long long *rep,
                                    int *__restrict__ wa, int *__restrict__ wb,
                                    unsigned *__restrict__ counts, int R, int *__restrict__ mn_a,
                                    int *__restrict__ q_a, int *__restrict__ mn_b,
                                    int *__restrict__ q_b, int *__restrict__ bad) {
    cg::grid_group grid = cg::this_grid();
    const long long nn = (n + blockDim.x - 1) / blockDim.x * blockDim.x;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < nn;
         x += (long long)gridDim.x * blockDim.x) {
        if (x < n) {
            long long y = lab[x];
            if (y < 0 || y >= n) {
                atomicExch(bad, 1);
                y = x;
            }
            f[x] = (int)y;
            p[x] = (int)y;
        }
    }
    grid.sync();
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < nn;
         x += (long long)gridDim.x * blockDim.x) {
        bool pend = false;
        if (x < n) {
            int y = f[x];
            if (y == x)
                rep[x] = x;
            else if (f[y] == x)
                rep[x] = min((long long)y, x);  // 2-cycle
            else
                pend = true;
        }
        push_compact_block(pend, (int)x, counts, wa);
    }
    grid.sync();
    int *cur = wa, *nxt = wb;
    bool single = false;
    unsigned cnt = 0, prev = 0xffffffffu;
    for (int r = 0;; ++r) {
        cnt = ld_count(counts + r);
        if (cnt == 0) return;
        if (r == R || (cnt == prev && (r >= 31 || (1u << r) >= cnt))) break;
        if (!single && cnt <= SMALL_LIST) {
            single = true;
            if (blockIdx.x != 0) return;
        }
        const unsigned start = single ? threadIdx.x : blockIdx.x * blockDim.x + threadIdx.x;
        const unsigned stride = single ? blockDim.x : gridDim.x * blockDim.x;
        const unsigned cc = (cnt + blockDim.x - 1) / blockDim.x * blockDim.x;
        for (unsigned t = start; t < cc; t += stride) {
            bool keep = false;
            int x = -1;
            if (t < cnt) {
                x = cur[t];
                int y = __ldcg(p + x);
                long long ry = __ldcg(rep + y);
                if (ry >= 0) {
                    __stcg(rep + x, ry);  // retire + publish
                } else {
                    p[x] = __ldcg(p + y);
                    keep = true;
                }
            }
            push_compact_block(keep, x, counts + r + 1, nxt);
        }
        if (single)
            __syncthreads();
        else
            grid.sync();
        int *tmp = cur;
        cur = nxt;
        nxt = tmp;
        prev = cnt;
    }
    // >= 3-cycles: min-doubling over cur[0..cnt)
    if (!single && cnt <= SMALL_LIST) {
        single = true;
        if (blockIdx.x != 0) return;
    }
    const unsigned start = single ? threadIdx.x : blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned stride = single ? blockDim.x : gridDim.x * blockDim.x;
    int K = 1;
    while (K < 31 && (1u << (K + 1)) < cnt) ++K;  // window 2^(K+1) >= cnt >= cycle length
    for (unsigned t = start; t < cnt; t += stride) {
        int x = cur[t];
        mn_a[x] = min(x, f[x]);
        q_a[x] = f[f[x]];
    }
    if (single)
        __syncthreads();
    else
        grid.sync();
    for (int k = 0; k < K; ++k) {
        for (unsigned t = start; t < cnt; t += stride) {
            int x = cur[t];
            int y = q_a[x];
            mn_b[x] = min(mn_a[x], mn_a[y]);
            q_b[x] = q_a[y];
        }
        if (single)
            __syncthreads();
        else
            grid.sync();
        int *t1 = mn_a;
        mn_a = mn_b;
        mn_b = t1;
        int *t2 = q_a;
        q_a = q_b;
        q_b = t2;
    }
    for (unsigned t = start; t < cnt; t += stride) {
        int x = cur[t];
        rep[x] = mn_a[p[x]];
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

// ---- top-T formulation (T <= TOPT_MAX) -------------------------------------
// A node's active slots are its first b = T - d0 occurrences in stream order
// (a later post-increment counter exceeds T), so instead of sorting all 2m
// slots by node, every node keeps the b smallest slot ids in a sorted list
// of S = round_up(T, 4) <= TOPT_MAX entries.  Insertion is a lock-free atomicMin cascade: position
// i keeps the running minimum of everything that reached it and passes the
// larger value on, so position i ends as the (i+1)-th smallest slot
// whatever the interleaving.  Entries only decrease, so a slot larger than
// the current b-th entry can be rejected by a plain read, and the cascade may
// start at the first entry larger than the slot (earlier positions would
// pass it on unchanged).  Slots rejected or pushed past position b-1 set the
// node's overflow flag (counter T + 1).  With a roughly in-order stream most
// slots cost one sector read; the inserted ones one atomic.
constexpr int TOPT_MAX = 16;
constexpr unsigned TOPT_INF = 0xffffffffu;

// Packed per-node state of the top-b pass, one 8-byte word read per slot:
// bits 0-31 thr (see below), byte 4 the overflow flag, byte 5 the seed d0
// clipped to 255 (written once per round by topt_state_kernel).
__device__ __forceinline__ unsigned *st_thr(unsigned long long *st, int x) {
    return reinterpret_cast<unsigned *>(st + x);
}
__device__ __forceinline__ unsigned char *st_ovf_byte(unsigned long long *st, int x) {
    return reinterpret_cast<unsigned char *>(st + x) + 4;
}
__device__ __forceinline__ unsigned st_thr_of(unsigned long long w) { return (unsigned)w; }
__device__ __forceinline__ bool st_ovf(unsigned long long w) { return (w >> 32) & 0xff; }
__device__ __forceinline__ int st_d8(unsigned long long w) { return (int)((w >> 40) & 0xff); }

__global__ void topt_state_kernel(long long n, const long long *__restrict__ d0,
                                  unsigned long long *__restrict__ st) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        const long long d = d0 ? d0[x] : 0;
        const unsigned long long d8 = (unsigned long long)(d < 0 ? 0 : (d > 255 ? 255 : d));
        st[x] = (unsigned long long)TOPT_INF | (d8 << 40);
    }
}

// thr[x] >= the current b-th entry of x's list (an upper bound that only
// decreases): a slot above it is not among x's b smallest -- one read of a
// 4-byte-per-node array rejects most slots without touching the list.  ovf
// is written only if it is not set yet (a node's later occurrences would
// otherwise store to the same byte again and again).
//
// Continue the cascade of v from position i (old = the value it displaced
// there, already known not to be TOPT_INF).
__device__ __noinline__ void topt_cascade(unsigned *__restrict__ A, int i, int b, unsigned v,
                                          unsigned old, unsigned long long *__restrict__ st,
                                          int x) {
    v = max(old, v);
    for (++i; i < b; ++i) {
        old = atomicMin(A + i, v);
        if (i == b - 1) atomicMin(st_thr(st, x), min(old, v));
        if (old == TOPT_INF) return;
        v = max(old, v);
    }
    if (!st_ovf(__ldcg(st + x))) *st_ovf_byte(st, x) = 1;  // the largest of b + 1 falls off
}

// one thread per pair of edges (one 128-bit load), this launch's nodes in
// [xlo, xhi); slot 2k = u, 2k+1 = v, the second slot of a self-loop is not a
// slot (bumped once, C/community.py:104-109); nodes whose seed exceeds T
// have no active slot.  Per iteration the four slots' dependent chains are
// issued phase by phase (threshold + overflow reads, list reads, first
// atomics) so their L2 round trips overlap, and the next pair is prefetched.
template <int S>  // list stride: 4, 8, 12 or 16 entries
__global__ void __launch_bounds__(TB, 6) topt_kernel(const int4 *__restrict__ E2, const int2 *__restrict__ E, long long m,
                            long long T, unsigned *__restrict__ list,
                            unsigned long long *__restrict__ st, int xlo, int xhi) {
    const long long pairs = (m + 1) / 2;
    const long long W = (long long)gridDim.x * blockDim.x;
    auto load = [&](long long i, int (&x)[4]) {
        if (i >= pairs) {
            x[0] = x[1] = x[2] = x[3] = -1;
            return;
        }
        if (2 * i + 1 < m && E2) {
            const int4 p = __ldcs(E2 + i);
            x[0] = p.x;
            x[1] = p.x == p.y ? -1 : p.y;
            x[2] = p.z;
            x[3] = p.z == p.w ? -1 : p.w;
        } else {
            const int2 p = __ldcs(E + 2 * i);
            x[0] = p.x;
            x[1] = p.x == p.y ? -1 : p.y;
            if (2 * i + 1 < m) {
                const int2 q = __ldcs(E + 2 * i + 1);
                x[2] = q.x;
                x[3] = q.x == q.y ? -1 : q.y;
            } else {
                x[2] = x[3] = -1;
            }
        }
    };
    int nx[4];
    load((long long)blockIdx.x * blockDim.x + threadIdx.x, nx);
    __shared__ unsigned s_qx[TB / 32][128], s_qv[TB / 32][128];
    __shared__ unsigned char s_qb[TB / 32][128];
    unsigned *qx = s_qx[threadIdx.x >> 5], *qv = s_qv[threadIdx.x >> 5];
    unsigned char *qb = s_qb[threadIdx.x >> 5];
    // warp-uniform trip count + __syncwarp per iteration: the inserts'
    // data-dependent branches would otherwise let the lanes of a warp drift
    // into different iterations (independent thread scheduling does not
    // reconverge them inside the loop: ncu showed 2.7 active lanes per
    // instruction)
    for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < pairs; i0 += W) {
        __syncwarp();
        const long long i = i0 + threadIdx.x;
        int x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = (nx[j] >= xlo && nx[j] < xhi) ? nx[j] : -1;
        load(i + W, nx);
        unsigned long long w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = x[j] >= 0 ? __ldcg(st + x[j]) : 0ull;
        int b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = x[j] < 0 ? -1 : (int)(T - st_d8(w[j]));
        // inserts are compacted across the warp (each lane's four slots ->
        // one shared queue) so the list read -> atomic chain runs once or
        // twice per lane per iteration instead of once per slot position
        // with the other lanes idle (four serialised phases per iteration)
        const int lane = lane_id();
        unsigned base = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned v = (unsigned)(4 * i + j);
            const bool ins = b[j] > 0 && st_thr_of(w[j]) >= v;
            // b == 0 (seed T): every occurrence overflows; b < 0: seed > T,
            // counter unchanged; a slot above the threshold overflows
            if (b[j] >= 0 && !ins && !st_ovf(w[j])) *st_ovf_byte(st, x[j]) = 1;
            const unsigned mk = __ballot_sync(0xffffffffu, ins);
            if (ins) {
                const unsigned q = base + __popc(mk & ((1u << lane) - 1));
                qx[q] = x[j];
                qv[q] = v;
                qb[q] = (unsigned char)b[j];
            }
            base += __popc(mk);
        }
        __syncwarp();
        // at most four entries per lane: list reads first, then the atomics
        unsigned ex[4], ev[4], eb[4], es[4];
        int ne = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const unsigned q = lane + 32u * r;
            if (q < base) {
                ex[r] = qx[q];
                ev[r] = qv[q];
                eb[r] = qb[q];
                ne = r + 1;
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r >= ne) break;
            const unsigned *A = list + (size_t)ex[r] * S;
            // the cascade may start at the first entry above v (earlier
            // entries are smaller and only decrease)
            int s0 = 0;
#pragma unroll
            for (int q = 0; q < S / 4; ++q) {
                const uint4 g = __ldcg(reinterpret_cast<const uint4 *>(A) + q);
                s0 += (g.x < ev[r]) + (g.y < ev[r]) + (g.z < ev[r]) + (g.w < ev[r]);
            }
            es[r] = (unsigned)min(s0, (int)eb[r] - 1);
        }
        unsigned old[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (r < ne) old[r] = atomicMin(list + (size_t)ex[r] * S + es[r], ev[r]);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r >= ne) break;
            if ((int)es[r] == (int)eb[r] - 1) atomicMin(st_thr(st, (int)ex[r]), min(old[r], ev[r]));
            if (old[r] != TOPT_INF)
                topt_cascade(list + (size_t)ex[r] * S, (int)es[r], (int)eb[r], ev[r], old[r], st,
                             (int)ex[r]);
        }
        __syncwarp();  // the queue is reused by the next iteration
    }
}

// per node: counters of its active slots (d0 + rank), everything else keeps
// the T + 1 prefill; then the parents / final write of the node as in
// node_parents_kernel, from the list instead of the sorted segment
template <class CT>
__global__ void topt_counters_kernel(long long n, int S, const unsigned *__restrict__ list,
                                     const unsigned long long *__restrict__ st, long long T,
                                     CT *__restrict__ cval) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        const long long d = st_d8(st[x]);
        if (d >= T) continue;
        const uint4 *A = reinterpret_cast<const uint4 *>(list + (size_t)x * S);
        const int b = (int)(T - d);
        for (int q = 0; q < (b + 3) / 4; ++q) {
            const uint4 v = A[q];
            const unsigned e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int r = 4 * q + j;
                if (r < b && e[j] != TOPT_INF) cval[e[j]] = (CT)(d + r + 1);
            }
            if (v.w == TOPT_INF) break;
        }
    }
}

__global__ void topt_parents_kernel(long long n, int S, const unsigned *__restrict__ list,
                                    const unsigned long long *__restrict__ st, long long T,
                                    const signed char *__restrict__ role,
                                    int *__restrict__ parent, int *__restrict__ finalw) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        const long long d = st_d8(st[x]);
        int last = -1;
        if (d < T) {
            const uint4 *A = reinterpret_cast<const uint4 *>(list + (size_t)x * S);
            const int b = (int)(T - d);
            for (int q = 0; q < (b + 3) / 4; ++q) {
                const uint4 v = A[q];
                const unsigned e[4] = {v.x, v.y, v.z, v.w};
                signed char ro[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    ro[j] = (4 * q + j < b && e[j] != TOPT_INF) ? role[e[j] >> 1] : (signed char)-2;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (ro[j] == -2) continue;
                    const signed char side = (signed char)(e[j] & 1);
                    if (ro[j] >= 0 && ro[j] != side) parent[e[j] >> 1] = last;  // event reads x
                    if (ro[j] == side) last = (int)(e[j] >> 1);                 // event writes x
                }
                if (v.w == TOPT_INF) break;
            }
        }
        finalw[x] = last;
    }
}

// final counter / label per node: deg = d0 if d0 > T, T + 1 on overflow,
// else d0 + (active slots); label = initial label of the last write's origin
__global__ void topt_finalize_kernel(long long n, int S, const unsigned *__restrict__ list,
                                     const unsigned long long *__restrict__ st,
                                     const int *__restrict__ finalw, const int *__restrict__ origin,
                                     const long long *__restrict__ d0,
                                     const long long *__restrict__ lab0, long long T,
                                     long long *__restrict__ deg_out,
                                     long long *__restrict__ lab_out) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        const unsigned long long w = st[x];
        // a seed above T leaves the counter unchanged: d0 itself (the clipped
        // byte is exact below 255)
        const long long d = st_d8(w) < 255 ? st_d8(w) : d0[x];
        long long deg = d;
        if (d <= T) {
            if (st_ovf(w)) {
                deg = T + 1;
            } else {
                const unsigned *A = list + (size_t)x * S;
                int c = 0;
                while (c < T - d && A[c] != TOPT_INF) ++c;
                deg = d + c;
            }
        }
        deg_out[x] = deg;
        const int fw = finalw[x];
        const long long src = fw >= 0 ? (long long)origin[fw] : x;
        lab_out[x] = lab0 ? lab0[src] : src;
    }
}

// ---- fast (racy) pass ------------------------------------------------------

// FU edges per thread in flight (grid-stride over the stream, W threads
// => FU * W edges in flight): the next edges are prefetched, and for all FU
// edges the counter checks, then the atomics, then the label loads are
// issued back to back so their L2 round trips overlap.  A counter that
// already reached T + 1 is not touched again (no atomic on saturated hubs).
// Labels: racy last-writer-wins (SPEC "benign races").
constexpr int FU = 2;

__global__ void __launch_bounds__(TB) fast_pass_kernel(const int2 *__restrict__ E, long long m,
                                                       const long long *__restrict__ d0,
                                                       long long T, int tie,
                                                       unsigned *__restrict__ cnt,
                                                       long long *lab) {
    const long long W = (long long)gridDim.x * blockDim.x;
    const long long k0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int2 nxt[FU];
#pragma unroll
    for (int u = 0; u < FU; ++u) {
        long long k = k0 + u * W;
        nxt[u] = k < m ? __ldcs(E + k) : make_int2(-1, -1);
    }
    for (long long kb = k0; kb < m; kb += FU * W) {
        int2 p[FU];
        long long du0[FU], dv0[FU];
#pragma unroll
        for (int u = 0; u < FU; ++u) {
            p[u] = nxt[u];
            long long kn = kb + (FU + u) * W;
            nxt[u] = kn < m ? __ldcs(E + kn) : make_int2(-1, -1);
        }
#pragma unroll
        for (int u = 0; u < FU; ++u) {
            const bool ok = p[u].x >= 0;
            du0[u] = (d0 && ok) ? __ldg(d0 + p[u].x) : 0;
            dv0[u] = (d0 && ok) ? __ldg(d0 + p[u].y) : 0;
        }
        bool nu[FU], nv[FU], au[FU], av[FU];
        unsigned cu[FU], cv[FU], ou[FU], ov[FU];
#pragma unroll
        for (int u = 0; u < FU; ++u) {
            const bool ok = p[u].x >= 0;
            nu[u] = ok && du0[u] <= T;
            nv[u] = ok && p[u].x != p[u].y && dv0[u] <= T;
            cu[u] = nu[u] ? __ldcg(cnt + p[u].x) : 0u;
            cv[u] = nv[u] ? __ldcg(cnt + p[u].y) : 0u;
        }
#pragma unroll
        for (int u = 0; u < FU; ++u) {
            au[u] = nu[u] && (long long)cu[u] < T + 1 - du0[u];
            av[u] = nv[u] && (long long)cv[u] < T + 1 - dv0[u];
            ou[u] = au[u] ? atomicAdd(cnt + p[u].x, 1u) : 0u;
            ov[u] = av[u] ? atomicAdd(cnt + p[u].y, 1u) : 0u;
        }
        int tgt[FU], src[FU];
#pragma unroll
        for (int u = 0; u < FU; ++u) {
            tgt[u] = -1;
            if (p[u].x < 0 || p[u].x == p[u].y) continue;
            const long long du =
                !nu[u] ? du0[u] : (au[u] ? min(du0[u] + (long long)ou[u] + 1, T + 1) : T + 1);
            const long long dv =
                !nv[u] ? dv0[u] : (av[u] ? min(dv0[u] + (long long)ov[u] + 1, T + 1) : T + 1);
            if (du > T || dv > T) continue;  // C/community.py:110-111
            if (du < dv || (du == dv && tie == 0)) {  // :112-113, :116-117
                tgt[u] = p[u].x;
                src[u] = p[u].y;
            } else if (dv < du || (du == dv && tie == 1)) {  // :114-115, :118-119
                tgt[u] = p[u].y;
                src[u] = p[u].x;
            }
        }
        long long val[FU];
#pragma unroll
        for (int u = 0; u < FU; ++u)
            if (tgt[u] >= 0) val[u] = __ldcg(lab + src[u]);
#pragma unroll
        for (int u = 0; u < FU; ++u)
            if (tgt[u] >= 0) __stcg(lab + tgt[u], val[u]);
    }
}

// North-star form of the racy pass: two edges per 128-bit load and
// warp-aggregated counter atomics -- lanes bumping the same node are
// grouped with __match_any_sync, the lowest one adds the group size, and
// each member takes old + (its rank in the group) + 1, i.e. the group's
// increments in lane order (one valid interleaving of the racy pass).  The
// four endpoint positions of a thread are aggregated one after the other.
// Warp-uniform trip counts (match_any needs every lane).
__global__ void __launch_bounds__(TB) fast_pass4_kernel(const int4 *__restrict__ E2,
                                                        const int2 *__restrict__ E, long long m,
                                                        const long long *__restrict__ d0,
                                                        long long T, int tie,
                                                        unsigned *__restrict__ cnt,
                                                        long long *lab) {
    const long long W = (long long)gridDim.x * blockDim.x;
    const long long pairs = (m + 1) / 2;
    const int lane = lane_id();
    const unsigned lt = (1u << lane) - 1;
    auto load = [&](long long j, int (&x)[4]) {
        if (j >= pairs) {
            x[0] = x[1] = x[2] = x[3] = -1;
        } else if (E2 && 2 * j + 1 < m) {
            const int4 p = __ldcs(E2 + j);
            x[0] = p.x;
            x[1] = p.y;
            x[2] = p.z;
            x[3] = p.w;
        } else {
            const int2 a = __ldcs(E + 2 * j);
            x[0] = a.x;
            x[1] = a.y;
            if (2 * j + 1 < m) {
                const int2 b = __ldcs(E + 2 * j + 1);
                x[2] = b.x;
                x[3] = b.y;
            } else {
                x[2] = x[3] = -1;
            }
        }
    };
    int nx[4];
    load((long long)blockIdx.x * blockDim.x + threadIdx.x, nx);
    for (long long jb = (long long)blockIdx.x * blockDim.x; jb < pairs; jb += W) {
        int x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = nx[q];
        load(jb + W + threadIdx.x, nx);
        long long d[4];
        bool need[4], live[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // the second slot of a self-loop is not bumped (C/community.py:104-109)
            live[q] = x[q] >= 0 && !((q & 1) && x[q] == x[q - 1]);
            d[q] = (d0 && live[q]) ? __ldg(d0 + x[q]) : 0;
        }
        unsigned c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            need[q] = live[q] && d[q] <= T;
            c[q] = need[q] ? __ldcg(cnt + x[q]) : 0u;
        }
        long long dd[4];  // post-increment counter of each slot
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool a = need[q] && (long long)c[q] < T + 1 - d[q];
            unsigned o = 0;
            if (__ballot_sync(0xffffffffu, a)) {  // no bumping lane: no match / atomic
                const unsigned key = a ? (unsigned)x[q] : (0x80000000u | (unsigned)lane);
                const unsigned peers = __match_any_sync(0xffffffffu, key);
                const int leader = __ffs(peers) - 1;
                unsigned old = 0;
                if (a && lane == leader) old = atomicAdd(cnt + x[q], (unsigned)__popc(peers));
                old = __shfl_sync(0xffffffffu, old, leader);
                o = old + __popc(peers & lt);
            }
            dd[q] = !need[q] ? d[q] : (a ? min(d[q] + (long long)o + 1, T + 1) : T + 1);
        }
        int tgt[2], src[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            tgt[u] = -1;
            const int a = x[2 * u], b = x[2 * u + 1];
            if (a < 0 || a == b) continue;
            const long long du = dd[2 * u], dv = dd[2 * u + 1];
            if (du > T || dv > T) continue;  // C/community.py:110-111
            if (du < dv || (du == dv && tie == 0)) {  // :112-113, :116-117
                tgt[u] = a;
                src[u] = b;
            } else if (dv < du || (du == dv && tie == 1)) {  // :114-115, :118-119
                tgt[u] = b;
                src[u] = a;
            }
        }
        long long val[2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (tgt[u] >= 0) val[u] = __ldcg(lab + src[u]);
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (tgt[u] >= 0) __stcg(lab + tgt[u], val[u]);
    }
}

__global__ void any_negative_kernel(const long long *__restrict__ v, long long n,
                                    int *__restrict__ flag) {
    bool neg = false;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        neg |= v[i] < 0;
    if (__any_sync(0xffffffffu, neg) && lane_id() == 0) atomicExch(flag, 1);
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

// ---- round driver helpers --------------------------------------------------

__global__ void size_hist_kernel(const long long *__restrict__ node_lab, long long n,
                                 unsigned *__restrict__ size, const int *__restrict__ gate = nullptr) {
    if (gate && !*gate) return;  // detect round: labels unchanged, nothing follows
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

// 4 nodes per thread, loads issued before the dependent rep[] gathers: the
// kernel is gather-latency-bound (one node per thread left ~470 GB/s)
constexpr int CITEMS = 4;
__global__ void compose_kernel(long long n, const long long *__restrict__ rep,
                               long long *__restrict__ node_lab, long long *__restrict__ prev,
                               long long *__restrict__ hist, int check, int *__restrict__ changed) {
    bool diff = false;
    const long long stride = (long long)gridDim.x * blockDim.x * CITEMS;
    for (long long x0 = (long long)blockIdx.x * blockDim.x * CITEMS + threadIdx.x; x0 < n;
         x0 += stride) {
        long long l[CITEMS], v[CITEMS], pv[CITEMS];
#pragma unroll
        for (int j = 0; j < CITEMS; ++j) {
            long long x = x0 + (long long)j * blockDim.x;
            l[j] = x < n ? node_lab[x] : 0;
            pv[j] = (check && x < n) ? prev[x] : 0;
        }
#pragma unroll
        for (int j = 0; j < CITEMS; ++j) {
            long long x = x0 + (long long)j * blockDim.x;
            v[j] = x < n ? rep[l[j]] : 0;
        }
#pragma unroll
        for (int j = 0; j < CITEMS; ++j) {
            long long x = x0 + (long long)j * blockDim.x;
            if (x < n) {
                node_lab[x] = v[j];
                if (hist) hist[x] = v[j];
                if (check) diff |= pv[j] != v[j];
                prev[x] = v[j];
            }
        }
    }
    // one flag write per block (per-warp atomics on one word serialise)
    if (__syncthreads_or(diff) && threadIdx.x == 0) atomicExch(changed, 1);
}

// stable relabel + drop-intra compaction (single pass, decoupled look-back)
constexpr int RITEMS = 8;
constexpr int RTILE = TB * RITEMS;

// int32 relabel map (4-byte gathers; ids < 2^31): bit 31 = saturation flag
constexpr unsigned SAT_BIT = 0x80000000u;
constexpr unsigned SAT_MASK = SAT_BIT - 1;

// map[x] = rep[x] | SAT_BIT if rep[x]'s community has >= Tn + 2 members
// (size == nullptr: no flag)
__global__ void pack_map_kernel(const long long *__restrict__ rep, long long n,
                                const unsigned *__restrict__ size, long long Tn,
                                unsigned *__restrict__ out, const int *__restrict__ gate = nullptr) {
    if (gate && !*gate) return;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (long long)gridDim.x * blockDim.x) {
        const unsigned r = (unsigned)rep[x];
        out[x] = (size && (long long)size[r] >= Tn + 2) ? (r | SAT_BIT) : r;
    }
}

// Dead-edge drop (identity order, threshold pinned at its cap): an edge
// whose two communities both have >= Tn + 2 members is a no-op in every later
// round -- their seeded counters exceed Tn, so neither end can adopt, be
// adopted or change (C/community.py:104-120, :258-261), its relabelled ends
// stay equal to themselves, and sizes only grow.  Such edges are counted
// (*d_dead) instead of written.  size == nullptr disables the drop.
__global__ void __launch_bounds__(TB) relabel_compact_kernel(
    const int2 *__restrict__ in, long long m, const unsigned *__restrict__ map,
    int2 *__restrict__ out, LookbackState st, unsigned long long *__restrict__ d_count,
    unsigned num_tiles, bool drop, unsigned long long *__restrict__ d_dead,
    const int *__restrict__ gate = nullptr) {
    if (gate && !*gate) return;  // every CTA leaves: no tile waits on a predecessor
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_prefix;
    const unsigned tile = acquire_tile(st, &s_tile);
    const long long base = (long long)tile * RTILE;
    int2 p[RITEMS];
    bool keep[RITEMS];
    unsigned dead = 0;
#pragma unroll
    for (int j = 0; j < RITEMS; ++j) {
        long long i = base + (long long)j * TB + threadIdx.x;
        p[j] = i < m ? __ldcs(in + i) : make_int2(-1, -1);
    }
    int2 e[RITEMS];
#pragma unroll
    for (int j = 0; j < RITEMS; ++j) {
        keep[j] = false;
        if (p[j].x >= 0) {
            // map carries the saturation flag in bit 31 (pack_map_kernel)
            const unsigned ma = __ldg(map + p[j].x), mb = __ldg(map + p[j].y);
            const int a = (int)(ma & SAT_MASK), b = (int)(mb & SAT_MASK);
            e[j] = make_int2(a, b);
            keep[j] = a != b;
            if (drop && keep[j] && (ma & mb & SAT_BIT)) {
                keep[j] = false;
                ++dead;
            }
        }
    }
    if (drop) {
        for (int o = 16; o > 0; o >>= 1) dead += __shfl_xor_sync(0xffffffffu, dead, o);
        if (lane_id() == 0 && dead) atomicAdd(d_dead, (unsigned long long)dead);
    }
    // warp ballots -> per (item, warp) counts -> one 64-entry scan by warp 0:
    // two block barriers per tile instead of one block scan per item
    constexpr int NW = TB / 32;
    __shared__ unsigned s_cnt[RITEMS * NW];
    __shared__ unsigned s_total;
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned bal[RITEMS];
#pragma unroll
    for (int j = 0; j < RITEMS; ++j) {
        bal[j] = __ballot_sync(0xffffffffu, keep[j]);
        if (lane == 0) s_cnt[j * NW + wid] = __popc(bal[j]);
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the RITEMS * NW counts, PER consecutive per lane
        constexpr int PER = RITEMS * NW / 32;
        static_assert(PER * 32 == RITEMS * NW, "scan layout");
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
        unsigned run = x - v;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            s_cnt[PER * lane + q] = run;
            run += a[q];
        }
        if (lane == 31) s_total = x;
    }
    __syncthreads();
    const unsigned total = s_total;
    unsigned long long prefix = tile_prefix(st, tile, (unsigned long long)total, &s_prefix);
    const unsigned lt = (1u << lane) - 1;
#pragma unroll
    for (int j = 0; j < RITEMS; ++j) {
        if (keep[j]) out[prefix + s_cnt[j * NW + wid] + __popc(bal[j] & lt)] = e[j];
    }
    if (threadIdx.x == 0 && tile == num_tiles - 1) *d_count = prefix + total;
}

// Stable radix sort of (key, value) pairs in place over two buffer pairs
// (CUB DoubleBuffer: no extra copy pass -- 1.16 vs 1.76 ms for 65M pairs on
// B200).  Returns with *k / *v pointing at the sorted data.
template <class T>
void cub_sort_pairs_db(unsigned *&k, unsigned *kalt, T *&v, T *valt, long long ns, int end_bit,
                       Scratch &sc, cudaStream_t s) {
    cub::DoubleBuffer<unsigned> dk(k, kalt);
    cub::DoubleBuffer<T> dv(v, valt);
    size_t tb = 0;
    CVZ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)ns, 0, end_bit, s));
    void *tmp = sc.alloc<char>(tb);
    {
        CVZ_REGION("cub_sort:scoda_slots", s);
        CVZ_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)ns, 0, end_bit, s));
    }
    count_launches(1 + (end_bit + 7) / 8);
    k = dk.Current();
    v = dv.Current();
}

int bits_for_value(unsigned long long v) {  // bits to hold 0..v
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

}  // namespace

// Deterministic pass.  E: stream-ordered edges.  lab0/d0 nullable.
// CT = per-slot counter type: u8 whenever T + 1 < 256 (the 2m-slot counter
// array then stays L2-resident for the scattered writes), else int/int64.
template <class CT>
static void det_pass_t(const int2 *E, long long m, long long n, long long T, int tie,
                       const int64_t *d0, const int64_t *lab0, int64_t *deg_out,
                       int64_t *lab_out, Scratch &sc, cudaStream_t s) {
    const long long ns_all = 2 * m;
    auto *d0p = reinterpret_cast<const long long *>(d0);
    int *seg_start = sc.alloc<int>(n), *seg_end = sc.alloc<int>(n), *finalw = sc.alloc<int>(n);
    CVZ_CUDA(cudaMemsetAsync(seg_start, 0xff, sizeof(int) * n, s));
    CVZ_CUDA(cudaMemsetAsync(finalw, 0xff, sizeof(int) * n, s));
    int *origin = nullptr;
    if (m > 0) {
        // 1. live slots in stream order (dead ones dropped, see slot_keys_kernel)
        auto *keys = sc.alloc<unsigned>(ns_all), *vals = sc.alloc<unsigned>(ns_all);
        long long ns;
        if (!d0p && (reinterpret_cast<uintptr_t>(E) & 15) == 0) {
            // no seeds (first round): every slot is live except a self-loop's
            // second one, which gets the sentinel key n instead of being
            // dropped -- a plain streaming pass, no compaction
            ns = ns_all;
            CVZ_LAUNCH(slot_keys_direct_kernel, grid_for(m, TB, 2, 16), TB, 0, s,
                       reinterpret_cast<const int4 *>(E), E, m, (unsigned)n, keys, vals);
        } else {
            unsigned tiles = (unsigned)((m + STILE - 1) / STILE);
            auto *status = sc.alloc<unsigned long long>(tiles);
            auto *ctr = sc.alloc<unsigned>(1);
            auto *dcount = sc.alloc<unsigned long long>(1);
            CVZ_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * tiles, s));
            CVZ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
            CVZ_LAUNCH(slot_keys_kernel, tiles, TB, 0, s, E, m, d0p, T, keys, vals,
                       LookbackState{status, ctr}, dcount, tiles);
            unsigned long long hns = 0;
            read_small(&hns, dcount, sizeof(hns), s);
            ns = (long long)hns;
        }
        // 2. stable sort by node: each node's slots in stream order
        unsigned *skeys = keys, *svals = vals;
        if (ns > 0)
            cub_sort_pairs_db(skeys, sc.alloc<unsigned>(ns), svals, sc.alloc<unsigned>(ns), ns,
                              bits_for_value((unsigned long long)n), sc, s);
        CVZ_LAUNCH(seg_bounds_kernel, grid_for((ns + 3) / 4, TB, 1, 16), TB, 0, s, skeys, ns, (unsigned)n,
                   seg_start, seg_end);
        // 3. post-increment counters (dead slots: T + 1)
        CT *cval = sc.alloc<CT>(ns_all);
        if (sizeof(CT) == 1)
            CVZ_CUDA(cudaMemsetAsync(cval, (int)(T + 1), ns_all, s));
        else
            CVZ_LAUNCH(fill_kernel<CT>, grid_for(ns_all, TB, 1, 8), TB, 0, s, cval, ns_all,
                       (CT)(T + 1));
        CVZ_LAUNCH(slot_counter_kernel<CT>, grid_for(ns, TB, 1, 16), TB, 0, s, skeys, svals, ns,
                   (unsigned)n, seg_start, d0p, T, cval);
        auto *role = sc.alloc<signed char>(m);
        CVZ_LAUNCH(edge_role_kernel<CT>, grid_for(m, TB, 1, 16), TB, 0, s, E, m, cval, T, tie,
                   role);
        // 4. each event's parent = last earlier write to its source node: a
        //    bounded backward scan over the node's <= T active slots, or for
        //    large thresholds (quadratic scans) a segmented "last write so
        //    far" max-scan over all node-sorted slots
        int *parent = sc.alloc<int>(m);
        static const bool slot_parents = getenv("CVZ_PARENTS_SLOT") != nullptr;
        if (T <= DIRECT_PARENTS_MAX_T && !slot_parents) {
            CVZ_LAUNCH(node_parents_kernel, grid_for(n, TB, 1, 16), TB, 0, s, skeys, svals, ns,
                       (unsigned)n, seg_start, seg_end, d0p, T, role, parent, finalw);
        } else if (T <= DIRECT_PARENTS_MAX_T) {
            CVZ_LAUNCH(direct_parents_kernel, grid_for(ns, TB, 1, 16), TB, 0, s, skeys, svals, ns,
                       (unsigned)n, seg_start, seg_end, d0p, T, role, parent, finalw);
        } else {
            int *lastw = sc.alloc<int>(ns);
            if (ns > 0) {
                WriteVal wv{skeys, svals, role, (unsigned)n};
                auto vin = thrust::make_transform_iterator(thrust::counting_iterator<int>(0), wv);
                size_t tb = 0;
                CVZ_CUDA(cub::DeviceScan::InclusiveScanByKey(nullptr, tb, skeys, vin, lastw,
                                                             MaxOp(), (int)ns, cub::Equality(),
                                                             s));
                void *tmp = sc.alloc<char>(tb);
                CVZ_REGION("cub_scan_by_key:scoda_lastw", s);
                CVZ_CUDA(cub::DeviceScan::InclusiveScanByKey(tmp, tb, skeys, vin, lastw, MaxOp(),
                                                             (int)ns, cub::Equality(), s));
                count_launches(2);
            }
            CVZ_LAUNCH(parents_kernel, grid_for(ns, TB, 1, 16), TB, 0, s, skeys, svals, ns,
                       (unsigned)n, role, lastw, parent, finalw);
        }
        // 5. event values by pointer jumping (one cooperative launch)
        origin = sc.alloc<int>(m);
        int *ptr = sc.alloc<int>(m);
        int *wa = sc.alloc<int>(m), *wb = sc.alloc<int>(m);
        const int R = bits_for_value((unsigned long long)m) + 2;
        unsigned *cnt = sc.alloc<unsigned>(R + 1);
        CVZ_CUDA(cudaMemsetAsync(cnt, 0, (R + 1) * sizeof(unsigned), s));
        CVZ_LAUNCH(events_init_kernel, grid_for(m, TB, EI_ITEMS, 8), TB, 0, s, E, m, role, parent,
                   origin, ptr, wa, cnt);
        CVZ_COOP(events_coop_kernel, CB, s, wa, wb, cnt, R, origin, ptr);
        if (getenv("CVZ_DEBUG_RESOLVE")) {  // development aid: event worklist per sweep
            std::vector<unsigned> h(R + 1);
            read_small(h.data(), cnt, (R + 1) * sizeof(unsigned), s);
            fprintf(stderr, "events m=%lld live slots=%lld counts:", m, ns);
            for (unsigned v : h) fprintf(stderr, " %u", v);
            fprintf(stderr, "\n");
        }
    }
    if (!origin) origin = sc.alloc<int>(1);
    CVZ_LAUNCH(det_finalize_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n, seg_start, seg_end,
               finalw, origin, d0p, reinterpret_cast<const long long *>(lab0), T,
               reinterpret_cast<long long *>(deg_out), reinterpret_cast<long long *>(lab_out));
}

// Exactly the resident grid: iteration k of every thread covers one
// contiguous window of the stream, so slots arrive nearly in stream order and
// most inserts append (one atomic).  An oversubscribed grid-stride launch
// spreads the first wave over the whole stream, and random arrival order
// turns inserts into dependent atomic cascades.
template <int S>
static void launch_topt(const int4 *E2, const int2 *E, long long m, long long pairs, long long T,
                        unsigned *list, unsigned long long *st, int lo, int hi, cudaStream_t s) {
    static DeviceCache occ;
    const int per_sm = occ.get([] {
        int b = 0;
        CVZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, topt_kernel<S>, TB, 0));
        return b < 1 ? 1 : b;
    });
    const unsigned grid = (unsigned)std::max<long long>(
        1, std::min<long long>((long long)per_sm * num_sms(), (pairs + TB - 1) / TB));
    CVZ_LAUNCH(topt_kernel<S>, grid, TB, 0, s, E2, E, m, T, list, st, lo, hi);
}

// Deterministic pass, top-T formulation (T <= TOPT_MAX, see topt_insert):
// no slot sort; lists of the b smallest slot ids per node replace the
// sorted segments.  Same events, parents and results as det_pass_t.
static void det_pass_topt(const int2 *E, long long m, long long n, long long T, int tie,
                          const int64_t *d0, const int64_t *lab0, int64_t *deg_out,
                          int64_t *lab_out, Scratch &sc, cudaStream_t s) {
    auto *d0p = reinterpret_cast<const long long *>(d0);
    const int S = (int)std::max(4LL, (T + 3) & ~3LL);  // list stride: whole 16-byte groups
    unsigned *list = sc.alloc<unsigned>((size_t)n * S);
    auto *st = sc.alloc<unsigned long long>(n);
    int *finalw = sc.alloc<int>(n);
    int *origin = sc.alloc<int>(m > 0 ? m : 1);
    CVZ_CUDA(cudaMemsetAsync(list, 0xff, sizeof(unsigned) * (size_t)n * S, s));
    CVZ_LAUNCH(topt_state_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n, d0p, st);
    if (m > 0) {
        const bool al = (reinterpret_cast<uintptr_t>(E) & 15) == 0;
        // (one pass over the stream; splitting the nodes into L2-sized ranges
        // with one pass each measured slower: the pass is latency-, not
        // capacity-bound)
        const long long pairs = (m + 1) / 2;
        const int4 *E2 = al ? reinterpret_cast<const int4 *>(E) : nullptr;
        const int hi = (int)n;
        switch (S) {
            case 4: launch_topt<4>(E2, E, m, pairs, T, list, st, 0, hi, s); break;
            case 8: launch_topt<8>(E2, E, m, pairs, T, list, st, 0, hi, s); break;
            case 12: launch_topt<12>(E2, E, m, pairs, T, list, st, 0, hi, s); break;
            default: launch_topt<16>(E2, E, m, pairs, T, list, st, 0, hi, s); break;
        }
        unsigned char *cval = sc.alloc<unsigned char>(2 * m);
        CVZ_CUDA(cudaMemsetAsync(cval, (int)(T + 1), 2 * m, s));
        CVZ_LAUNCH(topt_counters_kernel<unsigned char>, grid_for(n, TB, 1, 8), TB, 0, s, n, S,
                   list, st, T, cval);
        auto *role = sc.alloc<signed char>(m);
        CVZ_LAUNCH(edge_role_kernel<unsigned char>, grid_for(m, TB, 1, 16), TB, 0, s, E, m, cval,
                   T, tie, role);
        int *parent = sc.alloc<int>(m);
        CVZ_LAUNCH(topt_parents_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n, S, list, st, T, role,
                   parent, finalw);
        int *ptr = sc.alloc<int>(m);
        int *wa = sc.alloc<int>(m), *wb = sc.alloc<int>(m);
        const int R = bits_for_value((unsigned long long)m) + 2;
        unsigned *cnt = sc.alloc<unsigned>(R + 1);
        CVZ_CUDA(cudaMemsetAsync(cnt, 0, (R + 1) * sizeof(unsigned), s));
        CVZ_LAUNCH(events_init_kernel, grid_for(m, TB, EI_ITEMS, 8), TB, 0, s, E, m, role, parent,
                   origin, ptr, wa, cnt);
        CVZ_COOP(events_coop_kernel, CB, s, wa, wb, cnt, R, origin, ptr);
    } else {
        CVZ_CUDA(cudaMemsetAsync(finalw, 0xff, sizeof(int) * n, s));
    }
    CVZ_LAUNCH(topt_finalize_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n, S, list, st, finalw, origin,
               d0p, reinterpret_cast<const long long *>(lab0), T,
               reinterpret_cast<long long *>(deg_out), reinterpret_cast<long long *>(lab_out));
}

// seeds_nonneg: every d0 >= 0 (the top-T lists hold at most TOPT_MAX = b
// entries only then; detect's size seeds always are)
void scoda_pass_dev(const int2 *E, long long m, long long n, long long T, int tie, int mode,
                    const int64_t *d0, const int64_t *lab0, int64_t *deg_out, int64_t *lab_out,
                    Scratch &sc, cudaStream_t s, bool seeds_nonneg) {
    CVZ_REQUIRE(2 * m < (1LL << 31) - 1, CVZ_ERR_VALUE,
                "edge stream too long for one pass (2m must be < 2^31)");
    if (mode == CVZ_SCODA_DETERMINISTIC) {
        // top-T lists for the usual small thresholds (CVZ_DET_SORT=1: the
        // slot-sort formulation for every T)
        static const bool force_sort = getenv("CVZ_DET_SORT") != nullptr;
        if (T >= 0 && T <= TOPT_MAX && !force_sort && (seeds_nonneg || !d0)) {
            det_pass_topt(E, m, n, T, tie, d0, lab0, deg_out, lab_out, sc, s);
            return;
        }
        // per-slot counters fit a byte only for non-negative seeds (a
        // caller's negative counter stays active below zero, C/community.py
        // :104-109, and must not wrap)
        const bool nonneg = seeds_nonneg || !d0;
        if (!nonneg)
            det_pass_t<long long>(E, m, n, T, tie, d0, lab0, deg_out, lab_out, sc, s);
        else if (T < 255)
            det_pass_t<unsigned char>(E, m, n, T, tie, d0, lab0, deg_out, lab_out, sc, s);
        else if (T < (1LL << 30))
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
        static const long long wenv =
            getenv("CVZ_FAST_WINDOW_DIV") ? std::max(1LL, atoll(getenv("CVZ_FAST_WINDOW_DIV"))) : 0;
        const long long wdiv =
            wenv ? wenv : (m < (1LL << 20) ? FAST_WINDOW_DIV_SMALL : FAST_WINDOW_DIV);
        long long window = std::max(256LL, std::min(m / wdiv, 2048LL * num_sms() * FU));
        unsigned blocks = (unsigned)((window / FU + TB - 1) / TB);
        // default: per-edge int2 loads and plain atomics (fast_pass_kernel);
        // CVZ_FAST_AGG=1: 128-bit loads + warp-aggregated atomics
        // (fast_pass4_kernel, measured slower at C4: 0.82 vs 0.70 ms --
        // in-warp duplicate nodes are rare in a shuffled stream, so the
        // match costs more than the atomics it saves)
        static const bool plain = getenv("CVZ_FAST_AGG") == nullptr;
        const bool al = (reinterpret_cast<uintptr_t>(E) & 15) == 0;
        if (plain)
            CVZ_LAUNCH(fast_pass_kernel, blocks, TB, 0, s, E, m,
                       reinterpret_cast<const long long *>(d0), T, tie, cnt,
                       reinterpret_cast<long long *>(lab_out));
        else
            CVZ_LAUNCH(fast_pass4_kernel, blocks, TB, 0, s,
                       al ? reinterpret_cast<const int4 *>(E) : nullptr, E, m,
                       reinterpret_cast<const long long *>(d0), T, tie, cnt,
                       reinterpret_cast<long long *>(lab_out));
    }
    CVZ_LAUNCH(fast_finalize_kernel, grid_for(n, TB, 1, 8), TB, 0, s, n, cnt,
               reinterpret_cast<const long long *>(d0), T, reinterpret_cast<long long *>(deg_out));
}

// rep[x] = min id on the cycle reached from lab[x] (C/community.py:123-161),
// one cooperative launch.  The range check (labels in [0, n)) synchronises
// only when check != 0.
void resolve_dev(const int64_t *lab, long long n, int64_t *rep_out, bool check, Scratch &sc,
                 cudaStream_t s) {
    if (n <= 0) return;
    int *f = sc.alloc<int>(n), *p = sc.alloc<int>(n);
    int *wa = sc.alloc<int>(n), *wb = sc.alloc<int>(n);
    int *mn_a = sc.alloc<int>(n), *q_a = sc.alloc<int>(n);
    int *mn_b = sc.alloc<int>(n), *q_b = sc.alloc<int>(n);
    const int R = bits_for_value((unsigned long long)n) + 2;  // 2^R >= 2n
    unsigned *cnt = sc.alloc<unsigned>(R + 1);
    int *bad = sc.alloc<int>(1);
    CVZ_CUDA(cudaMemsetAsync(cnt, 0, (R + 1) * sizeof(unsigned), s));
    CVZ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    CVZ_CUDA(cudaMemsetAsync(rep_out, 0xff, sizeof(int64_t) * n, s));
    CVZ_COOP(resolve_coop_kernel, CB, s, reinterpret_cast<const long long *>(lab), (long long)n,
             f, p, reinterpret_cast<long long *>(rep_out), wa, wb, cnt, R, mn_a, q_a, mn_b, q_b,
             bad);
    if (getenv("CVZ_DEBUG_RESOLVE")) {  // development aid: worklist length per sweep
        std::vector<unsigned> h(R + 1);
        read_small(h.data(), cnt, (R + 1) * sizeof(unsigned), s);
        fprintf(stderr, "resolve n=%lld counts:", n);
        for (unsigned v : h) fprintf(stderr, " %u", v);
        fprintf(stderr, "\n");
    }
    if (check) {
        int hbad = 0;
        read_small(&hbad, bad, sizeof(int), s);
        CVZ_REQUIRE(!hbad, CVZ_ERR_RANGE, "labels must lie in [0, n)");
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
        // caller-supplied counters may be negative: the top-T path only
        // when they are not (one reduction + a sync on this test seam)
        int *neg = sc.alloc<int>(1);
        CVZ_CUDA(cudaMemsetAsync(neg, 0, sizeof(int), s));
        CVZ_LAUNCH(any_negative_kernel, grid_for(n, TB, 1, 4), TB, 0, s,
                   reinterpret_cast<const long long *>(d0), (long long)n, neg);
        int hneg = 0;
        read_small(&hneg, neg, sizeof(int), s);
        scoda_pass_dev(E, m, n, threshold, tie_code, mode, d0, l0, deg, raw, sc, s, hneg == 0);
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
                     int64_t next_threshold, int64_t *next_dead, void *stream) {
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
        scoda_pass_dev(E, m_cur, n, T, tie_code, mode, d0, nullptr, deg_out, raw, sc, s, true);
        resolve_dev(raw, n, rep, false, sc, s);
        // 4. compose + history + early-stop test (:266-269).  The next
        //    stream is built right behind it, gated on the device by the
        //    changed flag (an unchanged round's kernels exit at once), so
        //    the round ends with ONE host read of {kept, dead, changed}.
        //    ctl: [0] kept edges, [1] dead edges, [2] changed (int)
        auto *ctl = sc.alloc<unsigned long long>(3);
        CVZ_CUDA(cudaMemsetAsync(ctl, 0, 3 * sizeof(unsigned long long), s));
        int *dchg = reinterpret_cast<int *>(ctl + 2);
        if (round_index == 1) CVZ_CUDA(cudaMemsetAsync(dchg, 1, 1, s));  // first round: changed
        CVZ_LAUNCH(compose_kernel, grid_for(n, TB, CITEMS, 8), TB, 0, s, (long long)n,
                   reinterpret_cast<const long long *>(rep), reinterpret_cast<long long *>(node_lab),
                   reinterpret_cast<long long *>(prev_lab),
                   reinterpret_cast<long long *>(history_out), round_index > 1 ? 1 : 0, dchg);
        const int *gate = round_index > 1 ? dchg : nullptr;
        // 5. next stream: contract (:272-278) or restream (:274-276)
        const int2 *src = round_stream == 0 ? cur : reinterpret_cast<const int2 *>(orig_edges);
        long long msrc = round_stream == 0 ? m_cur : m_orig;
        const int64_t *map64 = round_stream == 0 ? rep : node_lab;
        unsigned tiles = (unsigned)((msrc + RTILE - 1) / RTILE);
        if (tiles == 0) tiles = 1;
        auto *status = sc.alloc<unsigned long long>(tiles);
        auto *ctr = sc.alloc<unsigned>(1);
        unsigned long long *dcount = ctl;
        CVZ_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * tiles, s));
        CVZ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
        // next round's community sizes (what its seeding computes) for the
        // dead-edge drop; contract streams only (restream rebuilds each round)
        unsigned *nsize = nullptr;
        if (next_threshold >= 0 && round_stream == 0) {
            nsize = sc.alloc<unsigned>(n);
            CVZ_CUDA(cudaMemsetAsync(nsize, 0, sizeof(unsigned) * n, s));
            CVZ_LAUNCH(size_hist_kernel, grid_for(n, TB, 1, 8), TB, 0, s,
                       reinterpret_cast<const long long *>(node_lab), (long long)n, nsize, gate);
        }
        unsigned *map = sc.alloc<unsigned>(n);
        CVZ_LAUNCH(pack_map_kernel, grid_for(n, TB, 1, 8), TB, 0, s,
                   reinterpret_cast<const long long *>(map64), (long long)n, nsize,
                   (long long)next_threshold, map, gate);
        CVZ_LAUNCH(relabel_compact_kernel, tiles, TB, 0, s, src, msrc, map,
                   reinterpret_cast<int2 *>(next_edges), LookbackState{status, ctr}, dcount, tiles,
                   nsize != nullptr, dcount + 1, gate);
        unsigned long long hm[3] = {0, 0, 0};
        read_small(hm, ctl, sizeof(hm), s);
        const int hchg = (int)(unsigned)hm[2];  // the int in ctl[2]'s low word
        *changed = hchg != 0;
        *next_m = hchg ? (int64_t)hm[0] : 0;
        if (next_dead) *next_dead = hchg ? (int64_t)hm[1] : 0;
    });
}

}  // extern "C"
