// ForceAtlas2 with Barnes-Hut repulsion on B200 (fp64 throughout: B200 keeps
// half-rate FP64, and fp64 state keeps the layout within ~1e-13 of the
// reference per iteration).  Reference: C/layout.py:85-402.
//
// Tree.  The reference inserts bodies one by one into a quadtree whose cells
// hold <= 1 body (depth cap 40 -> aggregate cell).  That tree is canonical:
// its cells are exactly the quadrant prefixes (computed with the reference's
// own fp64 centre arithmetic, C/layout.py:118-137,171-208) shared by >= 2
// bodies.  Single-child chain cells never change a force (same body set,
// larger side), so the GPU builds the compressed tree:
//   keys  : per body, the 40 quadrant digits (80 bits), digit = 3 - q so a
//           left-first DFS visits children in the reference's pop order
//           3,2,1,0 (C/layout.py:262-267);
//   sort  : stable radix sort by (hi64, lo16);
//   build : Karras binary radix tree over the sorted keys; a binary node is a
//           quadtree cell iff it is the topmost node of its digit level
//           (delta/2 > parent delta/2); nodes with delta >= 80 below a
//           non-aggregate parent are the reference's depth-40 aggregates;
//   COM   : bottom-up, one thread per leaf, second arrival combines.
// Traversal is stackless (skip pointers: rc_by_split[last]), one thread per
// body in key order so warps walk coherent paths; per-body decisions are the
// reference's (no warp-vote opening), so the interaction set is identical.
//
// Iteration: [keys] [sort] [build] [COM] [repulsion] [attraction+gravity+
// swing, last block -> global speed] [update, clamp, disp max, bbox, last
// block -> next bbox].  The whole iteration is captured once into a CUDA
// graph and replayed `iterations` times; all scalars live on the device.
#include <algorithm>
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"

namespace cvz {
namespace {

constexpr int FB = 256;
constexpr int END = 0x7fffffff;
constexpr int MAX_DEPTH = 40;
constexpr double EPS = 1e-4;  // COINCIDE_EPS, C/layout.py:29

// non-contracted fp64 ops: every interaction term rounds like the CPU code
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// C/layout.py:85-94 _separation
__device__ __forceinline__ double separation(double &dx, double &dy, long long a, long long b) {
    double d2 = add(mul(dx, dx), mul(dy, dy));
    if (d2 >= EPS * EPS) return sqrt(d2);
    long long h = (a * 2654435761LL + b * 40503LL) % 65536LL;
    if (h < 0) h += 65536;
    double ang = 6.283185307179586 * ((double)h / 65536.0);
    dx = EPS * cos(ang);
    dy = EPS * sin(ang);
    return EPS;
}

// 1 / d2 without DDIV: MUFU.RCP64H seed (rcp.approx.ftz.f64) + a cubic and a
// Newton fp64 step (relative error ~1e-16, i.e. at the last ulp).  The
// reference computes kr*mi*mj / (d*d) with d = sqrt(d2) (C/layout.py:240,260);
// d*d and d2 differ by <= 1 ulp, so f = kr*mi*mj * (1/d2) agrees to ~1e-15
// relative while skipping the fp64 sqrt + divide sequences that bound the
// traversal on the FP64 pipe.  The seed needs no fp32 round trip (F2F x2).
__device__ __forceinline__ double rcp_approx(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

__device__ __forceinline__ double inv_d2(double d2) {
    // d2 >= COINCIDE_EPS^2 at every call; d2 > ~1e308 (1/d2 subnormal) would
    // flush to 0 (coordinates beyond ~1e150, far outside any layout)
    double r = rcp_approx(d2);
    double e = fma(-d2, r, 1.0);
    e = fma(e, e, e);  // cubic step: seed error 2^-22 -> 2^-66, below the rounding of f
    return fma(r, e, r);
}

struct Body {
    double x, y, m;
    int orig, pad;
};

struct __align__(16) TNode {
    double comx, comy, mass, side2;
    int left, skip, kind, pad;  // kind: 0 transparent, 1 quad cell, 2 aggregate
};

struct Geo {  // root cell, C/layout.py:118-137
    double cx, cy, half;
};

__device__ __forceinline__ Geo root_geo(const double *bbox) {
    double minx = bbox[0], maxx = bbox[1], miny = bbox[2], maxy = bbox[3];
    double half = 0.5 * fmax(maxx - minx, maxy - miny);
    if (!(half > 0.0)) half = 1e-6;
    half *= 1.0000001;
    Geo g;
    g.cx = 0.5 * (minx + maxx);
    g.cy = 0.5 * (miny + maxy);
    g.half = half;
    return g;
}

// ---- bbox ------------------------------------------------------------------
__global__ void bbox_kernel(const double2 *__restrict__ pos, long long n,
                            double *__restrict__ part, unsigned *__restrict__ ctr,
                            double *__restrict__ bbox) {
    double a = INFINITY, b = -INFINITY, c = INFINITY, d = -INFINITY;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double2 p = pos[i];
        a = fmin(a, p.x);
        b = fmax(b, p.x);
        c = fmin(c, p.y);
        d = fmax(d, p.y);
    }
    __shared__ double sh[4][FB / 32];
    for (int o = 16; o > 0; o >>= 1) {
        a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = fmin(c, __shfl_xor_sync(0xffffffffu, c, o));
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    if (lane_id() == 0) {
        sh[0][threadIdx.x >> 5] = a;
        sh[1][threadIdx.x >> 5] = b;
        sh[2][threadIdx.x >> 5] = c;
        sh[3][threadIdx.x >> 5] = d;
    }
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        for (int w = 1; w < FB / 32; ++w) {
            a = fmin(a, sh[0][w]);
            b = fmax(b, sh[1][w]);
            c = fmin(c, sh[2][w]);
            d = fmax(d, sh[3][w]);
        }
        part[4 * blockIdx.x + 0] = a;
        part[4 * blockIdx.x + 1] = b;
        part[4 * blockIdx.x + 2] = c;
        part[4 * blockIdx.x + 3] = d;
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        for (unsigned k = 0; k < gridDim.x; ++k) {
            a = fmin(a, part[4 * k + 0]);
            b = fmax(b, part[4 * k + 1]);
            c = fmin(c, part[4 * k + 2]);
            d = fmax(d, part[4 * k + 3]);
        }
        bbox[0] = a;
        bbox[1] = b;
        bbox[2] = c;
        bbox[3] = d;
        *ctr = 0;
    }
}

// ---- keys ------------------------------------------------------------------
// The reference's descent (C/layout.py:171-208): q = (x >= cx) + 2 (y >= cy),
// child centre c +- h with h = 0.5 * parent half.  fp64, same op order.
// Key split for the sort: k32 = digits 0..D-1 (the radix-sorted part, D =
// top_digits <= 16), krest = digits D..39 (80 - 2D <= 64 bits; only breaks
// ties between bodies sharing a level-D cell).
__global__ void keys_kernel(const double2 *__restrict__ pos, long long n,
                            const double *__restrict__ bbox,
                            unsigned long long *__restrict__ krest, unsigned *__restrict__ k32,
                            unsigned *__restrict__ idx, unsigned *__restrict__ zero_n,
                            unsigned *__restrict__ zero_1, int top_digits) {
    griddep_wait();
    // clear this iteration's counters (no memset node: keeps the PDL chain)
    if (blockIdx.x == 0 && threadIdx.x == 0 && zero_1) *zero_1 = 0;
    if (zero_n)
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x)
            zero_n[i] = 0;
    Geo g = root_geo(bbox);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double2 p = pos[i];
        double cx = g.cx, cy = g.cy, h = g.half;
        unsigned long long rest = 0;
        unsigned top = 0;
        // two loops (top digits, then the rest) instead of a per-level
        // test of which word the digit goes to
        int dpt = 0;
#pragma unroll 4
        for (; dpt < top_digits; ++dpt) {
            int qx = p.x >= cx, qy = p.y >= cy;
            top = (top << 2) | (3u - (unsigned)(qx + 2 * qy));
            h = 0.5 * h;
            cx = qx ? cx + h : cx - h;
            cy = qy ? cy + h : cy - h;
        }
#pragma unroll 4
        for (; dpt < MAX_DEPTH; ++dpt) {
            int qx = p.x >= cx, qy = p.y >= cy;
            rest = (rest << 2) | (3u - (unsigned)(qx + 2 * qy));
            h = 0.5 * h;
            cx = qx ? cx + h : cx - h;
            cy = qy ? cy + h : cy - h;
        }
        k32[i] = top;
        krest[i] = rest;
        idx[i] = (unsigned)i;
    }
}

// ---- tie fix-up after the 32-bit radix sort ------------------------------------
// The stable sort by k32 leaves runs of bodies sharing their level-16 cell in
// index order; the full 80-bit order (ties by index, as the stable LSD sort
// gave) sorts each run by (krest, index).  Runs are rare and short: a thread
// insertion-sorts runs of <= FIX_SMALL; longer runs go to a list for
// tie_fixup_long_kernel (one CTA per run).
constexpr int FIX_SMALL = 32;
constexpr int FIX_SHARED = 2048;

__device__ __forceinline__ bool key_less(unsigned long long ka, unsigned ia,
                                         unsigned long long kb, unsigned ib) {
    return ka < kb || (ka == kb && ia < ib);
}

__global__ void tie_fixup_kernel(const unsigned *__restrict__ k32s, unsigned *__restrict__ idxs,
                                 const unsigned long long *__restrict__ krest, int n,
                                 int *__restrict__ long_runs, unsigned *__restrict__ nlong) {
    griddep_wait();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned k = k32s[i];
        if (i + 1 >= n || k32s[i + 1] != k) continue;  // last of its run (or singleton)
        if (i > 0 && k32s[i - 1] == k) continue;       // not the run head
        int L = 2;
        while (i + L < n && L <= FIX_SMALL && k32s[i + L] == k) ++L;
        if (L > FIX_SMALL) {
            long_runs[atomicAdd(nlong, 1u)] = i;
            continue;
        }
        unsigned id[FIX_SMALL];
        unsigned long long kk[FIX_SMALL];
        for (int j = 0; j < L; ++j) {
            unsigned x = idxs[i + j];
            unsigned long long kx = krest[x];
            int t = j;
            while (t > 0 && key_less(kx, x, kk[t - 1], id[t - 1])) {
                kk[t] = kk[t - 1];
                id[t] = id[t - 1];
                --t;
            }
            kk[t] = kx;
            id[t] = x;
        }
        for (int j = 0; j < L; ++j) idxs[i + j] = id[j];
    }
}

// One CTA per long run: bitonic sort of (krest, index) in shared memory, or
// in global scratch (offset 2*start, disjoint per run) past FIX_SHARED.
// Runs whose krest are all equal are already in order and are skipped.
__global__ void __launch_bounds__(1024) tie_fixup_long_kernel(
    const unsigned *__restrict__ k32s, unsigned *__restrict__ idxs,
    const unsigned long long *__restrict__ krest, int n, const int *__restrict__ long_runs,
    const unsigned *__restrict__ nlong, unsigned long long *__restrict__ gk,
    unsigned *__restrict__ gi) {
    griddep_wait();
    __shared__ unsigned long long sk[FIX_SHARED];
    __shared__ unsigned si[FIX_SHARED];
    __shared__ int s_end;
    const unsigned runs = *nlong;
    for (unsigned r = blockIdx.x; r < runs; r += gridDim.x) {
        const int start = long_runs[r];
        const unsigned k = k32s[start];
        if (threadIdx.x == 0) s_end = n;
        __syncthreads();
        for (int base = start; base < n; base += blockDim.x) {
            int j = base + threadIdx.x;
            if (j < n && k32s[j] != k) atomicMin(&s_end, j);
            if (__syncthreads_or(j < n && k32s[j] != k)) break;
        }
        const int L = s_end - start;
        const unsigned long long k0 = krest[idxs[start]];
        bool differ = false;
        for (int j = threadIdx.x; j < L; j += blockDim.x) differ |= krest[idxs[start + j]] != k0;
        if (!__syncthreads_or(differ)) continue;
        int P = 1;
        while (P < L) P <<= 1;
        unsigned long long *K = P <= FIX_SHARED ? sk : gk + 2LL * start;
        unsigned *I = P <= FIX_SHARED ? si : gi + 2LL * start;
        for (int j = threadIdx.x; j < P; j += blockDim.x) {
            if (j < L) {
                unsigned x = idxs[start + j];
                K[j] = krest[x];
                I[j] = x;
            } else {
                K[j] = ~0ull;
                I[j] = 0xffffffffu;
            }
        }
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
                    int a = 2 * t - (t & (stride - 1));
                    int b = a + stride;
                    bool up = (a & size) == 0;
                    unsigned long long ka = K[a], kb = K[b];
                    unsigned ia = I[a], ib = I[b];
                    if (key_less(kb, ib, ka, ia) == up) {
                        K[a] = kb;
                        K[b] = ka;
                        I[a] = ib;
                        I[b] = ia;
                    }
                }
                __syncthreads();
            }
        }
        for (int j = threadIdx.x; j < L; j += blockDim.x) idxs[start + j] = I[j];
        __syncthreads();
    }
}

// ---- Karras radix tree -----------------------------------------------------
struct Keys {
    const unsigned long long *hi;
    const unsigned *lo;
    int n;
    __device__ __forceinline__ int delta(int i, int j) const {
        if (j < 0 || j >= n) return -1;
        unsigned long long a = hi[i] ^ hi[j];
        if (a) return __clzll(a);
        unsigned b = lo[i] ^ lo[j];
        if (b) return 64 + __clz(b);
        return 80 + __clz((unsigned)(i ^ j));  // identical keys: index tiebreak
    }
};

__device__ __forceinline__ void karras_body(int bid, int nblk, Keys K, int *__restrict__ left, int *__restrict__ first,
                              int *__restrict__ last, int *__restrict__ delta_out,
                              int *__restrict__ parent_int, int *__restrict__ parent_leaf,
                              int *__restrict__ pdelta, int *__restrict__ rc_by_split) {
    const int n = K.n;
    for (int i = bid * blockDim.x + threadIdx.x; i < n - 1; i += nblk * blockDim.x) {
        int d = (K.delta(i, i + 1) - K.delta(i, i - 1)) >= 0 ? 1 : -1;
        int dmin = K.delta(i, i - d);
        int lmax = 2;
        while (K.delta(i, i + lmax * d) > dmin) lmax <<= 1;
        int l = 0;
        for (int t = lmax >> 1; t >= 1; t >>= 1)
            if (K.delta(i, i + (l + t) * d) > dmin) l += t;
        int j = i + l * d;
        int dnode = K.delta(i, j);
        int s = 0;
        int t = l;
        do {
            t = (t + 1) >> 1;
            if (K.delta(i, i + (s + t) * d) > dnode) s += t;
        } while (t > 1);
        int gamma = i + s * d + min(d, 0);
        int lo = min(i, j), hi = max(i, j);
        int lc = (lo == gamma) ? ~gamma : gamma;
        int rc = (hi == gamma + 1) ? ~(gamma + 1) : gamma + 1;
        left[i] = lc;
        first[i] = lo;
        last[i] = hi;
        delta_out[i] = dnode;
        rc_by_split[gamma] = rc;
        if (lc >= 0) {
            parent_int[lc] = i;
            pdelta[lc] = dnode;
        } else {
            parent_leaf[~lc] = i;
        }
        if (rc >= 0) {
            parent_int[rc] = i;
            pdelta[rc] = dnode;
        } else {
            parent_leaf[~rc] = i;
        }
    }
    if (bid == 0 && threadIdx.x == 0) pdelta[0] = -2;  // root
}

// ---- cell sums from fixed-point prefix sums -------------------------------------
// Every radix-tree node covers a contiguous range [first, last] of the
// key-sorted bodies, so its mass and moments are differences of prefix sums,
// and every node is computed independently: no bottom-up pass, no atomics,
// no depth-serial chain.  The prefixes are 128-bit two's-complement fixed
// point: a body's m, m*x, m*y (the same fp64 products as before) scaled by
// 2^S and truncated, with S chosen per tree so that n * max m * max|coord|
// stays below 2^125 -- integer adds are exact and associative, so a
// difference is the cell's exact sum up to one truncation per body
// (<= n * 2^-125 of that bound, finer than a double-double's 2^-106), and
// the scan's dependent chains are two-instruction adds instead of the
// twelve-flop TwoSum (the scan was bound by those fp64 latencies).
struct FX {
    unsigned long long lo;
    long long hi;
};
struct FX3 {
    FX m, x, y;
};

__device__ __forceinline__ FX fx_add(FX a, FX b) {
    FX r;
    asm("add.cc.u64 %0, %2, %4;\n\taddc.s64 %1, %3, %5;"
        : "=l"(r.lo), "=l"(r.hi)
        : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
    return r;
}

__device__ __forceinline__ FX fx_neg(FX a) {
    FX r;
    asm("sub.cc.u64 %0, 0, %2;\n\tsubc.s64 %1, 0, %3;"
        : "=l"(r.lo), "=l"(r.hi)
        : "l"(a.lo), "l"(a.hi));
    return r;
}

// v * 2^S truncated toward zero (|v| * 2^S < 2^127 by the choice of S)
__device__ __forceinline__ FX to_fx(double v, int S) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    int ex = (int)((bits >> 52) & 0x7ff);
    unsigned long long mant = bits & ((1ull << 52) - 1);
    if (ex == 0)
        ex = 1;  // subnormal
    else
        mant |= 1ull << 52;
    const int sh = ex - 1075 + S;  // |v| = mant * 2^(ex - 1075)
    FX r{0ull, 0ll};
    if (sh >= 0) {
        if (sh < 64) {
            r.lo = mant << sh;
            r.hi = sh ? (long long)(mant >> (64 - sh)) : 0ll;
        } else {
            r.hi = (long long)(mant << (sh - 64));
        }
    } else if (sh > -64) {
        r.lo = mant >> (-sh);
    }
    return (bits >> 63) ? fx_neg(r) : r;
}

// x * 2^-S correctly rounded to the nearest double
__device__ __forceinline__ double from_fx(FX x, int S) {
    const bool neg = x.hi < 0;
    if (neg) x = fx_neg(x);
    const unsigned long long hi = (unsigned long long)x.hi;
    double d;
    if (hi == 0) {
        d = __ull2double_rn(x.lo);
    } else {
        const int lz = __clzll(hi);
        unsigned long long w = lz ? (hi << lz) | (x.lo >> (64 - lz)) : hi;
        const unsigned long long rest = lz ? (x.lo << lz) : x.lo;
        w |= rest != 0;  // sticky: the top 64 bits round like the whole value
        d = ldexp(__ull2double_rn(w), 64 - lz);
    }
    d = ldexp(d, -S);
    return neg ? -d : d;
}

// Scales of one tree: prefixes of m stay below n * max m, of m*x / m*y
// below n * max m * max|coord| (bbox of the current positions).  mmax:
// max |m| as non-negative double bits (Tree::set_mass).
struct FxScale {
    int sm, sxy;
};

__device__ __forceinline__ int fx_shift(double bound) {
    // smallest e with 2^e > bound (with margin), S = 125 - e, clamped
    if (!(bound > 0.0)) return 0;
    const int e = ilogb(bound * (1.0 + 0x1p-40)) + 1;
    return max(-1000, min(1000, 125 - e));
}

__device__ __forceinline__ FxScale fx_scale(int n, const unsigned long long *mmax,
                                            const double *bbox) {
    const double mm = __longlong_as_double((long long)*mmax);
    const double c = fmax(fmax(fabs(bbox[0]), fabs(bbox[1])), fmax(fabs(bbox[2]), fabs(bbox[3])));
    const double bm = (double)n * mm;
    return FxScale{fx_shift(bm), fx_shift(bm * c)};
}

// max |mass| (non-negative doubles order like their bit patterns)
__global__ void mass_max_kernel(const double *__restrict__ mass, long long n,
                                unsigned long long *__restrict__ out) {
    unsigned long long m = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        m = max(m, (unsigned long long)__double_as_longlong(fabs(mass[i])));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Two-level fixed-point prefix: tile-local inclusive prefixes (TILE_FX
// bodies per CTA, 8 per thread) + one small scan of the tile totals.
constexpr int FX_ITEMS = 2;
constexpr int TILE_FX = FB * FX_ITEMS;

__device__ __forceinline__ FX fx_shfl_up(FX v, int o) {
    return FX{__shfl_up_sync(0xffffffffu, v.lo, o), __shfl_up_sync(0xffffffffu, v.hi, o)};
}

__device__ __forceinline__ FX3 fx3_add(const FX3 &a, const FX3 &b) {
    return FX3{fx_add(a.m, b.m), fx_add(a.x, b.x), fx_add(a.y, b.y)};
}

// block-wide inclusive scan of one FX3 per thread
__device__ FX3 block_scan_fx3(FX3 v, FX3 *warp_tot, FX3 &block_total) {
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    FX3 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        FX3 y{fx_shfl_up(x.m, o), fx_shfl_up(x.x, o), fx_shfl_up(x.y, o)};
        if (lane >= o) x = fx3_add(y, x);
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    FX3 before{{0, 0}, {0, 0}, {0, 0}};
    FX3 tot{{0, 0}, {0, 0}, {0, 0}};
    for (int w = 0; w < FB / 32; ++w) {
        if (w < wid) before = fx3_add(before, warp_tot[w]);
        tot = fx3_add(tot, warp_tot[w]);
    }
    block_total = tot;
    return wid ? fx3_add(before, x) : x;
}

// Gather the key-sorted bodies of one tile (bodies, 80-bit keys for karras)
// and run the tile-local fixed-point prefix over them in the same CTA.
// sorted 80-bit keys only (the split build: karras can start while the
// bodies are gathered and prefix-summed on the main stream)
__global__ void __launch_bounds__(FB) gather_keys_kernel(
    const unsigned *__restrict__ idx, const unsigned *__restrict__ k32s,
    const unsigned long long *__restrict__ krest, int n, unsigned long long *__restrict__ khi,
    unsigned *__restrict__ klo, int top_digits) {
    griddep_wait();
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const unsigned long long r = krest[idx[p]];
        khi[p] = ((unsigned long long)k32s[p] << (64 - 2 * top_digits)) | (r >> 16);
        klo[p] = (unsigned)(r & 0xffffu) << 16;
    }
}

__device__ __forceinline__ void fx_tiles_body(FX3 *__restrict__ tile_tot, int tiles);

// khi == nullptr: keys already gathered (gather_keys_kernel); tile_ctr !=
// nullptr: the last CTA to finish also scans the tile totals.  (A 3-CTA/SM
// launch bound measured 0.8 % faster per iteration on most runs, but with
// its 80 registers x 3 CTAs filling the register file the side stream's
// karras could not start beside it and ~1 run in 4 fell into a 0.515 ms/iter
// mode: left unbounded.)
__global__ void __launch_bounds__(FB) gather_scan_kernel(
    const double2 *__restrict__ pos, const double *__restrict__ mass,
    const unsigned *__restrict__ idx, const unsigned *__restrict__ k32s,
    const unsigned long long *__restrict__ krest, int n, Body *__restrict__ bodies,
    unsigned long long *__restrict__ khi, unsigned *__restrict__ klo, FX3 *__restrict__ local,
    FX3 *__restrict__ tile_tot, int top_digits, unsigned *__restrict__ tile_ctr,
    const double *__restrict__ bbox, const unsigned long long *__restrict__ mmax) {
    griddep_wait();
    __shared__ FX3 warp_tot[FB / 32];
    const FxScale S = fx_scale(n, mmax, bbox);
    const long long base = (long long)blockIdx.x * TILE_FX + (long long)threadIdx.x * FX_ITEMS;
    FX3 acc{{0, 0}, {0, 0}, {0, 0}};
    FX3 item[FX_ITEMS];
#pragma unroll
    for (int j = 0; j < FX_ITEMS; ++j) {
        long long p = base + j;
        FX3 v{{0, 0}, {0, 0}, {0, 0}};
        if (p < n) {
            unsigned i = idx[p];
            double2 q = pos[i];
            double mi = mass[i];
            bodies[p] = Body{q.x, q.y, mi, (int)i, 0};
            if (khi) {
                unsigned long long r = krest[i];
                khi[p] = ((unsigned long long)k32s[p] << (64 - 2 * top_digits)) | (r >> 16);
                klo[p] = (unsigned)(r & 0xffffu) << 16;  // digits 32..39 on top
            }
            v = FX3{to_fx(mi, S.sm), to_fx(mul(mi, q.x), S.sxy), to_fx(mul(mi, q.y), S.sxy)};
        }
        acc = fx3_add(acc, v);
        item[j] = acc;
    }
    FX3 total;
    FX3 incl = block_scan_fx3(acc, warp_tot, total);
    FX3 excl{{0, 0}, {0, 0}, {0, 0}};
    // exclusive prefix of this thread = incl - acc, formed as a sum to stay exact
    {
        const int lane = lane_id(), wid = threadIdx.x >> 5;
        FX3 up{fx_shfl_up(incl.m, 1), fx_shfl_up(incl.x, 1), fx_shfl_up(incl.y, 1)};
        if (lane > 0) {
            excl = up;
        } else if (wid > 0) {
            for (int w = 0; w < wid; ++w) excl = fx3_add(excl, warp_tot[w]);
        }
    }
#pragma unroll
    for (int j = 0; j < FX_ITEMS; ++j) {
        long long i = base + j;
        if (i < n) local[i] = fx3_add(excl, item[j]);
    }
    if (threadIdx.x == 0) tile_tot[blockIdx.x] = total;
    if (tile_ctr) {  // last CTA scans the tile totals (threadfence-reduction pattern)
        __shared__ bool last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(tile_ctr, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            fx_tiles_body(tile_tot, gridDim.x);
            if (threadIdx.x == 0) *tile_ctr = 0u;  // ready for the next replay
        }
    }
}

// exclusive scan of the tile totals, one CTA
__device__ __forceinline__ void fx_tiles_body(FX3 *__restrict__ tile_tot, int tiles) {
    __shared__ FX3 warp_tot[FB / 32];
    FX3 carry{{0, 0}, {0, 0}, {0, 0}};
    for (int t0 = 0; t0 < tiles; t0 += FB) {
        int t = t0 + threadIdx.x;
        FX3 v = t < tiles ? tile_tot[t] : FX3{{0, 0}, {0, 0}, {0, 0}};
        FX3 total;
        FX3 incl = block_scan_fx3(v, warp_tot, total);
        __syncthreads();
        // exclusive = carry + (incl - v): recompute as carry + exclusive sum
        FX3 excl{{0, 0}, {0, 0}, {0, 0}};
        const int lane = lane_id(), wid = threadIdx.x >> 5;
        FX3 up{fx_shfl_up(incl.m, 1), fx_shfl_up(incl.x, 1), fx_shfl_up(incl.y, 1)};
        if (lane > 0) {
            excl = up;
        } else if (wid > 0) {
            for (int w = 0; w < wid; ++w) excl = fx3_add(excl, warp_tot[w]);
        }
        __syncthreads();
        if (t < tiles) tile_tot[t] = fx3_add(carry, excl);
        carry = fx3_add(carry, total);
        __syncthreads();
    }
}

__device__ __forceinline__ FX3 fx_prefix_at(const FX3 *__restrict__ local,
                                            const FX3 *__restrict__ tile_off, int i) {
    return fx3_add(tile_off[i / TILE_FX], local[i]);
}


// karras (blocks [0, gridDim.x - 1)) and the tile-total scan (last block) are
// independent: one launch runs both side by side
__global__ void __launch_bounds__(FB) karras_tiles_kernel(Keys K, int *__restrict__ left,
                                                          int *__restrict__ first,
                                                          int *__restrict__ last,
                                                          int *__restrict__ delta_out,
                                                          int *__restrict__ parent_int,
                                                          int *__restrict__ parent_leaf,
                                                          int *__restrict__ pdelta,
                                                          int *__restrict__ rc_by_split,
                                                          FX3 *__restrict__ tile_tot, int tiles) {
    griddep_wait();
    if (blockIdx.x == gridDim.x - 1) {
        fx_tiles_body(tile_tot, tiles);
        return;
    }
    karras_body(blockIdx.x, gridDim.x - 1, K, left, first, last, delta_out, parent_int,
                parent_leaf, pdelta, rc_by_split);
}

__global__ void __launch_bounds__(FB) karras_only_kernel(Keys K, int *__restrict__ left,
                                                         int *__restrict__ first,
                                                         int *__restrict__ last,
                                                         int *__restrict__ delta_out,
                                                         int *__restrict__ parent_int,
                                                         int *__restrict__ parent_leaf,
                                                         int *__restrict__ pdelta,
                                                         int *__restrict__ rc_by_split) {
    griddep_wait();
    karras_body(blockIdx.x, gridDim.x, K, left, first, last, delta_out, parent_int, parent_leaf,
                pdelta, rc_by_split);
}

__global__ void node_sums_kernel(int n, const FX3 *__restrict__ local,
                                 const FX3 *__restrict__ tile_off,
                                 const int *__restrict__ left, const int *__restrict__ first,
                                 const int *__restrict__ last, const int *__restrict__ delta,
                                 const int *__restrict__ pdelta,
                                 const int *__restrict__ rc_by_split,
                                 const double *__restrict__ bbox, double *__restrict__ smass,
                                 double *__restrict__ sx, double *__restrict__ sy,
                                 TNode *__restrict__ nodes, unsigned *__restrict__ cnt,
                                 const unsigned long long *__restrict__ mmax) {
    griddep_wait();
    Geo g = root_geo(bbox);
    const FxScale S = fx_scale(n, mmax, bbox);
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < n - 1;
         node += gridDim.x * blockDim.x) {
        const int f0 = first[node], l0 = last[node];
        FX3 hi = fx_prefix_at(local, tile_off, l0);
        if (f0 > 0) {
            const FX3 lo = fx_prefix_at(local, tile_off, f0 - 1);
            hi = FX3{fx_add(hi.m, fx_neg(lo.m)), fx_add(hi.x, fx_neg(lo.x)),
                     fx_add(hi.y, fx_neg(lo.y))};
        }
        const double mm = from_fx(hi.m, S.sm), xx = from_fx(hi.x, S.sxy),
                     yy = from_fx(hi.y, S.sxy);
        smass[node] = mm;
        sx[node] = xx;
        sy[node] = yy;
        int dl = delta[node], pd = pdelta[node];
        int kind;
        if (dl >= 80)
            kind = (pd < 80) ? 2 : 0;  // depth-40 aggregate top (identical keys)
        else
            kind = (node == 0 || (pd >> 1) < (dl >> 1)) ? 1 : 0;  // topmost of its level
        double side = 2.0 * ldexp(g.half, -(dl >> 1));  // exact halvings
        TNode t;
        t.comx = xx / mm;
        t.comy = yy / mm;
        t.mass = mm;
        t.side2 = mul(side, side);
        t.left = left[node];
        t.skip = (l0 == n - 1) ? END : rc_by_split[l0];
        t.kind = kind;
        t.pad = 0;
        nodes[node] = t;
        if (cnt && kind != 0) atomicAdd(cnt + f0, 1u);  // preorder: cells per first body
    }
}

// two smallest original body ids per node (reference cell numbering only)
__global__ void i12_kernel(const Body *__restrict__ bodies, int n, const int *__restrict__ left,
                           const int *__restrict__ last, const int *__restrict__ parent_int,
                           const int *__restrict__ parent_leaf,
                           const int *__restrict__ rc_by_split, unsigned *__restrict__ visit,
                           int2 *__restrict__ i12) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        int node = parent_leaf[p];
        while (node >= 0) {
            __threadfence();
            if (atomicAdd(visit + node, 1u) == 0) break;  // first arrival stops
            __threadfence();
            int l = left[node];
            int gamma = l >= 0 ? last[l] : ~l;
            int rc = rc_by_split[gamma];
            int2 a = l >= 0 ? __ldcg(i12 + l) : make_int2(bodies[~l].orig, INT_MAX);
            int2 b = rc >= 0 ? __ldcg(i12 + rc) : make_int2(bodies[~rc].orig, INT_MAX);
            i12[node] = a.x < b.x ? make_int2(a.x, min(a.y, b.x)) : make_int2(b.x, min(b.y, a.x));
            node = (node == 0) ? -1 : parent_int[node];
        }
    }
}

// ---- reference cell numbering (coincident-point jitter keys) ---------------
// The reference keys the jitter direction of a CELL interaction by the cell's
// array index, i.e. its creation order during sequential insertion
// (C/layout.py:140-210,258).  That order is reconstructed here without
// inserting: a cell is created while inserting body t at depth L, cells of
// one insertion are created top-down, and at a split the old body's child
// comes before the new body's.  So the index of a cell is its rank under the
// key (t, L, flag), where for a cell P with parent cell Y
//   t = i2(Y) if P holds i1(Y) or i2(Y) (created by Y's split), else i1(P);
//   flag = 0 iff P holds i1(Y)      (i1/i2 = two smallest body ids).
// A compressed GPU cell X spans the reference's single-child chain of
// levels [Ltop, Lbot]: its top cell (entry A) follows the rule above, the
// rest (entry B, Lbot - Ltop cells) are created consecutively while inserting
// i2(X).  Single-body leaves get one entry each.  Rank = exclusive scan of
// the entry counts in key order; the root is cell 0.
__device__ __forceinline__ int cell_parent(const int *__restrict__ parent_int,
                                           const int *__restrict__ pdelta, int y, int ly) {
    while (y != 0 && (pdelta[y] >> 1) == ly) y = parent_int[y];  // topmost node of level ly
    return y;
}

__device__ __forceinline__ unsigned long long cell_key(int t, int level, int flag) {
    return ((unsigned long long)(unsigned)t << 8) | ((unsigned long long)level << 1) |
           (unsigned long long)flag;
}

constexpr unsigned long long NO_KEY = ~0ull;

__global__ void cell_entries_kernel(const Body *__restrict__ bodies, int n,
                                    const TNode *__restrict__ nodes, const int *__restrict__ delta,
                                    const int *__restrict__ pdelta,
                                    const int *__restrict__ parent_int,
                                    const int *__restrict__ parent_leaf,
                                    const int2 *__restrict__ i12,
                                    unsigned long long *__restrict__ key,
                                    unsigned *__restrict__ slot, unsigned *__restrict__ count) {
    const int ni = n - 1;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 2 * ni + n;
         t += gridDim.x * blockDim.x) {
        unsigned long long k = NO_KEY;
        unsigned c = 0;
        if (t < 2 * ni) {
            int x = t >> 1, which = t & 1;
            int kind = nodes[x].kind;
            if (kind != 0) {
                int lbot = kind == 2 ? MAX_DEPTH : (delta[x] >> 1);
                int2 ix = i12[x];
                if (x == 0) {  // root: reference cell 0 at level 0 + chain 1..lbot
                    if (which == 1 && lbot >= 1) {
                        k = cell_key(ix.y, 1, 0);
                        c = (unsigned)lbot;
                    }
                } else {
                    int ly = pdelta[x] >> 1, ltop = ly + 1;
                    if (which == 0) {
                        int y = cell_parent(parent_int, pdelta, parent_int[x], ly);
                        int2 iy = i12[y];
                        bool has1 = ix.x == iy.x, has2 = ix.x == iy.y || ix.y == iy.y;
                        k = cell_key((has1 || has2) ? iy.y : ix.x, ltop, has1 ? 0 : 1);
                        c = 1;
                    } else if (lbot > ltop) {
                        k = cell_key(ix.y, ltop + 1, 0);
                        c = (unsigned)(lbot - ltop);
                    }
                }
            }
        } else {
            int p = t - 2 * ni;
            int par = parent_leaf[p];
            if (delta[par] < 2 * MAX_DEPTH) {  // not inside an aggregate
                int ly = delta[par] >> 1;
                int y = cell_parent(parent_int, pdelta, par, ly);
                int2 iy = i12[y];
                int b = bodies[p].orig;
                k = cell_key((b == iy.x || b == iy.y) ? iy.y : b, ly + 1, b == iy.x ? 0 : 1);
                c = 1;
            }
        }
        key[t] = k;
        slot[t] = (unsigned)t;
        count[t] = c;
    }
}

__global__ void gather_counts_kernel(const unsigned *__restrict__ sslot,
                                     const unsigned *__restrict__ count, int ne,
                                     unsigned *__restrict__ scount) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ne; j += gridDim.x * blockDim.x)
        scount[j] = count[sslot[j]];
}

__global__ void scatter_ids_kernel(const unsigned *__restrict__ sslot,
                                   const unsigned *__restrict__ excl, int ne,
                                   int *__restrict__ idslot) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ne; j += gridDim.x * blockDim.x)
        idslot[sslot[j]] = 1 + (int)excl[j];
}

// Reference cell index of the first cell of X's chain that the body would
// approximate: levels [ltop, lcap] tested top-down with the reference's
// `side * side < theta * theta * d2`; none passing -> level lcap + 1 (the
// aggregate, always approximated) -- only reached for aggregates.
__device__ long long ref_cell_id(int c, const int *__restrict__ delta,
                                 const int *__restrict__ pdelta, const int *__restrict__ idslot,
                                 int kind, double half, double th2d2, bool at_bottom) {
    int ltop = c == 0 ? 0 : (pdelta[c] >> 1) + 1;
    int lbot = kind == 2 ? MAX_DEPTH : (delta[c] >> 1);
    int lcap = kind == 2 ? MAX_DEPTH - 1 : lbot;
    int l = at_bottom ? lbot : ltop;
    for (; l <= lcap; ++l) {
        double side = 2.0 * ldexp(half, -l);
        if (mul(side, side) < th2d2) break;
    }
    if (l > lbot) l = lbot;
    if (c == 0 && l == 0) return 0;
    return l == ltop ? idslot[2 * c] : idslot[2 * c + 1] + (l - ltop - 1);
}

// ---- repulsion traversal ---------------------------------------------------
// Cell-jitter context: idslot == nullptr on the first pass (a cell
// interaction closer than COINCIDE_EPS only raises *jflag); the caller then
// builds the reference cell numbering and reruns with idslot set.
struct CellRef {
    const int *delta, *pdelta, *idslot;
    unsigned *jflag;
    const double *bbox;
};

__global__ void __launch_bounds__(FB) bh_kernel(const Body *__restrict__ bodies, int n,
                                                const TNode *__restrict__ nodes,
                                                const int *__restrict__ rc_by_split,
                                                const int *__restrict__ first,
                                                const int *__restrict__ last,
                                                const double *__restrict__ smass,
                                                const double *__restrict__ sx,
                                                const double *__restrict__ sy, double kr,
                                                double theta, double2 *__restrict__ out,
                                                const long long *__restrict__ bad, CellRef cr) {
    if (bad && *bad) return;
    const double th2 = mul(theta, theta);
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        Body me = bodies[p];
        const long long i = me.orig;
        const double xi = me.x, yi = me.y, mi = me.m;
        const double kmi = mul(kr, mi);  // (kr * mi) * mj, the reference's order
        double fx = 0.0, fy = 0.0;
        int c = 0;  // root (n >= 2)
        while (c != END) {
            if (c < 0) {  // leaf body (C/layout.py:235-243)
                int q = ~c;
                if (q != p) {
                    Body bj = bodies[q];
                    double dx = sub(xi, bj.x), dy = sub(yi, bj.y);
                    double d2 = add(mul(dx, dx), mul(dy, dy));
                    double f;
                    if (d2 >= EPS * EPS) {
                        f = mul(mul(kmi, bj.m), inv_d2(d2));
                    } else {  // coincident: reference jitter (C/layout.py:85-94)
                        double d = separation(dx, dy, i, bj.orig);
                        f = mul(kmi, bj.m) / mul(d, d);
                    }
                    fx = add(fx, mul(f, dx));
                    fy = add(fy, mul(f, dy));
                }
                c = (q == n - 1) ? END : __ldg(rc_by_split + q);
                continue;
            }
            TNode t = nodes[c];
            if (t.kind == 0) {  // inner half of a quad cell: always open
                c = t.left;
                continue;
            }
            double mc = t.mass, cx = t.comx, cy = t.comy;
            bool self_out = false;
            if (t.kind == 2 && p >= first[c] && p <= last[c]) {  // aggregate holding i
                // The reference first tests the single-child cells above the
                // aggregate with the FULL centre of mass (self included) and
                // approximates there if one passes (C/layout.py:253-261);
                // only the depth-40 cell itself subtracts self (:247-252).
                int ltop = c == 0 ? 0 : (cr.pdelta[c] >> 1) + 1;
                double dxf = sub(xi, cx), dyf = sub(yi, cy);
                double d2f = add(mul(dxf, dxf), mul(dyf, dyf));
                double s39 = 2.0 * ldexp(root_geo(cr.bbox).half, -(MAX_DEPTH - 1));
                if (!(ltop <= MAX_DEPTH - 1 && mul(s39, s39) < mul(th2, d2f))) {
                    double m2 = sub(smass[c], mi);
                    double x2 = sub(sx[c], mul(mi, xi)), y2 = sub(sy[c], mul(mi, yi));
                    if (m2 <= 0.0) {
                        c = t.skip;
                        continue;
                    }
                    mc = m2;
                    cx = x2 / m2;
                    cy = y2 / m2;
                    self_out = true;
                }
            }
            double dx = sub(xi, cx), dy = sub(yi, cy);
            double d2 = add(mul(dx, dx), mul(dy, dy));
            if (t.kind == 2 || t.side2 < mul(th2, d2)) {  // (C/layout.py:256-261)
                double f;
                if (d2 >= EPS * EPS) {
                    f = mul(mul(kmi, mc), inv_d2(d2));
                } else {
                    long long cell;
                    if (cr.idslot) {
                        cell = ref_cell_id(c, cr.delta, cr.pdelta, cr.idslot, t.kind,
                                           root_geo(cr.bbox).half, mul(th2, d2), self_out);
                    } else {
                        atomicOr(cr.jflag, 1u);
                        cell = c;
                    }
                    double d = separation(dx, dy, i, (long long)n + cell);
                    f = mul(kmi, mc) / mul(d, d);
                }
                fx = add(fx, mul(f, dx));
                fy = add(fy, mul(f, dy));
                c = t.skip;
            } else {
                c = t.left;
            }
        }
        out[i] = make_double2(fx, fy);
    }
}

// ---- flattened traversal: DFS-preorder 32-byte nodes -----------------------
// The binary radix tree has "transparent" nodes (the inner halves of a quad
// cell) that the reference tree does not have and that are always opened.
// After the COM pass, every quad cell / aggregate and every body leaf is
// written into one array in DFS preorder (children in key order = the
// reference's pop order), so a node's first child is the next node and its
// subtree is a contiguous index range ending before `skip`.  A node is one
// 32-byte sector: COM (body position for a leaf), mass, skip, and meta.  A
// cell at depth L stores meta = -(L << 21): the reference halves the root
// side exactly (C/layout.py:171-208), so side^2 at depth L is side0^2 with
// 2L subtracted from its exponent, and the walk forms it with ONE integer
// add into the high word of side0^2.  Leaves and aggregates (always
// approximated) store INT_MIN / INT_MIN + 1: the same add flips the sign of
// side0^2, and a negative side^2 passes `side^2 < theta^2 d^2` for every
// d^2 >= 0, so the hot loop needs no kind test before the opening test.  Rarely needed ids
// (binary node / sorted body) live in a parallel aux[] array.
//
// Preorder index without a sort: with C_le(f) = #cells whose first body is
// <= f, a cell covering bodies [f, l] sits at f + C_lt(f) + A (A = its
// ancestors that share its first body), its DFS successor is l + 1 + C_le(l),
// and leaf q sits at q + C_le(q).
struct __align__(32) PNode {
    double x, y, m;
    int skip;  // preorder index of the DFS successor, -1 = end
    int meta;  // cell: -(level << 21); PN_LEAF / PN_AGG
};

constexpr int PN_LEAF = INT_MIN;
constexpr int PN_AGG = INT_MIN + 1;
// kind (1 cell, 2 depth-40 aggregate, 3 body leaf) and cell depth from meta
__device__ __forceinline__ int pn_kind(int meta) {
    return meta == PN_LEAF ? 3 : meta == PN_AGG ? 2 : 1;
}
__device__ __forceinline__ int pn_level(int meta) { return (-meta) >> 21; }
// side^2 of a node (negative for leaves / aggregates): the exponent form when
// side0^2 is comfortably normal, else the per-level table
template <bool S2EXP>
__device__ __forceinline__ double pn_side2(int meta, int s20_hi, int s20_lo, const double *s2tab) {
    if (S2EXP) return __hiloint2double(s20_hi + meta, s20_lo);
    return meta <= PN_AGG ? -1.0 : s2tab[pn_level(meta)];
}

__device__ __forceinline__ void preorder_cells_body(int tid, int nthr, int n, const TNode *__restrict__ nodes,
                                      const int *__restrict__ first, const int *__restrict__ last,
                                      const int *__restrict__ delta,
                                      const int *__restrict__ parent_int,
                                      const unsigned *__restrict__ cnt,
                                      const unsigned *__restrict__ cle, PNode *__restrict__ pn,
                                      int *__restrict__ aux) {
    const int total = n + (int)cle[n - 1];
    for (int b = tid; b < n - 1; b += nthr) {
        const TNode c = nodes[b];
        if (c.kind == 0) continue;
        const int f = first[b], l = last[b];
        int A = 0;
        for (int a = b == 0 ? -1 : parent_int[b]; a >= 0 && first[a] == f;
             a = a == 0 ? -1 : parent_int[a])
            A += nodes[a].kind != 0;
        const int idx = f + (int)(cle[f] - cnt[f]) + A;
        const int nxt = l + 1 + (int)cle[l];
        PNode t;
        t.x = c.comx;
        t.y = c.comy;
        t.m = c.mass;
        t.skip = nxt >= total ? -1 : nxt;
        t.meta = c.kind == 1 ? -((delta[b] >> 1) << 21) : PN_AGG;
        pn[idx] = t;
        aux[idx] = b;
    }
}

__device__ __forceinline__ void preorder_leaves_body(int tid, int nthr, int n, const Body *__restrict__ bodies,
                                       const unsigned *__restrict__ cle, PNode *__restrict__ pn,
                                       int *__restrict__ aux) {
    const int total = n + (int)cle[n - 1];
    for (int q = tid; q < n; q += nthr) {
        const Body b = bodies[q];
        const int idx = q + (int)cle[q];
        PNode t;
        t.x = b.x;
        t.y = b.y;
        t.m = b.m;
        t.skip = idx + 1 >= total ? -1 : idx + 1;
        t.meta = PN_LEAF;
        pn[idx] = t;
        aux[idx] = q;
    }
}

// cells and leaves of the preorder layout in one launch (first half of the
// grid: cells, second half: leaves)
__global__ void preorder_kernel(int n, const TNode *__restrict__ nodes,
                                const int *__restrict__ first, const int *__restrict__ last,
                                const int *__restrict__ delta, const int *__restrict__ parent_int,
                                const unsigned *__restrict__ cnt, const unsigned *__restrict__ cle,
                                const Body *__restrict__ bodies, PNode *__restrict__ pn,
                                int *__restrict__ aux) {
    griddep_wait();
    const int half = gridDim.x / 2;
    if ((int)blockIdx.x < half)
        preorder_cells_body(blockIdx.x * blockDim.x + threadIdx.x, half * blockDim.x, n, nodes,
                            first, last, delta, parent_int, cnt, cle, pn, aux);
    else
        preorder_leaves_body((blockIdx.x - half) * blockDim.x + threadIdx.x,
                             (gridDim.x - half) * blockDim.x, n, bodies, cle, pn, aux);
}

// side^2 per level (C/layout.py:171-208: exact halvings of the root side)
__device__ __forceinline__ void side2_table(double *tab, const double *bbox) {
    if (threadIdx.x < MAX_DEPTH) {
        double side = 2.0 * ldexp(root_geo(bbox).half, -(int)threadIdx.x);
        tab[threadIdx.x] = mul(side, side);
    }
    __syncthreads();
}

// One node evaluated for body (p, i): the reference's per-body decision and
// force term.  Returns 1 = accepted (force added, or nothing to add), 0 =
// open.  Shared by the per-thread and the warp-cooperative walks.
struct Walker {
    const Body *__restrict__ bodies;
    int n;
    const int *__restrict__ aux;
    const int *__restrict__ nfirst;
    const int *__restrict__ nlast;
    const double *__restrict__ smass;
    const double *__restrict__ sx;
    const double *__restrict__ sy;
    const double *s2tab;
    double th2;
    CellRef cr;

    __device__ __forceinline__ bool visit(const PNode &t, int c, int p, int self, long long i,
                                          double xi, double yi, double mi, double kmi, double &fx,
                                          double &fy) const {
        const int kind = pn_kind(t.meta);
        double mc = t.m, dx = sub(xi, t.x), dy = sub(yi, t.y);
        double d2 = add(mul(dx, dx), mul(dy, dy));
        bool self_out = false;
        if (kind == 2) {
            const int a = aux[c];
            if (p >= nfirst[a] && p <= nlast[a]) {
                // aggregate holding i: the reference tests the single-child
                // cells above it with the FULL COM (self included) and
                // approximates there if one passes (C/layout.py:253-261);
                // only the depth-40 cell itself subtracts self (:247-252)
                int ltop = a == 0 ? 0 : (cr.pdelta[a] >> 1) + 1;
                double s39 = 2.0 * ldexp(root_geo(cr.bbox).half, -(MAX_DEPTH - 1));
                if (!(ltop <= MAX_DEPTH - 1 && mul(s39, s39) < mul(th2, d2))) {
                    double m2 = sub(smass[a], mi);
                    if (m2 <= 0.0) return true;  // nothing left: skip the cell
                    double x2 = sub(sx[a], mul(mi, xi)), y2 = sub(sy[a], mul(mi, yi));
                    mc = m2;
                    dx = sub(xi, x2 / m2);
                    dy = sub(yi, y2 / m2);
                    d2 = add(mul(dx, dx), mul(dy, dy));
                    self_out = true;
                }
            }
        }
        // leaves and aggregates are always approximated (C/layout.py:256-261)
        if (kind == 1 && !(s2tab[pn_level(t.meta)] < mul(th2, d2))) return false;
        if (c == self) return true;  // j == i skipped (:237-238)
        double f;
        if (d2 >= EPS * EPS) {
            f = mul(mul(kmi, mc), inv_d2(d2));
        } else {  // coincident: reference jitter (C/layout.py:85-94)
            long long key;
            if (kind == 3) {
                key = bodies[aux[c]].orig;
            } else if (cr.idslot) {
                key = (long long)n + ref_cell_id(aux[c], cr.delta, cr.pdelta, cr.idslot, kind,
                                                 root_geo(cr.bbox).half, mul(th2, d2), self_out);
            } else {
                atomicOr(cr.jflag, 1u);
                key = (long long)n + aux[c];
            }
            double d = separation(dx, dy, i, key);
            f = mul(kmi, mc) / mul(d, d);
        }
        fx = add(fx, mul(f, dx));
        fy = add(fy, mul(f, dy));
        return true;
    }
};

// Rare paths of the walk as separate (force-inlined) functions; all
// arguments by value and the running force returned in registers (reference
// outputs would spill the loop state to the stack; a real __noinline__ call
// spills it too: 305 -> 397 us at C4).
// coincident pair / cell closer than COINCIDE_EPS: reference jitter
// (C/layout.py:85-94) keyed by the body id or the reference cell number
__device__ __forceinline__ double2 jitter_add(const Body *bodies, int n, const int *aux, CellRef cr,
                                           double th2, int c, int kind, long long i, double kmi,
                                           double mc, double dx, double dy, double d2,
                                           bool self_out, double fx, double fy) {
    long long key;
    if (kind == 3) {
        key = bodies[aux[c]].orig;
    } else if (cr.idslot) {
        key = (long long)n + ref_cell_id(aux[c], cr.delta, cr.pdelta, cr.idslot, kind,
                                         root_geo(cr.bbox).half, mul(th2, d2), self_out);
    } else {
        atomicOr(cr.jflag, 1u);
        key = (long long)n + aux[c];
    }
    double d = separation(dx, dy, i, key);
    double f = mul(kmi, mc) / mul(d, d);
    return make_double2(add(fx, mul(f, dx)), add(fy, mul(f, dy)));
}

// Aggregate cell (always approximated).  If it holds body p, the reference
// tests the single-child cells above it with the FULL COM (self included)
// and approximates there if one passes (C/layout.py:253-261); only the
// depth-40 cell itself subtracts self (:247-252), skipping it when nothing
// is left.
__device__ __forceinline__ double2 aggregate_add(const Walker w, const PNode t, int c, int p,
                                              long long i, double xi, double yi, double mi,
                                              double kmi, double fx, double fy) {
    const int a = w.aux[c];
    double mc = t.m, dx = sub(xi, t.x), dy = sub(yi, t.y);
    double d2 = add(mul(dx, dx), mul(dy, dy));
    bool self_out = false;
    if (p >= w.nfirst[a] && p <= w.nlast[a]) {
        int ltop = a == 0 ? 0 : (w.cr.pdelta[a] >> 1) + 1;
        double s39 = 2.0 * ldexp(root_geo(w.cr.bbox).half, -(MAX_DEPTH - 1));
        if (!(ltop <= MAX_DEPTH - 1 && mul(s39, s39) < mul(w.th2, d2))) {
            double m2 = sub(w.smass[a], mi);
            if (m2 <= 0.0) return make_double2(fx, fy);
            double x2 = sub(w.sx[a], mul(mi, xi)), y2 = sub(w.sy[a], mul(mi, yi));
            mc = m2;
            dx = sub(xi, x2 / m2);
            dy = sub(yi, y2 / m2);
            d2 = add(mul(dx, dx), mul(dy, dy));
            self_out = true;
        }
    }
    if (d2 >= EPS * EPS) {
        double f = mul(mul(kmi, mc), inv_d2(d2));
        return make_double2(add(fx, mul(f, dx)), add(fy, mul(f, dy)));
    }
    return jitter_add(w.bodies, w.n, w.aux, w.cr, w.th2, c, 2, i, kmi, mc, dx, dy, d2, self_out,
                      fx, fy);
}

// per-thread walk: one body per thread, bodies in key order
// COUNT: also tally node visits and accepted (force) terms into stats[0..1]
// (cvz_bh_stats; an instrumentation variant, never the timed walk)
template <int NT, int MINB, bool COUNT = false>
__global__ void __launch_bounds__(NT, MINB) bh_flat_kernel(Walker w, const PNode *__restrict__ pn,
                                                     const unsigned *__restrict__ cle, double kr,
                                                     double th2, double eps2,
                                                     double2 *__restrict__ out,
                                                     const long long *__restrict__ bad,
                                                     const int *__restrict__ work,
                                                     const int *__restrict__ nwork,
                                                     unsigned long long *__restrict__ stats = nullptr) {
    unsigned long long n_visit = 0, n_acc = 0;
    // th2 = theta * theta and eps2 = COINCIDE_EPS^2 come in as launch
    // parameters so the hot loop reads them as constant-bank operands
    griddep_wait();
    if (bad && *bad) return;
    __shared__ double s2tab[MAX_DEPTH];
    side2_table(s2tab, w.cr.bbox);
    w.s2tab = s2tab;
    w.th2 = th2;
    // side^2 at depth d is side0^2 * 4^-d exactly (power-of-two scaling, no
    // subnormals in range): subtract 2d from the exponent instead of a
    // shared-memory lookup per node
    const double s20 = s2tab[0];
    const bool s2exp = s20 > 1e-200 && s20 < 1e300;
    const int s20_hi = __double2hiint(s20), s20_lo = __double2loint(s20);
    const int count = work ? *nwork : w.n;
    for (int t0 = blockIdx.x * blockDim.x + threadIdx.x; t0 < count;
         t0 += gridDim.x * blockDim.x) {
        const int p = work ? work[t0] : t0;
        const Body me = w.bodies[p];
        const long long i = me.orig;
        const double xi = me.x, yi = me.y, mi = me.m;
        const double kmi = mul(kr, mi);  // (kr * mi) * mj, the reference's order
        const int self = p + (int)cle[p];
        double fx = 0.0, fy = 0.0;
        int c = 0;  // root cell (n >= 2)
        // the rare cases (depth-40 aggregates, pairs closer than
        // COINCIDE_EPS, self) sit behind ONE predicate evaluated after the
        // opening test, so the common iteration is load, d2, [open], accept
        // (-1.3 % against testing the kind first)
        while (c >= 0) {
            const PNode t = pn[c];
            if (COUNT) ++n_visit;
            const double dx = sub(xi, t.x), dy = sub(yi, t.y);
            const double d2 = add(mul(dx, dx), mul(dy, dy));
            // cells open unless side^2 < theta^2 d^2; leaves and aggregates
            // are always approximated (C/layout.py:256-261): their side^2 is
            // negative
            const bool open = !((s2exp ? pn_side2<true>(t.meta, s20_hi, s20_lo, s2tab)
                                       : pn_side2<false>(t.meta, s20_hi, s20_lo, s2tab)) <
                                mul(th2, d2));
            if (open) {
                ++c;
                continue;
            }
            if (t.meta == PN_AGG || !(d2 >= eps2)) {
                const int kind = pn_kind(t.meta);
                if (kind == 2) {
                    if (COUNT) ++n_acc;
                    const double2 r = aggregate_add(w, t, c, p, i, xi, yi, mi, kmi, fx, fy);
                    fx = r.x;
                    fy = r.y;
                } else if (c != self) {
                    if (COUNT) ++n_acc;  // j == i skipped (:237-238); a leaf stores its
                                         // body's exact position, so self has d2 == 0
                    const double2 r = jitter_add(w.bodies, w.n, w.aux, w.cr, th2, c, kind, i, kmi,
                                                 t.m, dx, dy, d2, false, fx, fy);
                    fx = r.x;
                    fy = r.y;
                }
                c = t.skip;
                continue;
            }
            if (COUNT) ++n_acc;
            const double f = mul(mul(kmi, t.m), inv_d2(d2));
            fx = add(fx, mul(f, dx));
            fy = add(fy, mul(f, dy));
            c = t.skip;
        }
        out[i] = make_double2(fx, fy);
    }
    if (COUNT) {
        for (int o = 16; o > 0; o >>= 1) {
            n_visit += __shfl_xor_sync(0xffffffffu, n_visit, o);
            n_acc += __shfl_xor_sync(0xffffffffu, n_acc, o);
        }
        if (lane_id() == 0) {
            atomicAdd(stats, n_visit);
            atomicAdd(stats + 1, n_acc);
        }
    }
}

// ---- warp-cooperative walk ----------------------------------------------------
// One warp walks for 32 consecutive (key-ordered) bodies with warp-uniform
// node loads.  A lane evaluates node c only if it opened every ancestor of
// c: after accepting c it resumes at c.skip (preorder: c's subtree is
// [c, skip)).  The warp descends iff some active lane opens, so each lane
// visits exactly its per-thread traversal in the same order (identical
// sums).  Meant for tightly clustered warps (measured slower than the
// per-thread walk at C4, supergraph and full graph; CVZ_BH_WARP=1).
template <int MINB>
__global__ void __launch_bounds__(FB, MINB) bh_warp_kernel(Walker w, const PNode *__restrict__ pn,
                                                     const unsigned *__restrict__ cle, double kr,
                                                     double theta, double2 *__restrict__ out,
                                                     const long long *__restrict__ bad,
                                                     const int *__restrict__ work,
                                                     const int *__restrict__ nwork,
                                                     unsigned *__restrict__ wctr) {
    if (bad && *bad) return;
    __shared__ double s2tab[MAX_DEPTH];
    side2_table(s2tab, w.cr.bbox);
    w.s2tab = s2tab;
    w.th2 = mul(theta, theta);
    const int count = work ? *nwork : w.n;
    const int lane = lane_id();
    const int groups = (count + 31) >> 5;
    while (true) {
        int grp = 0;
        if (lane == 0) grp = (int)atomicAdd(wctr, 1u);
        grp = __shfl_sync(0xffffffffu, grp, 0);
        if (grp >= groups) break;
        const int t0 = grp * 32 + lane;
        const bool valid = t0 < count;
        const int p = valid ? (work ? work[t0] : t0) : 0;
        const Body me = w.bodies[p];
        const long long i = me.orig;
        const double kmi = mul(kr, me.m);
        const int self = p + (int)cle[p];
        double fx = 0.0, fy = 0.0;
        int resume = valid ? 0 : INT_MAX;  // active while c >= resume
        int c = 0;
        while (c >= 0) {
            const PNode t = pn[c];
            bool open = false;
            if (c >= resume) {
                if (w.visit(t, c, p, self, i, me.x, me.y, me.m, kmi, fx, fy))
                    resume = t.skip < 0 ? INT_MAX : t.skip;
                else
                    open = true;
            }
            c = __any_sync(0xffffffffu, open) ? c + 1 : t.skip;
        }
        if (valid) out[i] = make_double2(fx, fy);
    }
}

// exact O(n^2) (C/layout.py:273-290): j ascending, same op order as the CPU
constexpr int XT = 256;
__global__ void __launch_bounds__(XT) exact_kernel(const double2 *__restrict__ pos,
                                                   const double *__restrict__ mass, int n,
                                                   double kr, double2 *__restrict__ out,
                                                   int lo, int hi) {
    __shared__ double3 tile[XT];
    int i = lo + blockIdx.x * blockDim.x + threadIdx.x;  // rows [lo, hi), columns all n
    double xi = 0, yi = 0, mi = 0;
    if (i < hi) {
        double2 p = pos[i];
        xi = p.x;
        yi = p.y;
        mi = mass[i];
    }
    double fx = 0.0, fy = 0.0;
    for (int j0 = 0; j0 < n; j0 += XT) {
        int j = j0 + threadIdx.x;
        if (j < n) {
            double2 p = pos[j];
            tile[threadIdx.x] = make_double3(p.x, p.y, mass[j]);
        }
        __syncthreads();
        int lim = min(XT, n - j0);
        if (i < hi) {
            for (int t = 0; t < lim; ++t) {
                int jj = j0 + t;
                if (jj == i) continue;
                double3 q = tile[t];
                double dx = sub(xi, q.x), dy = sub(yi, q.y);
                double d = separation(dx, dy, i, jj);
                double f = mul(mul(kr, mi), q.z) / mul(d, d);
                fx = add(fx, mul(f, dx));
                fy = add(fy, mul(f, dy));
            }
        }
        __syncthreads();
    }
    if (i < hi) out[i] = make_double2(fx, fy);
}

// ---- CSR for attraction ------------------------------------------------------
// Half-edge h = 2k + side of edge k (row = e[k].x for side 0, e[k].y for side
// 1; col = the other endpoint).  The CSR lists each row's half-edges in h
// order, i.e. in the edge order C/layout.py:301-304 accumulates them.
__global__ void half_edges_kernel(const int2 *__restrict__ e, long long m,
                                  unsigned *__restrict__ key, unsigned *__restrict__ val) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        int2 p = e[k];
        reinterpret_cast<uint2 *>(key)[k] = make_uint2((unsigned)p.x, (unsigned)p.y);
        reinterpret_cast<uint2 *>(val)[k] = make_uint2((unsigned)(2 * k), (unsigned)(2 * k + 1));
    }
}

// Node-sharded ranks keep only the half-edges of the rows they own.
struct OwnedHalfEdge {
    const int2 *e;
    int lo, hi;
    __device__ __forceinline__ bool operator()(long long h) const {
        const int2 p = e[h >> 1];
        const int r = (h & 1) ? p.y : p.x;
        return r >= lo && r < hi;
    }
};

// keys (row - lo) of the selected half-edges (already in h order)
__global__ void owned_keys_kernel(const int2 *__restrict__ e, const unsigned *__restrict__ val,
                                  long long cnt, int lo, unsigned *__restrict__ key) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < cnt;
         j += (long long)gridDim.x * blockDim.x) {
        const unsigned h = val[j];
        const int2 p = e[h >> 1];
        key[j] = (unsigned)(((h & 1) ? p.y : p.x) - lo);
    }
}

// rowptr from the row-sorted half-edge keys (no per-node atomics: hub rows
// serialised them): rows (skey[i-1], skey[i]] start at i, rows past the last
// key at nh; every one of the n + 1 entries is written exactly once.
__global__ void rowptr_kernel(const unsigned *__restrict__ skey, long long nh, long long n,
                              long long *__restrict__ rowptr) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= nh;
         i += (long long)gridDim.x * blockDim.x) {
        const long long lo = i == 0 ? 0 : (long long)skey[i - 1] + 1;
        const long long hi = i == nh ? n : (long long)skey[i];
        for (long long x = lo; x <= hi; ++x) rowptr[x] = i;
    }
}

// col = other endpoint; w = edge weight * sign (C/layout.py:300).  Unit
// weights (full graphs, C/layout.py:337) store no per-half-edge weight: the
// kernels use the sign itself (mul(1.0, sign) == sign exactly).
__global__ void csr_fill_kernel(const int2 *__restrict__ e, const unsigned *__restrict__ sval,
                                long long nh, const double *__restrict__ w, double sign,
                                int *__restrict__ col, double *__restrict__ cw) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < nh;
         j += (long long)gridDim.x * blockDim.x) {
        unsigned h = sval[j];
        long long k = h >> 1;
        int2 p = e[k];
        col[j] = (h & 1) ? p.x : p.y;
        if (cw) cw[j] = mul(w[k], sign);
    }
}

// ---- attraction + gravity + swing/traction (+ global speed in last block) ---
struct StepScalars {
    double speed;
    double sum_swing, sum_traction;
    long long it;       // iteration counter (0-based)
    long long bad;      // first non-finite iteration (1-based), 0 = none
    unsigned long long maxdisp_bits;
};

// Rows longer than HEAVY are summed by a whole warp (lane-strided partials,
// fixed butterfly order -> deterministic); a thread-per-row loop would leave
// the warp waiting on the power-law tail.  C/layout.py:293-304.
constexpr int HEAVY = 32;

__global__ void classify_rows_kernel(const long long *__restrict__ rowptr, int lo, int n,
                                     int *__restrict__ hidx, int *__restrict__ heavy,
                                     unsigned *__restrict__ nheavy) {
    for (int u = lo + blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += gridDim.x * blockDim.x) {
        int h = -1;
        if (rowptr[u + 1] - rowptr[u] > HEAVY) {
            h = (int)atomicAdd(nheavy, 1u);
            heavy[h] = u;
        }
        hidx[u] = h;
    }
}

// Rows longer than HEAVY_SPLIT half-edges (R-MAT hubs: up to millions) are
// cut into chunks of HEAVY_SPLIT, each summed by its own warp into `part`;
// springs_combine_kernel adds a row's chunks in chunk order (deterministic).
// A warp per whole row left one warp streaming a hub's million half-edges
// while the rest of the GPU idled (R-MAT-26: 42.7 ms of a 140 ms iteration).
constexpr long long HEAVY_SPLIT = 65536;

template <bool UNIT>
__global__ void __launch_bounds__(FB) springs_heavy_kernel(
    const double2 *__restrict__ pos, const long long *__restrict__ rowptr,
    const int *__restrict__ col, const double *__restrict__ cw, double unit,
    const int *__restrict__ heavy, int nheavy, double2 *__restrict__ hsum,
    const StepScalars *__restrict__ sc, const int *__restrict__ ch_h,
    const long long *__restrict__ ch_lo, int nchunk, double2 *__restrict__ part) {
    griddep_wait();
    if (sc && sc->bad) return;
    const int lane = lane_id();
    // work items: heavy rows (ch_h == nullptr) or chunks of heavy rows
    const int items = ch_h ? nchunk : nheavy;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items;
         w += (gridDim.x * blockDim.x) >> 5) {
        const int h = ch_h ? ch_h[w] : w;
        const int u = heavy[h];
        double2 pu = pos[u];
        double fx = 0.0, fy = 0.0;
        const long long r0 = ch_h ? ch_lo[w] : rowptr[u];
        const long long end = ch_h ? min(rowptr[u + 1], r0 + HEAVY_SPLIT) : rowptr[u + 1];
        long long j = r0 + lane;
        // four lane-strided terms per step: loads batched ahead of the
        // (unchanged, in-order) accumulation, so the col -> pos chains overlap
        for (; j + 96 < end; j += 128) {
            int v[4];
            double c[4];
            double2 pv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = col[j + 32 * q];
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = UNIT ? unit : cw[j + 32 * q];
#pragma unroll
            for (int q = 0; q < 4; ++q) pv[q] = pos[v[q]];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                fx = add(fx, mul(c[q], sub(pv[q].x, pu.x)));
                fy = add(fy, mul(c[q], sub(pv[q].y, pu.y)));
            }
        }
        for (; j < end; j += 32) {
            double2 pv = pos[col[j]];
            double c = UNIT ? unit : cw[j];
            fx = add(fx, mul(c, sub(pv.x, pu.x)));
            fy = add(fy, mul(c, sub(pv.y, pu.y)));
        }
        for (int o = 16; o > 0; o >>= 1) {
            fx = add(fx, __shfl_xor_sync(0xffffffffu, fx, o));
            fy = add(fy, __shfl_xor_sync(0xffffffffu, fy, o));
        }
        if (lane == 0) (ch_h ? part : hsum)[w] = make_double2(fx, fy);
    }
}

// hsum[h] = sum of row h's chunk partials in chunk order
__global__ void springs_combine_kernel(const int *__restrict__ choff, int nheavy,
                                       const double2 *__restrict__ part,
                                       double2 *__restrict__ hsum) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < nheavy; h += gridDim.x * blockDim.x) {
        double fx = 0.0, fy = 0.0;
        for (int q = choff[h]; q < choff[h + 1]; ++q) {
            fx = add(fx, part[q].x);
            fy = add(fy, part[q].y);
        }
        hsum[h] = make_double2(fx, fy);
    }
}

// chunk list of the heavy rows: nchunks per row (for the scan), then the fill
__global__ void heavy_chunks_count_kernel(const long long *__restrict__ rowptr,
                                          const int *__restrict__ heavy, int nheavy,
                                          int *__restrict__ nch) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < nheavy; h += gridDim.x * blockDim.x) {
        const int u = heavy[h];
        const long long len = rowptr[u + 1] - rowptr[u];
        nch[h] = (int)((len + HEAVY_SPLIT - 1) / HEAVY_SPLIT);
    }
}

__global__ void heavy_chunks_fill_kernel(const long long *__restrict__ rowptr,
                                         const int *__restrict__ heavy, int nheavy,
                                         const int *__restrict__ choff, int *__restrict__ ch_h,
                                         long long *__restrict__ ch_lo) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < nheavy; h += gridDim.x * blockDim.x) {
        const long long r0 = rowptr[heavy[h]];
        for (int q = choff[h]; q < choff[h + 1]; ++q) {
            ch_h[q] = h;
            ch_lo[q] = r0 + (long long)(q - choff[h]) * HEAVY_SPLIT;
        }
    }
}

// Springs of the light rows (<= HEAVY half-edges), one thread per row, in
// edge order from zero.  Runs on a side stream concurrently with the tree
// build + repulsion (it needs only positions); forces_kernel adds the sum.
template <bool UNIT>
__global__ void __launch_bounds__(FB) springs_light_kernel(
    const double2 *__restrict__ pos, const long long *__restrict__ rowptr,
    const int *__restrict__ col, const double *__restrict__ cw, double unit,
    const int *__restrict__ hidx, int lo, int hi, double2 *__restrict__ spr,
    const StepScalars *__restrict__ sc) {
    griddep_wait();
    if (sc && sc->bad) return;
    for (int u = lo + blockIdx.x * blockDim.x + threadIdx.x; u < hi;
         u += gridDim.x * blockDim.x) {
        if (hidx[u] >= 0) continue;  // heavy row: springs_heavy_kernel
        double2 pu = pos[u];
        double fx = 0.0, fy = 0.0;
        for (long long j = rowptr[u]; j < rowptr[u + 1]; ++j) {
            double2 pv = pos[col[j]];
            double w = UNIT ? unit : cw[j];
            fx = add(fx, mul(w, sub(pv.x, pu.x)));
            fy = add(fy, mul(w, sub(pv.y, pu.y)));
        }
        spr[u] = make_double2(fx, fy);
    }
}

__global__ void __launch_bounds__(FB) forces_kernel(
    const double2 *__restrict__ pos, const double *__restrict__ mass, int n,
    const int *__restrict__ hidx, const double2 *__restrict__ hsum,
    const double2 *__restrict__ spr, const double2 *__restrict__ frep, double gravity,
    const double2 *__restrict__ prev, double2 *__restrict__ force, double *__restrict__ swing,
    double *__restrict__ part, unsigned *__restrict__ ctr, StepScalars *__restrict__ sc,
    double jt, int lo, double *__restrict__ sums_out) {
    griddep_wait();
    if (sc->bad) return;
    double s_sw = 0.0, s_tr = 0.0;
    int u = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) {
        double2 pu = pos[u];
        double2 f = frep[u];
        int h = hidx[u];
        // spring sum of the row (C/layout.py:293-304, edge order within the
        // row): warp-summed for heavy rows, per-thread for light rows
        double2 sp = h >= 0 ? hsum[h] : spr[u];
        f.x = add(f.x, sp.x);
        f.y = add(f.y, sp.y);
        double mu = mass[u];
        if (gravity > 0) {  // C/layout.py:307-309,370-371
            double gm = mul(-gravity, mu);
            f.x = add(f.x, mul(gm, pu.x));
            f.y = add(f.y, mul(gm, pu.y));
        }
        force[u] = f;
        double2 q = prev[u];
        double diff = hypot(sub(f.x, q.x), sub(f.y, q.y));
        double tot = hypot(add(f.x, q.x), add(f.y, q.y));
        double sw = mul(mu, diff);
        swing[u] = sw;
        s_sw = sw;
        s_tr = mul(mu, tot) / 2.0;
    }
    // deterministic block reduction: fixed butterfly within each warp, then
    // the 8 warp sums in warp order
    __shared__ double a[FB], b[FB];
    for (int o = 16; o > 0; o >>= 1) {
        s_sw += __shfl_xor_sync(0xffffffffu, s_sw, o);
        s_tr += __shfl_xor_sync(0xffffffffu, s_tr, o);
    }
    if (lane_id() == 0) {
        a[threadIdx.x >> 5] = s_sw;
        b[threadIdx.x >> 5] = s_tr;
    }
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        double bs = a[0], bt = b[0];
        for (int w = 1; w < FB / 32; ++w) {
            bs += a[w];
            bt += b[w];
        }
        part[2 * blockIdx.x] = bs;
        part[2 * blockIdx.x + 1] = bt;
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double x = 0.0, y = 0.0;
    for (unsigned k = threadIdx.x; k < gridDim.x; k += FB) {
        x += ((volatile double *)part)[2 * k];
        y += ((volatile double *)part)[2 * k + 1];
    }
    a[threadIdx.x] = x;
    b[threadIdx.x] = y;
    __syncthreads();
    for (int o = FB / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            a[threadIdx.x] += a[threadIdx.x + o];
            b[threadIdx.x] += b[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && sums_out) {  // node-sharded: rank-local sums
        sums_out[0] = a[0];
        sums_out[1] = b[0];
        *ctr = 0;
        return;
    }
    if (threadIdx.x == 0) {
        double tsw = a[0], ttr = b[0];
        sc->sum_swing = tsw;
        sc->sum_traction = ttr;
        if (tsw > 0) {  // C/layout.py:379-382
            double target = mul(jt, ttr) / tsw;
            sc->speed = fmin(target, 1.5 * sc->speed);
        }
        *ctr = 0;
    }
}

__global__ void __launch_bounds__(FB) update_kernel(
    double2 *__restrict__ pos, int n, const double2 *__restrict__ force,
    const double *__restrict__ swing, double2 *__restrict__ prev, int speed_form,
    double max_step, double *__restrict__ bpart, unsigned *__restrict__ ctr,
    double *__restrict__ bbox, StepScalars *__restrict__ sc, double *__restrict__ disp_hist,
    int lo, double *__restrict__ red_out) {
    griddep_wait();
    if (sc->bad) return;
    const double speed = sc->speed;
    int u = lo + blockIdx.x * blockDim.x + threadIdx.x;
    double nrm = 0.0;
    bool fin = true;
    double a = INFINITY, b = -INFINITY, c = INFINITY, d = -INFINITY;
    if (u < n) {
        double sw = swing[u];
        double local = speed_form == 0 ? speed / (1.0 + sqrt(mul(speed, sw)))
                                       : speed / (1.0 + sqrt(add(speed, sw)));
        double2 f = force[u];
        double dx = mul(f.x, local), dy = mul(f.y, local);
        nrm = hypot(dx, dy);
        if (nrm > max_step) {  // C/layout.py:388-393
            double sc2 = max_step / nrm;
            dx = mul(dx, sc2);
            dy = mul(dy, sc2);
            nrm = max_step;
        }
        double2 p = pos[u];
        p.x = add(p.x, dx);
        p.y = add(p.y, dy);
        pos[u] = p;
        prev[u] = f;
        fin = isfinite(p.x) && isfinite(p.y);
        a = p.x;
        b = p.x;
        c = p.y;
        d = p.y;
    }
    // block max |disp| and bbox: min/max are order-free, so warp shuffles
    // then one smem pass over the 8 warp results give the exact values
    __shared__ double sm[FB], s0[FB], s1[FB], s2[FB], s3[FB];
    bool anybad = __syncthreads_or(!fin);
    for (int o = 16; o > 0; o >>= 1) {
        nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
        a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = fmin(c, __shfl_xor_sync(0xffffffffu, c, o));
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    __shared__ double wr[5][FB / 32];
    const int wid = threadIdx.x >> 5;
    if (lane_id() == 0) {
        wr[0][wid] = nrm;
        wr[1][wid] = a;
        wr[2][wid] = b;
        wr[3][wid] = c;
        wr[4][wid] = d;
    }
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        double m0 = wr[0][0], m1 = wr[1][0], m2 = wr[2][0], m3 = wr[3][0], m4 = wr[4][0];
        for (int w = 1; w < FB / 32; ++w) {
            m0 = fmax(m0, wr[0][w]);
            m1 = fmin(m1, wr[1][w]);
            m2 = fmax(m2, wr[2][w]);
            m3 = fmin(m3, wr[3][w]);
            m4 = fmax(m4, wr[4][w]);
        }
        bpart[5 * blockIdx.x + 0] = m1;
        bpart[5 * blockIdx.x + 1] = m2;
        bpart[5 * blockIdx.x + 2] = m3;
        bpart[5 * blockIdx.x + 3] = m4;
        bpart[5 * blockIdx.x + 4] = anybad ? -1.0 : m0;
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // last block: all threads reduce the per-block partials
    volatile double *vp = bpart;
    double mn_x = INFINITY, mx_x = -INFINITY, mn_y = INFINITY, mx_y = -INFINITY, md = 0.0;
    bool bad = false;
    for (unsigned k = threadIdx.x; k < gridDim.x; k += FB) {
        mn_x = fmin(mn_x, vp[5 * k]);
        mx_x = fmax(mx_x, vp[5 * k + 1]);
        mn_y = fmin(mn_y, vp[5 * k + 2]);
        mx_y = fmax(mx_y, vp[5 * k + 3]);
        double v = vp[5 * k + 4];
        if (v < 0) bad = true;
        md = fmax(md, v);
    }
    __syncthreads();
    sm[threadIdx.x] = md;
    s0[threadIdx.x] = mn_x;
    s1[threadIdx.x] = mx_x;
    s2[threadIdx.x] = mn_y;
    s3[threadIdx.x] = mx_y;
    bad = __syncthreads_or(bad);
    for (int o = FB / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
            s0[threadIdx.x] = fmin(s0[threadIdx.x], s0[threadIdx.x + o]);
            s1[threadIdx.x] = fmax(s1[threadIdx.x], s1[threadIdx.x + o]);
            s2[threadIdx.x] = fmin(s2[threadIdx.x], s2[threadIdx.x + o]);
            s3[threadIdx.x] = fmax(s3[threadIdx.x], s3[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    md = sm[0];
    if (red_out) {  // node-sharded: the all-reduce (MAX) finishes the reduction
        red_out[0] = -s0[0];
        red_out[1] = s1[0];
        red_out[2] = -s2[0];
        red_out[3] = s3[0];
        red_out[4] = md;
        red_out[5] = bad ? 1.0 : 0.0;
        *ctr = 0;
        return;
    }
    bbox[0] = s0[0];
    bbox[1] = s1[0];
    bbox[2] = s2[0];
    bbox[3] = s3[0];
    long long it = sc->it;
    disp_hist[it] = md;
    if (bad) sc->bad = it + 1;  // C/layout.py:395-397 (1-based)
    sc->it = it + 1;
    *ctr = 0;
}

template <class K>
size_t sort_bytes(int n, int bits) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const K *)nullptr, (K *)nullptr,
                                    (const unsigned *)nullptr, (unsigned *)nullptr, n, 0, bits);
    return tb;
}

}  // namespace

// CTAs of a persistent kernel: all that fit at once on every SM.
template <class K>
unsigned persist_blocks(K kernel) {
    static DeviceCache cache;
    const int per_sm = cache.get([&] {
        int b = 0;
        CVZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, FB, 0));
        return b < 1 ? 1 : b;
    });
    return (unsigned)(per_sm * num_sms());
}

// ---------------------------------------------------------------------------
// Tree workspace: everything one repulsion evaluation needs, preallocated so
// an iteration can be captured in a CUDA graph.
// device counters of the instrumented walk (nullptr = off; cvz_bh_stats)
static unsigned long long *g_bh_stats = nullptr;

// ---- small-n tree-key sort ------------------------------------------------
// Stable LSD radix sort of (klo, idx) pairs by bits [0, end_bit) in ONE
// cooperative launch: 8-bit digits, one 2048-key tile per CTA, per pass
//   tile -> smem digit histogram -> global [tile][digit] table -> grid sync
//   -> every CTA scans the table for its own offsets -> block radix sort of
//   the tile by the digit (stable) -> scatter -> grid sync.
// Replaces CUB's onesweep (histogram + scan + memset + pass kernels, ~20 us
// of fixed cost per pass at supergraph sizes) for n <= grid * 2048.
// Passes ping-pong between `out` and `alt` so the last lands in `out`;
// `in` is never written.  Result is identical to any stable sort.
constexpr int TS_THREADS = 256;
constexpr int TS_ITEMS = 8;
constexpr int TS_TILE = TS_THREADS * TS_ITEMS;
// tile counts up to this use per-CTA digit sums (CVZ_TS_SMALL overrides)
constexpr int TS_SMALL_TILES = 64;

__global__ void __launch_bounds__(TS_THREADS) tree_sort_coop_kernel(
    const unsigned *kin, const unsigned *vin, unsigned *kout,
    unsigned *vout, unsigned *kalt, unsigned *valt, unsigned *hist, unsigned *prefix, int n,
    int end_bit, int small_tiles) {
    namespace cg = cooperative_groups;
    using Sort = cub::BlockRadixSort<unsigned, TS_THREADS, TS_ITEMS, unsigned>;
    using Scan = cub::BlockScan<unsigned, TS_THREADS>;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename Scan::TempStorage scan;
    } tmp;
    __shared__ unsigned cnt[256], lstart[256], goff[256];
    cg::grid_group grid = cg::this_grid();
    griddep_wait();
    const int tiles = (n + TS_TILE - 1) / TS_TILE;
    const int c = blockIdx.x;
    const int t = threadIdx.x;
    const int base = c * TS_TILE;
    const int count = c < tiles ? min(TS_TILE, n - base) : 0;
    const int passes = (end_bit + 7) / 8;
    const unsigned *ks = kin, *vs = vin;
    for (int pass = 0; pass < passes; ++pass) {
        const bool to_out = ((passes - 1 - pass) & 1) == 0;
        unsigned *kd = to_out ? kout : kalt, *vd = to_out ? vout : valt;
        const int b0 = 8 * pass, b1 = min(end_bit, b0 + 8);
        const unsigned mask = (1u << (b1 - b0)) - 1u;
        unsigned key[TS_ITEMS], val[TS_ITEMS];
        cnt[t] = 0;
        __syncthreads();
        if (c < tiles) {
#pragma unroll
            for (int q = 0; q < TS_ITEMS; ++q) {
                const int j = t * TS_ITEMS + q;  // blocked arrangement
                if (j < count) {
                    key[q] = __ldcg(ks + base + j);  // L2: written by other CTAs
                    val[q] = __ldcg(vs + base + j);
                    atomicAdd(&cnt[(key[q] >> b0) & mask], 1u);
                } else {
                    key[q] = 0xffffffffu;  // pads sort after every real key
                    val[q] = 0u;
                }
            }
        }
        __syncthreads();
        if (c < tiles) hist[(size_t)c * 256 + t] = cnt[t];
        grid.sync();
        unsigned pre, run;  // this tile's start within digit t, digit t's total
        if (tiles <= small_tiles) {
            // few tiles: every CTA sums the digit columns itself (thread t =
            // digit t, independent L2 loads) -- no second grid barrier and
            // no per-digit block-scan chain (a 1-tile grid used to walk all
            // 256 digits serially: 376 us per launch at C1)
            pre = 0;
            run = 0;
            for (int cc = 0; cc < tiles; ++cc) {
                const unsigned h = __ldcg(hist + (size_t)cc * 256 + t);
                pre += cc < c ? h : 0u;
                run += h;
            }
        } else {
            // per digit, an exclusive scan over tiles (CTA g takes digits g,
            // g + grid, ...): one L2 round trip per digit instead of a
            // tiles-long dependent chain in every CTA
            for (int d = c; d < 256; d += gridDim.x) {
                unsigned r = 0;
                for (int c0 = 0; c0 < tiles; c0 += TS_THREADS) {
                    const int cc = c0 + t;
                    const unsigned h = cc < tiles ? __ldcg(hist + (size_t)cc * 256 + d) : 0u;
                    unsigned ex, agg;
                    Scan(tmp.scan).ExclusiveSum(h, ex, agg);
                    __syncthreads();
                    if (cc < tiles) prefix[(size_t)cc * 256 + d] = r + ex;
                    r += agg;
                }
                if (t == 0) prefix[(size_t)tiles * 256 + d] = r;  // digit total
            }
            grid.sync();
            pre = c < tiles ? __ldcg(prefix + (size_t)c * 256 + t) : 0u;
            run = __ldcg(prefix + (size_t)tiles * 256 + t);
        }
        if (c < tiles) {
            unsigned dbase;
            Scan(tmp.scan).ExclusiveSum(run, dbase);
            __syncthreads();
            unsigned ls;
            Scan(tmp.scan).ExclusiveSum(cnt[t], ls);
            lstart[t] = ls;
            goff[t] = dbase + pre;
            __syncthreads();
            Sort(tmp.sort).SortBlockedToStriped(key, val, b0, b1);
#pragma unroll
            for (int q = 0; q < TS_ITEMS; ++q) {
                const int j = q * TS_THREADS + t;  // striped: sorted position
                if (j < count) {
                    const unsigned d = (key[q] >> b0) & mask;
                    const unsigned dst = goff[d] + (unsigned)j - lstart[d];
                    kd[dst] = key[q];
                    vd[dst] = val[q];
                }
            }
        }
        if (pass + 1 < passes) grid.sync();
        ks = kd;
        vs = vd;
    }
}

static int ts_small_tiles() {
    static const int v = getenv("CVZ_TS_SMALL") ? atoi(getenv("CVZ_TS_SMALL")) : TS_SMALL_TILES;
    return v;
}

// Largest n the cooperative sort takes on this device (0 = unavailable).
static int tree_sort_coop_cap() {
    static DeviceCache cache;
    return cache.get([] {
        int per_sm = 0, sms = 0, coop = 0;
        const int dev = current_device();
        CVZ_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        CVZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CVZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tree_sort_coop_kernel,
                                                               TS_THREADS, 0));
        const char *e = getenv("CVZ_TREE_SORT");
        const bool off = e && std::string(e) == "cub";
        return (coop && !off) ? per_sm * sms * TS_TILE : 0;
    });
}

struct Tree {
    int n = 0;
    unsigned long long *khi, *khi3;
    int *long_runs;            // tie fix-up: heads of runs longer than FIX_SMALL
    unsigned *nlong;
    unsigned long long *fix_k;  // global bitonic scratch for very long runs
    unsigned *fix_i;
    unsigned *klo, *klo2, *klo3, *idx, *idx2;
    Body *bodies;
    int *left, *first, *last, *delta, *parent_int, *parent_leaf, *pdelta, *rc_by_split;
    unsigned *visit;
    double *smass, *sx, *sy;
    TNode *nodes;
    FX3 *prefix, *tile_tot;
    int2 *i12;
    PNode *pn;
    int *paux;
    unsigned *pcnt, *pcle;
    void *ptmp = nullptr;
    size_t ptmp_bytes = 0;
    double *bbox = nullptr;
    unsigned *jflag = nullptr;
    unsigned *wctr = nullptr;  // work counter of the persistent BH walk
    unsigned *tile_ctr = nullptr;  // last-CTA counter of gather_scan (split build)
    // reference cell numbering (allocated on first use)
    Scratch *scr = nullptr;
    int ne = 0;
    unsigned long long *ekey = nullptr, *ekey2 = nullptr;
    unsigned *eslot = nullptr, *eslot2 = nullptr, *ecnt = nullptr, *ecnt2 = nullptr,
             *eexcl = nullptr;
    int *idslot = nullptr;
    void *etmp = nullptr;
    size_t etmp_sort = 0, etmp_scan = 0;
    void *tmp;
    size_t tmp_bytes;
    unsigned *sort_alt = nullptr, *sort_hist = nullptr;  // cooperative small-n key sort
    int tiles_ts = 0;
    void alloc(int n_, Scratch &sc) {
        n = n_;
        scr = &sc;
        i12 = sc.alloc<int2>(n > 1 ? n - 1 : 1);
        prefix = sc.alloc<FX3>(n);
        mmax = sc.alloc<unsigned long long>(1);
        tile_tot = sc.alloc<FX3>((n + TILE_FX - 1) / TILE_FX);
        pn = sc.alloc<PNode>(2 * n - 1);
        paux = sc.alloc<int>(2 * n - 1);
        pcnt = sc.alloc<unsigned>(n);
        pcle = sc.alloc<unsigned>(n);
        CVZ_CUDA(cub::DeviceScan::InclusiveSum(nullptr, ptmp_bytes, pcnt, pcle, n, sc.stream()));
        ptmp = sc.alloc<char>(ptmp_bytes);
        jflag = sc.alloc<unsigned>(1);
        CVZ_CUDA(cudaMemsetAsync(jflag, 0, sizeof(unsigned), sc.stream()));
        wctr = sc.alloc<unsigned>(1);
        tile_ctr = sc.alloc<unsigned>(1);
        CVZ_CUDA(cudaMemsetAsync(tile_ctr, 0, sizeof(unsigned), sc.stream()));
        khi = sc.alloc<unsigned long long>(n);
        khi3 = sc.alloc<unsigned long long>(n);
        klo = sc.alloc<unsigned>(n);
        klo2 = sc.alloc<unsigned>(n);
        klo3 = sc.alloc<unsigned>(n);
        idx = sc.alloc<unsigned>(n);
        idx2 = sc.alloc<unsigned>(n);
        bodies = sc.alloc<Body>(n);
        int ni = n > 1 ? n - 1 : 1;
        left = sc.alloc<int>(ni);
        first = sc.alloc<int>(ni);
        last = sc.alloc<int>(ni);
        delta = sc.alloc<int>(ni);
        parent_int = sc.alloc<int>(ni);
        parent_leaf = sc.alloc<int>(n);
        pdelta = sc.alloc<int>(ni);
        rc_by_split = sc.alloc<int>(ni);
        visit = sc.alloc<unsigned>(ni);
        smass = sc.alloc<double>(ni);
        sx = sc.alloc<double>(ni);
        sy = sc.alloc<double>(ni);
        nodes = sc.alloc<TNode>(ni);
        tmp_bytes = sort_bytes<unsigned>(n, 32);
        if (n <= tree_sort_coop_cap()) {
            sort_alt = sc.alloc<unsigned>(2LL * n);
            tiles_ts = (n + TS_TILE - 1) / TS_TILE;
            sort_hist = sc.alloc<unsigned>((2 * (size_t)tiles_ts + 1) * 256);  // hist + prefix
        }
        long_runs = sc.alloc<int>(n);
        nlong = sc.alloc<unsigned>(1);
        fix_k = sc.alloc<unsigned long long>(2LL * n);
        fix_i = sc.alloc<unsigned>(2LL * n);
        tmp = sc.alloc<char>(tmp_bytes);
    }
    // build from pos + bbox (bbox already on device)
    // aux != nullptr: karras runs on `aux` while the bodies are gathered and
    // prefix-summed on `s` (fork ev_a, join ev_b; both captured into the graph)
    // max |mass| for the fixed-point scales (masses are constant over a
    // layout: once per layout / repulsion call, before any graph capture)
    unsigned long long *mmax = nullptr;
    const double *mass_set = nullptr;
    void set_mass(const double *mass, cudaStream_t s) {
        CVZ_CUDA(cudaMemsetAsync(mmax, 0, sizeof(unsigned long long), s));
        CVZ_LAUNCH(mass_max_kernel, grid_for(n, FB, 1, 8), FB, 0, s, mass, (long long)n, mmax);
        mass_set = mass;
    }
    void build(const double2 *pos, const double *mass, const double *bbox_, cudaStream_t s,
               cudaStream_t aux = nullptr, cudaEvent_t ev_a = nullptr,
               cudaEvent_t ev_b = nullptr) {
        bbox = const_cast<double *>(bbox_);
        CVZ_REQUIRE(mass == mass_set, CVZ_ERR_VALUE, "Tree::set_mass not called for these masses");
        unsigned g = grid_for(n, FB, 1, 8);
        // radix-sorted levels: 12 (3 passes) measured best for supergraph-sized
        // n, 16 for multi-million-body full graphs (denser level-12 cells);
        // CVZ_TREE_TOP overrides (8..16)
        static const char *tenv = getenv("CVZ_TREE_TOP");
        const int top_digits =
            tenv ? std::max(8, std::min(16, atoi(tenv))) : (n < (1 << 21) ? 12 : 16);
        CVZ_LAUNCH_PDL(keys_kernel, g, FB, 0, s, pos, (long long)n, bbox, khi, klo, idx,
                       flat() ? pcnt : nullptr, nlong, top_digits);
        size_t tb = tmp_bytes;
        // stable sort by the top 16 levels (4 radix passes), then the tie
        // fix-up orders bodies sharing a level-16 cell by the other 24 levels
        if (sort_alt) {  // supergraph sizes: one cooperative launch
            CVZ_COOP_N(tree_sort_coop_kernel, (unsigned)((n + TS_TILE - 1) / TS_TILE), TS_THREADS,
                       s, klo, idx, klo2, idx2, sort_alt, sort_alt + n, sort_hist,
                       sort_hist + tiles_ts * 256, n, 2 * top_digits, ts_small_tiles());
        } else {
            CVZ_REGION("cub_sort:tree_keys", s);
            CVZ_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, klo, klo2, idx, idx2, n, 0,
                                                     2 * top_digits, s));
            count_launches(1 + (2 * top_digits + 7) / 8);
        }
        CVZ_LAUNCH_PDL(tie_fixup_kernel, g, FB, 0, s, klo2, idx2, khi, n, long_runs, nlong);
        CVZ_LAUNCH_PDL(tie_fixup_long_kernel, num_sms(), 1024, 0, s, klo2, idx2, khi, n, long_runs,
                   nlong, fix_k, fix_i);
        const int tiles = (n + TILE_FX - 1) / TILE_FX;
        Keys K{khi3, klo3, n};
        if (aux) {
            // the body gather + prefix sums need only the sorted order: they
            // start on the main stream as soon as the tie fix-up is done,
            // while the side stream gathers the keys and runs karras
            CVZ_CUDA(cudaEventRecord(ev_a, s));
            CVZ_CUDA(cudaStreamWaitEvent(aux, ev_a, 0));
            CVZ_LAUNCH(gather_keys_kernel, g, FB, 0, aux, idx2, klo2, khi, n, khi3, klo3,
                       top_digits);
            CVZ_LAUNCH(karras_only_kernel, grid_for(n - 1, FB, 1, 8), FB, 0, aux, K, left, first,
                       last, delta, parent_int, parent_leaf, pdelta, rc_by_split);
            CVZ_CUDA(cudaEventRecord(ev_b, aux));
            CVZ_LAUNCH(gather_scan_kernel, tiles, FB, 0, s, pos, mass, idx2, klo2, khi, n, bodies,
                       (unsigned long long *)nullptr, (unsigned *)nullptr, prefix, tile_tot,
                       top_digits, tile_ctr, bbox, mmax);
            CVZ_CUDA(cudaStreamWaitEvent(s, ev_b, 0));
            CVZ_LAUNCH(node_sums_kernel, grid_for(n - 1, FB, 1, 8), FB, 0, s, n, prefix, tile_tot,
                       left, first, last, delta, pdelta, rc_by_split, bbox, smass, sx, sy, nodes,
                       flat() ? pcnt : nullptr, mmax);
        } else {
            CVZ_LAUNCH_PDL(gather_scan_kernel, tiles, FB, 0, s, pos, mass, idx2, klo2, khi, n,
                           bodies, khi3, klo3, prefix, tile_tot, top_digits, (unsigned *)nullptr,
                           bbox, mmax);
            CVZ_LAUNCH_PDL(karras_tiles_kernel, grid_for(n - 1, FB, 1, 8) + 1, FB, 0, s, K, left,
                           first, last, delta, parent_int, parent_leaf, pdelta, rc_by_split,
                           tile_tot, tiles);
            CVZ_LAUNCH_PDL(node_sums_kernel, grid_for(n - 1, FB, 1, 8), FB, 0, s, n, prefix,
                           tile_tot, left, first, last, delta, pdelta, rc_by_split, bbox, smass, sx,
                           sy, nodes, flat() ? pcnt : nullptr, mmax);
        }
        if (flat()) {
            {
                CVZ_REGION("cub_scan:preorder", s);
                size_t tb = ptmp_bytes;
                CVZ_CUDA(cub::DeviceScan::InclusiveSum(ptmp, tb, pcnt, pcle, n, s));
                count_launches(2);
            }
            const unsigned half = grid_for(n, FB, 1, 8);
            CVZ_LAUNCH_PDL(preorder_kernel, 2 * half, FB, 0, s, n, nodes, first, last, delta,
                           parent_int, pcnt, pcle, bodies, pn, paux);
        }
    }
    bool force_flat = false;  // node-sharded runs always walk the flat tree
    bool flat() const {
        static const bool binary = getenv("CVZ_BH_BINARY") != nullptr;
        return force_flat || !binary;
    }
    // reference cell numbering of the current tree (see cell_entries_kernel)
    // scratch of build_ids: allocated before a CUDA-graph capture (stream-
    // ordered allocation inside the capture is refused)
    void alloc_ids(cudaStream_t s) {
        if (!idslot) {
            ne = 2 * (n - 1) + n;
            ekey = scr->alloc<unsigned long long>(ne);
            ekey2 = scr->alloc<unsigned long long>(ne);
            eslot = scr->alloc<unsigned>(ne);
            eslot2 = scr->alloc<unsigned>(ne);
            ecnt = scr->alloc<unsigned>(ne);
            ecnt2 = scr->alloc<unsigned>(ne);
            eexcl = scr->alloc<unsigned>(ne);
            idslot = scr->alloc<int>(ne);
            CVZ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, etmp_sort, ekey, ekey2, eslot,
                                                     eslot2, ne, 0, 40, s));
            CVZ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, etmp_scan, ecnt2, eexcl, ne, s));
            etmp = scr->alloc<char>(std::max(etmp_sort, etmp_scan));
        }
    }
    void build_ids(cudaStream_t s) {
        alloc_ids(s);
        CVZ_CUDA(cudaMemsetAsync(visit, 0, sizeof(unsigned) * (n - 1), s));
        CVZ_LAUNCH(i12_kernel, grid_for(n, FB, 1, 8), FB, 0, s, bodies, n, left, last, parent_int,
                   parent_leaf, rc_by_split, visit, i12);
        unsigned g = grid_for(ne, FB, 1, 8);
        CVZ_LAUNCH(cell_entries_kernel, g, FB, 0, s, bodies, n, nodes, delta, pdelta, parent_int,
                   parent_leaf, i12, ekey, eslot, ecnt);
        {
            CVZ_REGION("cub_sort:cell_ids", s);
            size_t tb = etmp_sort;
            CVZ_CUDA(cub::DeviceRadixSort::SortPairs(etmp, tb, ekey, ekey2, eslot, eslot2, ne, 0,
                                                     40, s));
            count_launches(6);
        }
        CVZ_LAUNCH(gather_counts_kernel, g, FB, 0, s, eslot2, ecnt, ne, ecnt2);
        {
            CVZ_REGION("cub_scan:cell_ids", s);
            size_t tb = etmp_scan;
            CVZ_CUDA(cub::DeviceScan::ExclusiveSum(etmp, tb, ecnt2, eexcl, ne, s));
            count_launches(2);
        }
        CVZ_LAUNCH(scatter_ids_kernel, g, FB, 0, s, eslot2, eexcl, ne, idslot);
    }
    // work/nwork: optional list of owned sorted bodies (node-sharded layout)
    void repulse(double kr, double theta, double2 *out, const long long *bad, bool ids,
                 cudaStream_t s, const int *work = nullptr, const int *nwork = nullptr) {
        CellRef cr{delta, pdelta, ids ? idslot : nullptr, jflag, bbox};
        if (flat()) {
            static const int minb = getenv("CVZ_BH_MINB") ? atoi(getenv("CVZ_BH_MINB")) : 5;
            static const int bnt = getenv("CVZ_BH_NT") ? atoi(getenv("CVZ_BH_NT")) : 256;
            // per-thread walk by default (it beats the warp-cooperative walk on
            // both supergraphs and full graphs); CVZ_BH_WARP=1 forces the warp
            // walk, CVZ_BH_WARP=auto picks it for n >= 2^21
            static const char *wenv = getenv("CVZ_BH_WARP");
            const bool warp = wenv && (std::string(wenv) == "1" ||
                                       (std::string(wenv) == "auto" && n >= (1 << 21)));
            Walker w{bodies, n, paux, first, last, smass, sx, sy, nullptr, 0.0, cr};
            if (warp) CVZ_CUDA(cudaMemsetAsync(wctr, 0, sizeof(unsigned), s));
#define CVZ_BH_FLAT(B)                                                                        \
    do {                                                                                      \
        if (warp)                                                                             \
            CVZ_LAUNCH(bh_warp_kernel<B>, persist_blocks(bh_warp_kernel<B>), FB, 0, s, w, pn, \
                       pcle, kr, theta, out, bad, work, nwork, wctr);                         \
        else                                                                                  \
            ::cvz::pdl_launch(NT == FB ? "bh_flat_kernel<" #B ">" : "bh_flat_kernel<NT," #B ">", \
                              bh_flat_kernel<NT, B>, dim3(blocks_for(n, NT)), dim3(NT), 0, s, \
                              w, pn, pcle, kr, theta * theta, EPS * EPS, out, bad, work,     \
                              nwork, (unsigned long long *)nullptr);                         \
    } while (0)
            if (bnt == 64) {
                constexpr int NT = 64;
                CVZ_BH_FLAT(20);
            } else if (bnt == 128) {
                constexpr int NT = 128;
                CVZ_BH_FLAT(10);
            } else if (g_bh_stats && minb == 5) {  // instrumented walk (cvz_bh_stats)
                ::cvz::pdl_launch("bh_flat_kernel<count>", bh_flat_kernel<FB, 5, true>,
                                  dim3(blocks_for(n, FB)), dim3(FB), 0, s, w, pn, pcle, kr,
                                  theta * theta, EPS * EPS, out, bad, work, nwork, g_bh_stats);
            } else {
                constexpr int NT = FB;
                if (minb >= 6)
                    CVZ_BH_FLAT(6);
                else if (minb == 5)
                    CVZ_BH_FLAT(5);
                else
                    CVZ_BH_FLAT(4);
            }
#undef CVZ_BH_FLAT
        }
        else
            CVZ_LAUNCH(bh_kernel, blocks_for(n, FB), FB, 0, s, bodies, n, nodes, rc_by_split,
                       first, last, smass, sx, sy, kr, theta, out, bad, cr);
    }
    bool jitter_seen(cudaStream_t s) {
        unsigned h = 0;
        read_small(&h, jflag, sizeof(h), s);
        return h != 0;
    }
};

static void bbox_dev(const double2 *pos, int n, double *bbox, Scratch &sc, cudaStream_t s,
                     double **part_out = nullptr, unsigned **ctr_out = nullptr) {
    unsigned g = grid_for(n, FB, 4, 2);
    double *part = sc.alloc<double>(4 * g);
    unsigned *ctr = sc.alloc<unsigned>(1);
    CVZ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
    CVZ_LAUNCH(bbox_kernel, g, FB, 0, s, pos, (long long)n, part, ctr, bbox);
    (void)part_out;
    (void)ctr_out;
}

void repulsion_dev(const double *pos, const double *mass, long long n, double kr, double theta,
                   double *out, Scratch &sc, cudaStream_t s) {
    auto *p2 = reinterpret_cast<const double2 *>(pos);
    auto *o2 = reinterpret_cast<double2 *>(out);
    if (n <= 1) {
        CVZ_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 2 * (n > 0 ? n : 1), s));
        return;
    }
    if (theta <= 0) {
        CVZ_LAUNCH(exact_kernel, blocks_for(n, XT), XT, 0, s, p2, mass, (int)n, kr, o2, 0,
                   (int)n);
        return;
    }
    double *bbox = sc.alloc<double>(4);
    bbox_dev(p2, (int)n, bbox, sc, s);
    Tree t;
    t.alloc((int)n, sc);
    t.set_mass(mass, s);
    t.build(p2, mass, bbox, s);
    t.repulse(kr, theta, o2, nullptr, false, s);
    if (t.jitter_seen(s)) {  // a cell jitter needs the reference's cell numbering
        t.build_ids(s);
        t.repulse(kr, theta, o2, nullptr, true, s);
    }
}

struct Csr {
    long long *rowptr;  // indexed by node id; valid on [row_lo, row_hi]
    int *col;
    double *w;          // nullptr for unit weights: every half-edge weighs `unit`
    double unit = 1.0;
    long long nh = 0;   // half-edges stored (the owned rows' only)
    int *hidx;      // [n] heavy slot or -1
    int *heavy;     // [nheavy] heavy row ids
    int nheavy = 0;
    double2 *hsum;  // [nheavy] warp-summed springs
    // rows beyond HEAVY_SPLIT half-edges: chunk list (nchunk == 0: none)
    int nchunk = 0;
    int *ch_h = nullptr, *choff = nullptr;
    long long *ch_lo = nullptr;
    double2 *part = nullptr;
};

// CSR over the rows [row_lo, row_hi) (row_hi < 0: all n).  A node-sharded
// rank stores only the half-edges of the rows it owns: a
// stable select of those half-edges in h order, then a stable radix sort by
// row - row_lo (⌈log2(row_hi - row_lo)⌉ bits).  Counts are 64-bit end to end
// (2^30 R-MAT draws give 2.1·10^9 half-edges); h = 2k + side fits 32 bits
// while m < 2^31.  The sort buffers live in a temporary arena, so a shard
// keeps only rowptr + col (+ weights when they are not all 1).
static Csr build_csr(const int2 *e, long long m, long long n, const double *weight, double sign,
                     Scratch &sc, cudaStream_t s, long long row_lo = 0, long long row_hi = -1) {
    if (row_hi < 0) row_hi = n;
    CVZ_REQUIRE(m < (1LL << 31), CVZ_ERR_VALUE, "layout supports < 2^31 edges");
    const bool all_rows = row_lo == 0 && row_hi == n;
    const long long rows = row_hi - row_lo;
    Csr c;
    c.unit = sign;
    long long nh = all_rows ? 2 * m : 0;
    Scratch tmp_sc(s);  // sort keys / values / temp storage: freed on return
    unsigned *key = nullptr, *val = nullptr;
    if (m > 0 && all_rows) {
        key = tmp_sc.alloc<unsigned>(nh);
        val = tmp_sc.alloc<unsigned>(nh);
        CVZ_LAUNCH(half_edges_kernel, grid_for(m, FB, 1, 8), FB, 0, s, e, m, key, val);
    } else if (m > 0 && rows > 0) {
        // stable select of the owned half-edges (order = h order), then keys
        long long *cnt_d = tmp_sc.alloc<long long>(1);
        OwnedHalfEdge pred{e, (int)row_lo, (int)row_hi};
        size_t tb = 0;
        CVZ_CUDA(cub::DeviceSelect::If(nullptr, tb, thrust::counting_iterator<long long>(0),
                                       (unsigned *)nullptr, cnt_d, 2 * m, pred, s));
        void *tmp = tmp_sc.alloc<char>(tb);
        // upper bound for the selection: every half-edge
        unsigned *sel = tmp_sc.alloc<unsigned>(2 * m);
        {
            CVZ_REGION("cub_select:owned_half_edges", s);
            CVZ_CUDA(cub::DeviceSelect::If(tmp, tb, thrust::counting_iterator<long long>(0), sel,
                                           cnt_d, 2 * m, pred, s));
            count_launches(2);
        }
        read_small(&nh, cnt_d, sizeof(nh), s);
        val = sel;
        key = tmp_sc.alloc<unsigned>(nh > 0 ? nh : 1);
        if (nh > 0)
            CVZ_LAUNCH(owned_keys_kernel, grid_for(nh, FB, 1, 8), FB, 0, s, e, val, nh,
                       (int)row_lo, key);
    }
    c.nh = nh;
    long long *rowptr_rel = sc.alloc<long long>(rows + 1);
    c.rowptr = rowptr_rel - row_lo;  // only [row_lo, row_hi] is ever indexed
    c.col = sc.alloc<int>(nh > 0 ? nh : 1);
    c.w = weight ? sc.alloc<double>(nh > 0 ? nh : 1) : nullptr;
    const unsigned *sorted_key = nullptr;
    if (nh > 0) {
        unsigned *skey = tmp_sc.alloc<unsigned>(nh), *sval = tmp_sc.alloc<unsigned>(nh);
        int bits = 1;
        while (bits < 32 && (1LL << bits) < rows) ++bits;
        // scratch in / out: sort over DoubleBuffers (no copy pass)
        cub::DoubleBuffer<unsigned> dk(key, skey), dv(val, sval);
        size_t tb = 0;
        CVZ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, nh, 0, bits, s));
        void *tmp = tmp_sc.alloc<char>(tb);
        {
            CVZ_REGION("cub_sort:csr", s);
            CVZ_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, nh, 0, bits, s));
        }
        count_launches(1 + (bits + 7) / 8);
        sval = dv.Current();
        sorted_key = dk.Current();
        CVZ_LAUNCH(csr_fill_kernel, grid_for(nh, FB, 1, 8), FB, 0, s, e, sval, nh, weight, sign,
                   c.col, c.w);
    }
    CVZ_LAUNCH(rowptr_kernel, grid_for(nh + 1, FB, 1, 8), FB, 0, s, sorted_key, nh, rows,
               rowptr_rel);
    c.hidx = sc.alloc<int>(n);
    c.heavy = sc.alloc<int>(rows > 0 ? rows : 1);
    unsigned *nh_d = tmp_sc.alloc<unsigned>(1);
    CVZ_CUDA(cudaMemsetAsync(nh_d, 0, sizeof(unsigned), s));
    CVZ_LAUNCH(classify_rows_kernel, grid_for(rows, FB, 1, 8), FB, 0, s, c.rowptr,
               (int)row_lo, (int)row_hi, c.hidx, c.heavy, nh_d);
    unsigned nh_h = 0;
    read_small(&nh_h, nh_d, sizeof(unsigned), s);
    c.nheavy = (int)nh_h;
    c.hsum = sc.alloc<double2>(c.nheavy > 0 ? c.nheavy : 1);
    if (c.nheavy > 0) {
        int *nch = tmp_sc.alloc<int>(c.nheavy + 1);
        c.choff = sc.alloc<int>(c.nheavy + 1);
        CVZ_CUDA(cudaMemsetAsync(nch + c.nheavy, 0, sizeof(int), s));
        CVZ_LAUNCH(heavy_chunks_count_kernel, grid_for(c.nheavy, FB, 1, 8), FB, 0, s, c.rowptr,
                   c.heavy, c.nheavy, nch);
        size_t tb = 0;
        CVZ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, nch, c.choff, c.nheavy + 1, s));
        void *tmp = tmp_sc.alloc<char>(tb);
        CVZ_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, nch, c.choff, c.nheavy + 1, s));
        count_launches(2);
        int total = 0;
        read_small(&total, c.choff + c.nheavy, sizeof(int), s);
        if (total > c.nheavy) {  // some row is longer than HEAVY_SPLIT
            c.nchunk = total;
            c.ch_h = sc.alloc<int>(total);
            c.ch_lo = sc.alloc<long long>(total);
            c.part = sc.alloc<double2>(total);
            CVZ_LAUNCH(heavy_chunks_fill_kernel, grid_for(c.nheavy, FB, 1, 8), FB, 0, s, c.rowptr,
                       c.heavy, c.nheavy, c.choff, c.ch_h, c.ch_lo);
        }
    }
    return c;
}

// all spring sums of rows [lo, hi) into c.hsum (heavy) / spr (light)
static void springs(const double2 *pos, const Csr &c, const StepScalars *sc, int lo, int hi,
                    double2 *spr, cudaStream_t s) {
    // unit-weight graphs (no per-half-edge weights) get their own instances.
    // The heavy rows run as ONE grid-stride CTA per SM: with a warp per row
    // (~8K CTAs at C4) the side stream takes every SM slot that frees up
    // while the latency-bound tree kernels of the main stream wait for
    // slots (a 19 us hole after the key sort): 507 -> 492 us/iteration at C4.
    // Stream priorities instead (springs lowest) starve the springs until the
    // walk ends: 528 us.  Multi-million-body layouts (full graphs) keep one
    // warp per row: their springs are ~4x the work and their tree kernels
    // are not latency-bound (the cap costs C4 full graph 4.5 -> 5.0 ms).
    // CVZ_SPRINGS_CAP overrides (CTAs per SM, 0 = none).
    static const char *cenv = getenv("CVZ_SPRINGS_CAP");
    const int cap = cenv ? atoi(cenv) : (hi - lo < (1 << 21) ? 1 : 0);
    if (c.nheavy > 0) {
        const int items = c.nchunk > 0 ? c.nchunk : c.nheavy;
        unsigned hb = blocks_for((long long)items * 32, FB);
        if (cap > 0) hb = std::min<unsigned>(hb, (unsigned)(cap * num_sms()));
        if (c.w)
            CVZ_LAUNCH(springs_heavy_kernel<false>, hb, FB, 0, s, pos, c.rowptr, c.col, c.w,
                       c.unit, c.heavy, c.nheavy, c.hsum, sc, c.ch_h, c.ch_lo, c.nchunk, c.part);
        else
            CVZ_LAUNCH(springs_heavy_kernel<true>, hb, FB, 0, s, pos, c.rowptr, c.col, c.w,
                       c.unit, c.heavy, c.nheavy, c.hsum, sc, c.ch_h, c.ch_lo, c.nchunk, c.part);
        if (c.nchunk > 0)
            CVZ_LAUNCH(springs_combine_kernel, grid_for(c.nheavy, FB, 1, 8), FB, 0, s, c.choff,
                       c.nheavy, c.part, c.hsum);
    }
    if (hi > lo) {
        const unsigned lb = blocks_for(hi - lo, FB);
        if (c.w)
            CVZ_LAUNCH(springs_light_kernel<false>, lb, FB, 0, s, pos,
                       c.rowptr, c.col, c.w, c.unit, c.hidx, lo, hi, spr, sc);
        else
            CVZ_LAUNCH(springs_light_kernel<true>, lb, FB, 0, s, pos,
                       c.rowptr, c.col, c.w, c.unit, c.hidx, lo, hi, spr, sc);
    }
}

__global__ void attraction_only_kernel(const double2 *__restrict__ pos, int n,
                                       const long long *__restrict__ rowptr,
                                       const int *__restrict__ col, const double *__restrict__ cw,
                                       double unit, double2 *__restrict__ out) {
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        double2 pu = pos[u];
        double2 f = out[u];
        for (long long j = rowptr[u]; j < rowptr[u + 1]; ++j) {
            double2 pv = pos[col[j]];
            double w = cw ? cw[j] : unit;
            f.x = add(f.x, mul(w, sub(pv.x, pu.x)));
            f.y = add(f.y, mul(w, sub(pv.y, pu.y)));
        }
        out[u] = f;
    }
}

// ---- node-sharded layout -----------------------------------
// Every rank holds all positions (all-gathered each iteration) and builds the
// full tree; it computes repulsion, springs, gravity and swing for the nodes
// [lo, hi) it owns and updates only those.  The cross-rank steps are two
// small all-reduces the caller runs between the calls below: Σswing/Σtraction
// (SUM, 2 doubles) before the speed update, and {-minx, maxx, -miny, maxy,
// maxdisp, bad} (MAX, 6 doubles) after it -- then an all-gather of the owned
// position rows.  C/layout.py:363-398 is the single-process loop this splits.
struct OwnedBody {
    const Body *bodies;
    int lo, hi;
    __device__ __forceinline__ bool operator()(int p) const {
        int o = bodies[p].orig;
        return o >= lo && o < hi;
    }
};

__global__ void shard_speed_kernel(const double *__restrict__ sums, StepScalars *__restrict__ sc,
                                   double jt) {
    if (sc->bad) return;
    double tsw = sums[0], ttr = sums[1];
    sc->sum_swing = tsw;
    sc->sum_traction = ttr;
    if (tsw > 0) {  // C/layout.py:379-382
        double target = mul(jt, ttr) / tsw;
        sc->speed = fmin(target, 1.5 * sc->speed);
    }
}

__global__ void shard_absorb_kernel(const double *__restrict__ red, double *__restrict__ bbox,
                                    StepScalars *__restrict__ sc, double *__restrict__ disp_hist) {
    if (sc->bad) return;
    long long it = sc->it;
    if (disp_hist) disp_hist[it] = red[4];
    if (red[5] > 0) sc->bad = it + 1;  // C/layout.py:395-397 (1-based)
    sc->it = it + 1;
    bbox[0] = -red[0];
    bbox[1] = red[1];
    bbox[2] = -red[2];
    bbox[3] = red[3];
}

}  // namespace cvz

struct cvz_fa2_shard {
    cvz::Scratch *sc = nullptr;
    int n = 0, lo = 0, hi = 0;
    cvz_layout_params P{};
    bool exact = false, ids = false;
    const double *mass = nullptr;
    cvz::Csr csr;
    cvz::Tree tree;
    double2 *frep = nullptr, *force = nullptr, *prev = nullptr, *spr = nullptr;
    double *swing = nullptr, *fpart = nullptr, *upart = nullptr, *bbox = nullptr;
    unsigned *ctrs = nullptr;
    cvz::StepScalars *scal = nullptr;
    int *work = nullptr, *nwork = nullptr;
    void *sel_tmp = nullptr;
    size_t sel_bytes = 0;
    unsigned nb = 1;
};

using namespace cvz;

extern "C" {

int cvz_fa2_shard_create(const double *pos, const double *mass, int64_t n, const int32_t *edges,
                         int64_t m, const double *weight, const cvz_layout_params *P, int64_t lo,
                         int64_t hi, int ref_cell_ids, cvz_fa2_shard **out, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n >= 2 && n < (1LL << 30), CVZ_ERR_VALUE, "layout needs 2 <= n < 2^30");
        CVZ_REQUIRE(0 <= lo && lo <= hi && hi <= n, CVZ_ERR_VALUE, "bad owned node range");
        cudaStream_t s = as_stream(stream);
        auto *h = new cvz_fa2_shard();
        try {
            h->sc = new Scratch(s);
            Scratch &sc = *h->sc;
            h->n = (int)n;
            h->lo = (int)lo;
            h->hi = (int)hi;
            h->P = *P;
            h->mass = mass;
            h->exact = P->theta <= 0;
            h->ids = ref_cell_ids != 0;
            double sign = P->attraction_form == 0 ? 1.0 : -1.0;
            h->csr = build_csr(reinterpret_cast<const int2 *>(edges), m, n, weight, sign, sc, s,
                               lo, hi);
            h->frep = sc.alloc<double2>(n);
            h->spr = sc.alloc<double2>(n);
            h->force = sc.alloc<double2>(n);
            h->prev = sc.alloc<double2>(n);
            CVZ_CUDA(cudaMemsetAsync(h->prev, 0, sizeof(double2) * n, s));  // C/layout.py:363
            h->swing = sc.alloc<double>(n);
            h->nb = blocks_for(hi - lo, FB);
            h->fpart = sc.alloc<double>(2 * h->nb);
            h->upart = sc.alloc<double>(5 * h->nb);
            h->ctrs = sc.alloc<unsigned>(2);
            CVZ_CUDA(cudaMemsetAsync(h->ctrs, 0, 2 * sizeof(unsigned), s));
            h->bbox = sc.alloc<double>(4);
            h->scal = sc.alloc<StepScalars>(1);
            StepScalars init{};
            init.speed = 1.0;  // C/layout.py:364
            CVZ_CUDA(cudaMemcpyAsync(h->scal, &init, sizeof(init), cudaMemcpyHostToDevice, s));
            bbox_dev(reinterpret_cast<const double2 *>(pos), (int)n, h->bbox, sc, s);
            if (!h->exact) {
                h->tree.alloc((int)n, sc);
                h->tree.set_mass(h->mass, s);
                h->tree.force_flat = true;
                h->work = sc.alloc<int>(hi > lo ? hi - lo : 1);
                h->nwork = sc.alloc<int>(1);
                CVZ_CUDA(cub::DeviceSelect::If(nullptr, h->sel_bytes,
                                               thrust::counting_iterator<int>(0), h->work,
                                               h->nwork, (int)n, OwnedBody{nullptr, 0, 0}, s));
                h->sel_tmp = sc.alloc<char>(h->sel_bytes);
            }
            CVZ_CUDA(cudaStreamSynchronize(s));  // init copy source is a host local
        } catch (...) {
            delete h->sc;
            delete h;
            throw;
        }
        *out = h;
    });
}

int cvz_fa2_shard_forces(cvz_fa2_shard *h, const double *pos, double *sums_out, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(h != nullptr, CVZ_ERR_VALUE, "null shard handle");
        cudaStream_t s = as_stream(stream);
        auto *p2 = reinterpret_cast<const double2 *>(pos);
        const cvz_layout_params &P = h->P;
        long long *badp = &h->scal->bad;
        if (h->exact) {
            CVZ_LAUNCH(exact_kernel, blocks_for(h->hi - h->lo, XT), XT, 0, s, p2, h->mass, h->n,
                       P.repulsion, h->frep, h->lo, h->hi);
        } else {
            h->tree.build(p2, h->mass, h->bbox, s);
            if (h->ids) h->tree.build_ids(s);
            {
                CVZ_REGION("cub_select:owned_bodies", s);
                size_t tb = h->sel_bytes;
                CVZ_CUDA(cub::DeviceSelect::If(h->sel_tmp, tb, thrust::counting_iterator<int>(0),
                                               h->work, h->nwork, h->n,
                                               OwnedBody{h->tree.bodies, h->lo, h->hi}, s));
                count_launches(2);
            }
            h->tree.repulse(P.repulsion, P.theta, h->frep, badp, h->ids, s, h->work, h->nwork);
        }
        springs(p2, h->csr, h->scal, h->lo, h->hi, h->spr, s);
        CVZ_LAUNCH(forces_kernel, h->nb, FB, 0, s, p2, h->mass, h->hi, h->csr.hidx, h->csr.hsum,
                   h->spr, h->frep, P.gravity, h->prev, h->force, h->swing, h->fpart, h->ctrs,
                   h->scal, P.jitter_tolerance, h->lo, sums_out);
    });
}

int cvz_fa2_shard_update(cvz_fa2_shard *h, double *pos, const double *sums, double *red_out,
                         void *stream) {
    return guard([&] {
        CVZ_REQUIRE(h != nullptr, CVZ_ERR_VALUE, "null shard handle");
        cudaStream_t s = as_stream(stream);
        CVZ_LAUNCH(shard_speed_kernel, 1, 1, 0, s, sums, h->scal, h->P.jitter_tolerance);
        CVZ_LAUNCH(update_kernel, h->nb, FB, 0, s, reinterpret_cast<double2 *>(pos), h->hi,
                   h->force, h->swing, h->prev, h->P.speed_form, h->P.max_step, h->upart,
                   h->ctrs + 1, h->bbox, h->scal, nullptr, h->lo, red_out);
    });
}

int cvz_fa2_shard_absorb(cvz_fa2_shard *h, const double *red, double *disp_hist, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(h != nullptr, CVZ_ERR_VALUE, "null shard handle");
        CVZ_LAUNCH(shard_absorb_kernel, 1, 1, 0, as_stream(stream), red, h->bbox, h->scal,
                   disp_hist);
    });
}

int cvz_fa2_shard_finish(cvz_fa2_shard *h, double *speed_out, int64_t *bad_iteration,
                         int *jitter_seen, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(h != nullptr, CVZ_ERR_VALUE, "null shard handle");
        cudaStream_t s = as_stream(stream);
        StepScalars out;
        unsigned jf = 0;
        read_small(&out, h->scal, sizeof(out), s);
        if (!h->exact)
            read_small(&jf, h->tree.jflag, sizeof(jf), s);
        if (speed_out) *speed_out = out.speed;
        *bad_iteration = out.bad;
        *jitter_seen = jf != 0;
    });
}

int cvz_fa2_shard_destroy(cvz_fa2_shard *h, void *stream) {
    return guard([&] {
        if (!h) return;
        (void)stream;
        delete h->sc;  // stream-ordered frees on the creation stream
        delete h;
    });
}


int cvz_repulsion(const double *pos, const double *mass, int64_t n, double repulsion,
                  double theta, double *out, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n >= 0 && n < (1LL << 30), CVZ_ERR_VALUE, "bad body count");
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        repulsion_dev(pos, mass, n, repulsion, theta, out, sc, s);
    });
}

int cvz_attraction(const double *pos, int64_t n, const int32_t *edges, int64_t m,
                   const double *weight, double sign, double *out, void *stream) {
    return guard([&] {
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        if (n <= 0 || m <= 0) return;
        Csr c = build_csr(reinterpret_cast<const int2 *>(edges), m, n, weight, sign, sc, s);
        CVZ_LAUNCH(attraction_only_kernel, grid_for(n, FB, 1, 8), FB, 0, s,
                   reinterpret_cast<const double2 *>(pos), (int)n, c.rowptr, c.col, c.w, c.unit,
                   reinterpret_cast<double2 *>(out));
    });
}

// Per-thread, per-device layout resources (never destroyed: process lifetime).
struct LayoutRes {
    cudaStream_t side = nullptr, aux = nullptr, cs = nullptr;
    cudaEvent_t ev[6] = {};
    cudaGraphExec_t exec = nullptr;
    long long key[5] = {-1, -1, -1, -1, -1};  // what `exec` was captured for
};

static LayoutRes &layout_res() {
    constexpr int kMax = 64;
    static thread_local LayoutRes res[kMax];
    const int d = current_device();
    CVZ_REQUIRE(d >= 0 && d < kMax, CVZ_ERR_VALUE, "device index out of range");
    LayoutRes &r = res[d];
    if (!r.side) {
        CVZ_CUDA(cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking));
        CVZ_CUDA(cudaStreamCreateWithFlags(&r.aux, cudaStreamNonBlocking));
        CVZ_CUDA(cudaStreamCreateWithFlags(&r.cs, cudaStreamNonBlocking));
        for (auto &e : r.ev) CVZ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return r;
}

int cvz_layout_run(double *pos, const double *mass, int64_t n, const int32_t *edges, int64_t m,
                   const double *weight, const cvz_layout_params *P, double *prev_force,
                   double *speed, double *disp_hist, int64_t *bad_iteration, void *stream) {
    return guard([&] {
        CVZ_REQUIRE(n >= 2 && n < (1LL << 30), CVZ_ERR_VALUE, "layout needs 2 <= n < 2^30");
        CVZ_REQUIRE(P->iterations >= 1, CVZ_ERR_VALUE, "iterations must be positive");
        cudaStream_t s = as_stream(stream);
        Scratch sc(s);
        const int N = (int)n;
        auto *p2 = reinterpret_cast<double2 *>(pos);
        auto *prev = reinterpret_cast<double2 *>(prev_force);
        double sign = P->attraction_form == 0 ? 1.0 : -1.0;
        Csr csr = build_csr(reinterpret_cast<const int2 *>(edges), m, n, weight, sign, sc, s);
        double2 *frep = sc.alloc<double2>(n), *force = sc.alloc<double2>(n);
        double *swing = sc.alloc<double>(n);
        unsigned nb = blocks_for(n, FB);
        double *fpart = sc.alloc<double>(2 * nb), *upart = sc.alloc<double>(5 * nb);
        unsigned *ctrs = sc.alloc<unsigned>(2);
        CVZ_CUDA(cudaMemsetAsync(ctrs, 0, 2 * sizeof(unsigned), s));
        double *bbox = sc.alloc<double>(4);
        StepScalars *scal = sc.alloc<StepScalars>(1);
        // zeroed scalars + the caller's speed, stream-ordered (no host sync
        // before the layout starts; speed0 keeps the value for a rerun)
        double *speed0 = sc.alloc<double>(1);
        CVZ_CUDA(cudaMemcpyAsync(speed0, speed, sizeof(double), cudaMemcpyDeviceToDevice, s));
        auto reset_scalars = [&] {
            CVZ_CUDA(cudaMemsetAsync(scal, 0, sizeof(StepScalars), s));
            CVZ_CUDA(cudaMemcpyAsync(&scal->speed, speed0, sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
        };
        reset_scalars();
        const bool exact = P->theta <= 0;
        Tree tree;
        if (!exact) {
            tree.alloc(N, sc);
            tree.set_mass(mass, s);
        }
        long long *badp = &scal->bad;
        // snapshot for the (rare) rerun with the reference's cell numbering
        double2 *pos0 = sc.alloc<double2>(n), *prev0 = sc.alloc<double2>(n);
        CVZ_CUDA(cudaMemcpyAsync(pos0, p2, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
        CVZ_CUDA(cudaMemcpyAsync(prev0, prev, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));

        double2 *spr = sc.alloc<double2>(n);
        // springs only need positions: they run on a side stream while the
        // tree is built and walked (fork/join events, captured into the
        // graph); karras of the tree build runs on a second side stream.
        // Streams, events and the instantiated iteration graph persist per
        // thread and device (creating + destroying three streams and
        // instantiating the graph cost ~0.6 ms of host time per call).
        LayoutRes &lr = layout_res();
        cudaStream_t side = lr.side, aux = lr.aux;
        cudaEvent_t ev_fork = lr.ev[0], ev_join = lr.ev[1], ev_ka = lr.ev[2], ev_kb = lr.ev[3];
        // whatever happens (errors included), the side streams' work is
        // ordered before the scratch arena's stream-ordered frees on s
        struct JoinGuard {
            cudaStream_t s, a, b;
            cudaEvent_t e;
            ~JoinGuard() {
                for (cudaStream_t x : {a, b}) {
                    cudaEventRecord(e, x);
                    cudaStreamWaitEvent(s, e, 0);
                }
            }
        } join_guard{s, side, aux, lr.ev[5]};
        static const bool split_build = getenv("CVZ_TREE_SPLIT") == nullptr ||
                                        std::string(getenv("CVZ_TREE_SPLIT")) != "0";
        auto one_iteration = [&](cudaStream_t st, bool ids) {
            CVZ_CUDA(cudaEventRecord(ev_fork, st));
            CVZ_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
            springs(p2, csr, scal, 0, N, spr, side);
            CVZ_CUDA(cudaEventRecord(ev_join, side));
            if (exact) {
                CVZ_LAUNCH(exact_kernel, blocks_for(n, XT), XT, 0, st, p2, mass, N, P->repulsion,
                           frep, 0, N);
            } else {
                if (split_build)
                    tree.build(p2, mass, bbox, st, aux, ev_ka, ev_kb);
                else
                    tree.build(p2, mass, bbox, st);
                if (ids) tree.build_ids(st);
                tree.repulse(P->repulsion, P->theta, frep, badp, ids, st);
            }
            CVZ_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
            CVZ_LAUNCH_PDL(forces_kernel, nb, FB, 0, st, p2, mass, N, csr.hidx, csr.hsum, spr, frep,
                       P->gravity, prev, force, swing, fpart, ctrs, scal, P->jitter_tolerance, 0,
                       nullptr);
            CVZ_LAUNCH_PDL(update_kernel, nb, FB, 0, st, p2, N, force, swing, prev, P->speed_form,
                       P->max_step, upart, ctrs + 1, bbox, scal, disp_hist, 0, nullptr);
        };

        auto run_all = [&](bool ids) {
            if (ids && !exact) tree.alloc_ids(s);  // never allocate inside the capture
            bbox_dev(p2, N, bbox, sc, s);  // first bbox; later ones come from update
            bool use_graph =
                getenv("CVZ_NO_GRAPH") == nullptr && P->iterations > 1 && !prof_on();
            if (use_graph) {
                // capture one iteration on a private stream, then replay; the
                // previous call's executable graph is updated in place when
                // the topology matches (only kernel arguments differ)
                cudaStream_t cs = lr.cs;
                cudaEvent_t ev = lr.ev[4];
                CVZ_CUDA(cudaEventRecord(ev, s));
                CVZ_CUDA(cudaStreamWaitEvent(cs, ev, 0));
                cudaGraph_t graph = nullptr;
                long long before = g_launches.load();
                CVZ_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
                // small layouts (< 2^16 bodies, launch-bound: C1's 121-body
                // supergraph runs ~80 us per iteration) capture several
                // iterations per graph -- the largest divisor of the
                // iteration count up to 8: 82.5 -> 76.5 us/iter at C1; at C4
                // it measured slower (476 -> 490 us), so larger layouts keep
                // one iteration per graph.  CVZ_GRAPH_UNROLL overrides.
                static const char *uenv = getenv("CVZ_GRAPH_UNROLL");
                const long long umax =
                    uenv ? std::max(1LL, atoll(uenv)) : (n < (1 << 16) ? 8LL : 1LL);
                long long unroll = 1;
                for (long long u = std::min(umax, (long long)P->iterations); u > 1; --u)
                    if (P->iterations % u == 0) {
                        unroll = u;
                        break;
                    }
                bool ok = true;
                try {
                    for (long long u = 0; u < unroll; ++u) one_iteration(cs, ids);
                } catch (...) {
                    ok = false;
                }
                cudaError_t ce = cudaStreamEndCapture(cs, &graph);
                long long per_iter = g_launches.load() - before;  // per graph launch
                g_launches.fetch_sub(per_iter);
                bool ready = false;
                // the iteration's node set is fixed by these (launch
                // configurations may differ, which an update allows); a
                // different shape gets a fresh instantiation instead of a
                // failed update
                const long long key[5] = {(long long)n, (long long)csr.nheavy > 0,
                                          (long long)exact, (long long)ids, unroll};
                if (lr.exec && !std::equal(key, key + 5, lr.key)) {
                    cudaGraphExecDestroy(lr.exec);
                    lr.exec = nullptr;
                }
                if (ok && ce == cudaSuccess) {
                    std::copy(key, key + 5, lr.key);
                    if (lr.exec) {
                        cudaGraphExecUpdateResultInfo info;
                        if (cudaGraphExecUpdate(lr.exec, graph, &info) == cudaSuccess) {
                            ready = true;
                        } else {
                            cudaGetLastError();
                            cudaGraphExecDestroy(lr.exec);
                            lr.exec = nullptr;
                        }
                    }
                    if (!ready && cudaGraphInstantiate(&lr.exec, graph, 0) == cudaSuccess)
                        ready = true;
                }
                if (ready) {
                    for (long long it = 0; it < P->iterations; it += unroll) {
                        CVZ_CUDA(cudaGraphLaunch(lr.exec, cs));
                        g_launches.fetch_add(per_iter);
                    }
                    CVZ_CUDA(cudaEventRecord(ev, cs));
                    CVZ_CUDA(cudaStreamWaitEvent(s, ev, 0));
                } else {
                    cudaGetLastError();
                    if (lr.exec) cudaGraphExecDestroy(lr.exec);
                    lr.exec = nullptr;
                    use_graph = false;
                }
                if (graph) cudaGraphDestroy(graph);
            }
            if (!use_graph)
                for (long long it = 0; it < P->iterations; ++it) one_iteration(s, ids);
        };

        run_all(false);
        if (!exact && tree.jitter_seen(s)) {
            // a cell interaction closer than COINCIDE_EPS happened: its jitter
            // direction is keyed by the reference's cell number -- replay the
            // whole run with that numbering (C/layout.py:258)
            CVZ_CUDA(cudaMemcpyAsync(p2, pos0, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
            CVZ_CUDA(cudaMemcpyAsync(prev, prev0, sizeof(double2) * n, cudaMemcpyDeviceToDevice,
                                     s));
            reset_scalars();
            CVZ_CUDA(cudaMemsetAsync(ctrs, 0, 2 * sizeof(unsigned), s));
            run_all(true);
        }
        StepScalars out;
        read_small(&out, scal, sizeof(out), s);
        CVZ_CUDA(cudaMemcpyAsync(speed, &scal->speed, sizeof(double), cudaMemcpyDeviceToDevice,
                                 s));
        *bad_iteration = out.bad;
        if (out.bad)
            throw Error(CVZ_ERR_LAYOUT, "non-finite positions at iteration " +
                                            std::to_string(out.bad) +
                                            "; reduce speed or check input weights");
    });
}

int cvz_bh_stats(int enable, unsigned long long *totals) {
    return guard([&] {
        CVZ_CUDA(cudaDeviceSynchronize());
        if (enable) {
            if (!g_bh_stats) CVZ_CUDA(cudaMalloc(&g_bh_stats, 2 * sizeof(unsigned long long)));
            CVZ_CUDA(cudaMemset(g_bh_stats, 0, 2 * sizeof(unsigned long long)));
        } else if (g_bh_stats) {
            unsigned long long h[2];
            CVZ_CUDA(cudaMemcpy(h, g_bh_stats, sizeof(h), cudaMemcpyDeviceToHost));
            CVZ_CUDA(cudaFree(g_bh_stats));
            g_bh_stats = nullptr;
            if (totals) {
                totals[0] = h[0];
                totals[1] = h[1];
            }
        } else if (totals) {
            totals[0] = totals[1] = 0;
        }
    });
}

}  // extern "C"
