// Native make_schedule (C/community.py:164-195): the
// edge-processing order emulating `workers` chunked stream readers.
//
// "random" replays numpy's Generator exactly: PCG64 (128-bit LCG, XSL-RR
// output; state and increment come from numpy's SeedSequence on the host),
// Generator.integers(k) = Lemire's bounded draw on 32-bit words taken from
// the bit generator's buffered next_uint32 (low half of a 64-bit draw first,
// high half on the next call -- the buffer lives in the generator state).
// Checked bit-for-bit against numpy in tests/test_host.py.
// "roundrobin" is the closed form of np.lexsort((chunk, within)).
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/cvz_b200.h"

namespace {

struct Pcg64 {
    unsigned __int128 state, inc;
    bool has32;
    uint32_t u32;
    uint64_t next64() {
        const unsigned __int128 mult =
            ((unsigned __int128)0x2360ed051fc65da4ull << 64) | 0x4385df649fccf645ull;
        state = state * mult + inc;
        uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        uint64_t x = hi ^ lo;
        unsigned r = (unsigned)(hi >> 58);
        return (x >> r) | (x << ((64 - r) & 63));
    }
    uint32_t next32() {
        if (has32) {
            has32 = false;
            return u32;
        }
        uint64_t n = next64();
        has32 = true;
        u32 = (uint32_t)(n >> 32);
        return (uint32_t)n;
    }
    // Generator.integers(k), 1 <= k <= 2^32 - 1 (numpy random_bounded_uint64_fill)
    uint32_t integers(uint32_t k) {
        uint32_t rng = k - 1;
        if (rng == 0) return 0;
        uint32_t ex = rng + 1;
        uint64_t m = (uint64_t)next32() * ex;
        uint32_t left = (uint32_t)m;
        if (left < ex) {
            uint32_t th = (0xFFFFFFFFu - rng) % ex;
            while (left < th) {
                m = (uint64_t)next32() * ex;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};

}  // namespace

extern "C" {

int cvz_make_schedule(int64_t m, int workers, int interleave, uint64_t state_hi,
                      uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int has_uint32,
                      uint32_t uinteger, int64_t *out) {
    if (m < 0 || workers < 1 || !out || (interleave != 0 && interleave != 1)) return CVZ_ERR_VALUE;
    if (workers <= 1 || m < 2) {
        for (int64_t i = 0; i < m; ++i) out[i] = i;
        return CVZ_OK;
    }
    std::vector<int64_t> bounds(workers + 1);
    for (int w = 0; w <= workers; ++w) bounds[w] = (int64_t)((__int128)m * w / workers);
    if (interleave == 1) {  // round-robin: i-th element of every chunk, chunks ascending
        int64_t k = 0;
        int64_t longest = 0;
        for (int w = 0; w < workers; ++w) longest = std::max(longest, bounds[w + 1] - bounds[w]);
        for (int64_t r = 0; r < longest; ++r)
            for (int w = 0; w < workers; ++w)
                if (bounds[w] + r < bounds[w + 1]) out[k++] = bounds[w] + r;
        return CVZ_OK;
    }
    Pcg64 g{((unsigned __int128)state_hi << 64) | state_lo,
            ((unsigned __int128)inc_hi << 64) | inc_lo, has_uint32 != 0, uinteger};
    std::vector<int64_t> ptr(bounds.begin(), bounds.end() - 1);
    std::vector<int> live;
    for (int w = 0; w < workers; ++w)
        if (bounds[w] < bounds[w + 1]) live.push_back(w);
    int64_t done = 0;
    while (!live.empty()) {
        uint32_t pick = g.integers((uint32_t)live.size());
        int w = live[pick];
        out[done++] = ptr[w]++;
        if (ptr[w] >= bounds[w + 1]) live.erase(live.begin() + pick);
    }
    return CVZ_OK;
}

}  // extern "C"
