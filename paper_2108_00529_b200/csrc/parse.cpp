// Native edge-list tokenizer: the host half of C/graph.py:50-92
// parse_edge_list.  Text -> external id pairs, with the
// reference's line semantics; the first-seen id remap runs on the GPU
// (cvz_first_seen_remap in graph.cu).
//
// Semantics restated for ASCII input (anything else returns
// CVZ_PARSE_UNSUPPORTED and the caller uses the Python line loop, which is
// the reference's own algorithm):
//  * lines are str.splitlines(): \n, \r, \r\n, \v, \f, \x1c, \x1d, \x1e;
//  * a line is stripped of str whitespace (space, \t-\r, \x1c-\x1f); empty
//    lines and lines starting with '#' or '%' are skipped;
//  * exactly two whitespace-separated tokens, else ParseError "expected two
//    tokens, got K" naming the 1-based line;
//  * each token is Python int(): optional sign, decimal digits with single
//    underscores between digits; anything else -> "non-integer token";
//    values outside int64 -> unsupported (Python ints are unbounded);
//  * u == v lines are dropped before the remap.
// The first error in line order wins, as in the sequential loop.
//
// Parallel form: the text is cut into one byte range per thread; a thread
// owns every line that STARTS in its range, so lines never split.  Each
// thread counts its lines, so error line numbers come from a prefix sum.
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cvz_b200.h"

namespace {

inline bool is_break(unsigned char c) {
    return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d ||
           c == 0x1e;
}
inline bool is_space(unsigned char c) {
    return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

// A line starts at p if p == 0 or text[p-1] ends a line break (the \r of a
// \r\n pair does not).
inline bool line_start(const unsigned char *t, int64_t len, int64_t p) {
    if (p == 0) return true;
    if (p >= len) return false;
    unsigned char c = t[p - 1];
    if (!is_break(c)) return false;
    return !(c == '\r' && t[p] == '\n');
}

enum Status { OK = 0, TOKENS = 1, NONINT = 2, UNSUPPORTED = 3 };

// Python int() on an ASCII token: 0 ok, NONINT, UNSUPPORTED (overflow)
inline int parse_int(const unsigned char *s, const unsigned char *e, int64_t &out) {
    bool neg = false;
    if (s < e && (*s == '+' || *s == '-')) {
        neg = *s == '-';
        ++s;
    }
    if (s == e || !(*s >= '0' && *s <= '9')) return NONINT;
    unsigned long long v = 0;
    bool prev_digit = false, overflow = false;
    for (; s < e; ++s) {
        unsigned char c = *s;
        if (c >= '0' && c <= '9') {
            unsigned d = c - '0';
            if (v > (0xFFFFFFFFFFFFFFFFull - d) / 10) overflow = true;
            v = v * 10 + d;
            prev_digit = true;
        } else if (c == '_') {
            if (!prev_digit || s + 1 == e || !(s[1] >= '0' && s[1] <= '9')) return NONINT;
            prev_digit = false;
        } else {
            return NONINT;
        }
    }
    if (overflow) return UNSUPPORTED;
    if (neg) {
        if (v > 0x8000000000000000ull) return UNSUPPORTED;
        out = (int64_t)(0 - v);
    } else {
        if (v > 0x7FFFFFFFFFFFFFFFull) return UNSUPPORTED;
        out = (int64_t)v;
    }
    return OK;
}

struct Chunk {
    int64_t begin = 0, end = 0;  // [begin, end): line starts owned
    std::vector<int64_t> pairs;
    int64_t lines = 0;
    int64_t err_line = -1;  // local 1-based line of the first error
    int err = OK, err_tokens = 0;
};

void parse_chunk(const unsigned char *t, int64_t len, Chunk &c) {
    int64_t p = c.begin;
    int64_t line = 0;
    while (p < c.end) {
        // one line: [p, q) then skip its break
        int64_t q = p;
        while (q < len && !is_break(t[q])) {
            if (t[q] >= 0x80) {
                c.err = UNSUPPORTED;
                c.err_line = line + 1;
                return;
            }
            ++q;
        }
        ++line;
        // tokens
        const unsigned char *a = t + p, *b = t + q;
        while (a < b && is_space(*a)) ++a;
        if (a < b && *a != '#' && *a != '%') {
            const unsigned char *tok[3][2];
            int k = 0;
            const unsigned char *x = a;
            while (x < b) {
                while (x < b && is_space(*x)) ++x;
                if (x >= b) break;
                const unsigned char *y = x;
                while (y < b && !is_space(*y)) ++y;
                if (k < 3) {
                    tok[k][0] = x;
                    tok[k][1] = y;
                }
                ++k;
                x = y;
            }
            if (k != 2) {
                c.err = TOKENS;
                c.err_tokens = k;
                c.err_line = line;
                return;
            }
            int64_t u = 0, v = 0;
            int su = parse_int(tok[0][0], tok[0][1], u);
            int sv = su == OK ? parse_int(tok[1][0], tok[1][1], v) : OK;
            // int(parts[0]) is evaluated before int(parts[1])
            int s = su != OK ? su : sv;
            if (s != OK) {
                c.err = s;
                c.err_line = line;
                return;
            }
            if (u != v) {  // C/graph.py:79-80 self-loops dropped before the remap
                c.pairs.push_back(u);
                c.pairs.push_back(v);
            }
        }
        // skip the break (\r\n counts once)
        if (q < len) {
            if (t[q] == '\r' && q + 1 < len && t[q + 1] == '\n')
                q += 2;
            else
                q += 1;
        }
        p = q;
    }
    c.lines = line;
}

struct ParseState {
    std::vector<Chunk> chunks;
    int64_t m = 0;
};

thread_local std::string g_parse_msg;

}  // namespace

extern "C" {

int cvz_parse_begin(const char *text, int64_t len, int threads, void **handle, int64_t *m_out,
                    int64_t *err_line, int *err_code, int *err_tokens) {
    *handle = nullptr;
    *m_out = 0;
    *err_line = 0;
    *err_code = 0;
    *err_tokens = 0;
    if (len < 0 || (len > 0 && text == nullptr)) return CVZ_ERR_VALUE;
    try {
        const auto *t = reinterpret_cast<const unsigned char *>(text);
        // threads <= 0: all hardware threads, one per MiB at most; an explicit
        // count is honoured (tests use it to exercise chunk seams)
        int T = threads > 0 ? (int)std::max<int64_t>(1, std::min<int64_t>(threads, len))
                            : (int)std::max<int64_t>(
                                  1, std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                                       len / (1 << 20) + 1));
        auto *st = new ParseState();
        st->chunks.resize(T);
        // chunk boundaries moved forward to the next line start
        std::vector<int64_t> cut(T + 1);
        cut[0] = 0;
        cut[T] = len;
        for (int i = 1; i < T; ++i) {
            int64_t p = std::max(cut[i - 1], len * i / T);
            while (p < len && !line_start(t, len, p)) ++p;
            cut[i] = p;
        }
        for (int i = 0; i < T; ++i) {
            st->chunks[i].begin = cut[i];
            st->chunks[i].end = cut[i + 1];
        }
        std::vector<std::thread> pool;
        for (int i = 1; i < T; ++i) pool.emplace_back(parse_chunk, t, len, std::ref(st->chunks[i]));
        parse_chunk(t, len, st->chunks[0]);
        for (auto &th : pool) th.join();
        // first error in line order; a chunk with an error stops early, so
        // later chunks' line bases are only needed up to the first error
        int64_t base = 0;
        for (auto &c : st->chunks) {
            if (c.err != OK) {
                *err_code = c.err;
                *err_line = base + c.err_line;
                *err_tokens = c.err_tokens;
                delete st;
                return CVZ_OK;
            }
            base += c.lines;
            st->m += (int64_t)c.pairs.size() / 2;
        }
        *m_out = st->m;
        *handle = st;
        return CVZ_OK;
    } catch (const std::exception &e) {
        g_parse_msg = e.what();
        return CVZ_ERR_OOM;
    }
}

int cvz_parse_take(void *handle, int64_t *pairs_out) {
    auto *st = static_cast<ParseState *>(handle);
    if (!st) return CVZ_ERR_VALUE;
    std::vector<std::thread> pool;
    int64_t off = 0;
    for (auto &c : st->chunks) {
        int64_t *dst = pairs_out + off;
        off += (int64_t)c.pairs.size();
        if (pairs_out)
            pool.emplace_back([dst, &c] {
                if (!c.pairs.empty()) std::memcpy(dst, c.pairs.data(), c.pairs.size() * 8);
            });
    }
    for (auto &th : pool) th.join();
    delete st;
    return CVZ_OK;
}

}  // extern "C"
