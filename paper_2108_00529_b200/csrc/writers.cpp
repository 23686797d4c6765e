// Native text writers for the path's output formats:
// the TSV tables of C/supergraph.py:79-91, C/community.py:284-294,
// C/graph.py:100-111, C/sketch.py:101-102 and C/cli.py:200-215 (nodes.tsv),
// and the SVG of C/render.py:96-139.  The reference formats row by row with
// Python f-strings; here rows are formatted in parallel (one contiguous row
// range per thread) into one buffer the caller writes out.
//
// Floats use "%.3f": glibc printf and Python's format(x, ".3f") are both
// correctly rounded from the exact binary value, so the text is identical
// (including "-0.000", "nan", "inf").
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cvz_b200.h"

namespace {

struct Text {
    std::vector<std::string> parts;
    int64_t bytes() const {
        int64_t b = 0;
        for (auto &p : parts) b += (int64_t)p.size();
        return b;
    }
};

inline void put_i64(std::string &s, int64_t v) {
    char buf[24];
    char *e = buf + sizeof(buf), *p = e;
    uint64_t u = v < 0 ? 0 - (uint64_t)v : (uint64_t)v;
    do {
        *--p = (char)('0' + u % 10);
        u /= 10;
    } while (u);
    if (v < 0) *--p = '-';
    s.append(p, e - p);
}

inline void put_f3(std::string &s, double v) {
    char buf[64];
    int k = snprintf(buf, sizeof(buf), "%.3f", v);
    if (k >= (int)sizeof(buf)) {  // |v| >= 1e60: rare, format at full length
        std::vector<char> big(k + 1);
        snprintf(big.data(), big.size(), "%.3f", v);
        s.append(big.data(), k);
    } else {
        s.append(buf, k);
    }
}

// run fn(lo, hi, out) over row chunks in parallel, keep chunk order
template <class F>
Text parallel_rows(int64_t rows, F fn) {
    int T = (int)std::max<int64_t>(
        1, std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), rows / 4096 + 1));
    Text t;
    t.parts.resize(T);
    std::vector<std::thread> pool;
    for (int i = 0; i < T; ++i) {
        int64_t lo = rows * i / T, hi = rows * (i + 1) / T;
        if (i == 0) continue;
        pool.emplace_back([&, i, lo, hi] { fn(lo, hi, t.parts[i]); });
    }
    fn(0, rows / T, t.parts[0]);
    for (auto &th : pool) th.join();
    return t;
}

int finish(Text &&t, void **handle, int64_t *bytes) {
    auto *h = new Text(std::move(t));
    *bytes = h->bytes();
    *handle = h;
    return CVZ_OK;
}

}  // namespace

extern "C" {

int cvz_format_table(int64_t nrows, int ncols, const int *kinds, const void *const *cols,
                     char sep, void **handle, int64_t *bytes) {
    if (nrows < 0 || ncols < 1 || !kinds || !cols || !handle || !bytes) return CVZ_ERR_VALUE;
    for (int c = 0; c < ncols; ++c)
        if (kinds[c] < 0 || kinds[c] > 2 || (kinds[c] != 2 && !cols[c])) return CVZ_ERR_VALUE;
    try {
        Text t = parallel_rows(nrows, [&](int64_t lo, int64_t hi, std::string &s) {
            s.reserve((size_t)(hi - lo) * (size_t)ncols * 10);
            for (int64_t r = lo; r < hi; ++r) {
                for (int c = 0; c < ncols; ++c) {
                    if (c) s.push_back(sep);
                    if (kinds[c] == 0)
                        put_i64(s, static_cast<const int64_t *>(cols[c])[r]);
                    else if (kinds[c] == 1)
                        put_f3(s, static_cast<const double *>(cols[c])[r]);
                    else
                        put_i64(s, r);
                }
                s.push_back('\n');
            }
        });
        return finish(std::move(t), handle, bytes);
    } catch (...) {
        return CVZ_ERR_OOM;
    }
}

int cvz_format_svg(int64_t n, const double *pos, const double *radii, const int64_t *classes,
                   const char *const *palette, int ncolors, int64_t ne, const int64_t *edges,
                   const double *mult, double margin, void **handle, int64_t *bytes) {
    if (n < 1 || !pos || !radii || !classes || !palette || ncolors < 1 || !handle || !bytes)
        return CVZ_ERR_VALUE;
    for (int64_t i = 0; i < n; ++i)
        if (classes[i] < 0 || classes[i] >= ncolors) return CVZ_ERR_VALUE;
    try {
        // C/render.py:105-111: lo/hi = min/max -+ max radius, span >= 1e-6
        double mnx = pos[0], mxx = pos[0], mny = pos[1], mxy = pos[1], rmax = radii[0];
        for (int64_t i = 0; i < n; ++i) {
            mnx = std::min(mnx, pos[2 * i]);
            mxx = std::max(mxx, pos[2 * i]);
            mny = std::min(mny, pos[2 * i + 1]);
            mxy = std::max(mxy, pos[2 * i + 1]);
            rmax = std::max(rmax, radii[i]);
        }
        double lox = mnx - rmax, loy = mny - rmax, hix = mxx + rmax, hiy = mxy + rmax;
        double sx = std::max(hix - lox, 1e-6), sy = std::max(hiy - loy, 1e-6);
        double px = margin * sx, py = margin * sy;
        double x0 = lox - px, y0 = loy - py, w = sx + 2 * px, h = sy + 2 * py;
        std::string head = "<svg xmlns=\"http://www.w3.org/2000/svg\" viewBox=\"";
        put_f3(head, x0);
        head.push_back(' ');
        put_f3(head, y0);
        head.push_back(' ');
        put_f3(head, w);
        head.push_back(' ');
        put_f3(head, h);
        head += "\">\n";
        Text out;
        out.parts.push_back(std::move(head));
        if (ne > 0 && edges) {  // :114-123, edges under nodes
            double top = 1.0;
            if (mult) {
                top = mult[0];
                for (int64_t e = 1; e < ne; ++e) top = std::max(top, mult[e]);
            }
            Text te = parallel_rows(ne, [&](int64_t lo, int64_t hi, std::string &s) {
                s.reserve((size_t)(hi - lo) * 120);
                for (int64_t e = lo; e < hi; ++e) {
                    int64_t u = edges[2 * e], v = edges[2 * e + 1];
                    double op = 0.1 + 0.6 * (mult ? mult[e] : 1.0) / top;
                    s += "<line x1=\"";
                    put_f3(s, pos[2 * u]);
                    s += "\" y1=\"";
                    put_f3(s, pos[2 * u + 1]);
                    s += "\" x2=\"";
                    put_f3(s, pos[2 * v]);
                    s += "\" y2=\"";
                    put_f3(s, pos[2 * v + 1]);
                    s += "\" stroke=\"#999999\" stroke-opacity=\"";
                    put_f3(s, op);
                    s += "\" stroke-width=\"0.5\"/>\n";
                }
            });
            for (auto &p : te.parts) out.parts.push_back(std::move(p));
        }
        // :124-128 nodes in (class, index) order: largest classes on top
        std::vector<int64_t> order(n);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](int64_t a, int64_t b) { return classes[a] < classes[b]; });
        Text tn = parallel_rows(n, [&](int64_t lo, int64_t hi, std::string &s) {
            s.reserve((size_t)(hi - lo) * 80);
            for (int64_t k = lo; k < hi; ++k) {
                int64_t i = order[k];
                s += "<circle cx=\"";
                put_f3(s, pos[2 * i]);
                s += "\" cy=\"";
                put_f3(s, pos[2 * i + 1]);
                s += "\" r=\"";
                put_f3(s, radii[i]);
                s += "\" fill=\"";
                s += palette[classes[i]];
                s += "\"/>\n";
            }
        });
        for (auto &p : tn.parts) out.parts.push_back(std::move(p));
        out.parts.push_back("</svg>\n");
        return finish(std::move(out), handle, bytes);
    } catch (...) {
        return CVZ_ERR_OOM;
    }
}

int cvz_text_take(void *handle, char *out) {
    auto *t = static_cast<Text *>(handle);
    if (!t) return CVZ_ERR_VALUE;
    if (out) {
        std::vector<std::thread> pool;
        char *dst = out;
        for (auto &p : t->parts) {
            char *d = dst;
            dst += p.size();
            pool.emplace_back([d, &p] { std::memcpy(d, p.data(), p.size()); });
        }
        for (auto &th : pool) th.join();
    }
    delete t;
    return CVZ_OK;
}

}  // extern "C"
