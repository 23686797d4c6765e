/* C-only client of libcvz_b200.so: shows the C-ABI is usable without Python
 * or torch (plain pointers, cudaMalloc'ed buffers, NULL stream) and checks
 * known answers.  Host entry points run anywhere; `--gpu` adds a small
 * device pipeline: compaction, degrees, degree stats, one deterministic
 * SCoDA pass + resolve, and repulsion of a 2-body system.
 *
 *   gcc abi_smoke.c -I../../include -L<lib dir> -lcvz_b200 [-DWITH_CUDA ...]
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cvz_b200.h"

#ifdef WITH_CUDA
#include <cuda_runtime.h>
#endif

static int fails = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            fprintf(stderr, "FAIL %s:%d: %s (%s)\n", __FILE__, __LINE__, #c, \
                    cvz_last_error());                                  \
            ++fails;                                                    \
        }                                                               \
    } while (0)

static void host_checks(void) {
    CHECK(cvz_version() == 1);
    /* C/graph.py:50-92 line semantics: comments, \r\n, self-loop dropped */
    const char *text = "# comment\n10 20\r\n20 30\n7 7\n";
    void *h = NULL;
    int64_t m = 0, line = 0;
    int code = 0, ntok = 0;
    CHECK(cvz_parse_begin(text, (int64_t)strlen(text), 2, &h, &m, &line, &code, &ntok) == CVZ_OK);
    CHECK(code == 0 && m == 2);
    int64_t pairs[4] = {0};
    CHECK(cvz_parse_take(h, pairs) == CVZ_OK);
    CHECK(pairs[0] == 10 && pairs[1] == 20 && pairs[2] == 20 && pairs[3] == 30);
    /* ParseError: wrong token count names the 1-based line */
    const char *bad = "1 2\n\n3\n";
    CHECK(cvz_parse_begin(bad, (int64_t)strlen(bad), 1, &h, &m, &line, &code, &ntok) == CVZ_OK);
    CHECK(code == 1 && line == 3 && ntok == 1);
    /* C/community.py:164-195 make_schedule(10, 3, seed=5): numpy's PCG64
     * state for default_rng(5), replayed natively */
    int64_t order[10];
    const int64_t want_random[10] = {6, 7, 0, 8, 3, 4, 5, 1, 9, 2};
    const int64_t want_rr[10] = {0, 3, 6, 1, 4, 7, 2, 5, 8, 9};
    CHECK(cvz_make_schedule(10, 3, 0, 0xe500c1d129ce9183ull, 0xd973b921e554efeeull,
                            0xaf6f7b8c936ab4a4ull, 0x4f020b7b2d10234dull, 0, 0, order) == CVZ_OK);
    CHECK(memcmp(order, want_random, sizeof(order)) == 0);
    CHECK(cvz_make_schedule(10, 3, 1, 0, 0, 0, 0, 0, 0, order) == CVZ_OK);
    CHECK(memcmp(order, want_rr, sizeof(order)) == 0);
    /* C/supergraph.py:79-83 supernodes.tsv rows */
    int64_t comm[2] = {0, 3}, weight[2] = {7, 8};
    int kinds[3] = {2, 0, 0};
    const void *cols[3] = {NULL, comm, weight};
    int64_t nbytes = 0;
    CHECK(cvz_format_table(2, 3, kinds, cols, '\t', &h, &nbytes) == CVZ_OK);
    char buf[64] = {0};
    CHECK(nbytes == (int64_t)strlen("0\t0\t7\n1\t3\t8\n"));
    CHECK(cvz_text_take(h, buf) == CVZ_OK);
    CHECK(strcmp(buf, "0\t0\t7\n1\t3\t8\n") == 0);
    /* bad arguments come back as status codes, never as crashes */
    CHECK(cvz_make_schedule(-1, 2, 0, 0, 0, 0, 0, 0, 0, order) == CVZ_ERR_VALUE);
}

#ifdef WITH_CUDA
static void gpu_checks(void) {
    /* two triangles joined by one edge, a self-loop to drop (C/graph.py:117) */
    const int64_t e_h[] = {0, 1, 1, 2, 2, 0, 3, 4, 4, 5, 5, 3, 2, 3, 4, 4};
    const int64_t m_in = 8;
    int64_t *e_d, *scal, *deg, *stats, *lab, *cnt;
    int32_t *e32;
    cudaMalloc((void **)&e_d, sizeof(e_h));
    cudaMalloc((void **)&e32, m_in * 2 * sizeof(int32_t));
    cudaMalloc((void **)&scal, 2 * sizeof(int64_t));
    cudaMemcpy(e_d, e_h, sizeof(e_h), cudaMemcpyHostToDevice);
    CHECK(cvz_edges_compact(e_d, 0, m_in, e32, scal, scal + 1, 1, NULL) == CVZ_OK);
    int64_t sh[2];
    cudaMemcpy(sh, scal, sizeof(sh), cudaMemcpyDeviceToHost);
    CHECK(sh[0] == 7 && sh[1] == 5); /* 7 edges kept, max id 5 -> n = 6 */
    const int64_t n = 6, m = 7;
    cudaMalloc((void **)&deg, n * sizeof(int64_t));
    CHECK(cvz_degree_count(e32, m, n, deg, NULL) == CVZ_OK);
    int64_t dh[6];
    cudaMemcpy(dh, deg, sizeof(dh), cudaMemcpyDeviceToHost);
    CHECK(dh[0] == 2 && dh[2] == 3 && dh[3] == 3 && dh[5] == 2);
    cudaMalloc((void **)&stats, 3 * sizeof(int64_t));
    CHECK(cvz_degree_stats(deg, n, stats, NULL) == CVZ_OK);
    int64_t st[3];
    cudaMemcpy(st, stats, sizeof(st), cudaMemcpyDeviceToHost);
    CHECK(st[0] == 2 && st[1] == 14 && st[2] == 3); /* mode, sum, max */
    /* one deterministic pass at threshold 2 from fresh labels / counters */
    int64_t l0[6] = {0, 1, 2, 3, 4, 5}, c0[6] = {0};
    cudaMalloc((void **)&lab, n * sizeof(int64_t));
    cudaMalloc((void **)&cnt, n * sizeof(int64_t));
    cudaMemcpy(lab, l0, sizeof(l0), cudaMemcpyHostToDevice);
    cudaMemcpy(cnt, c0, sizeof(c0), cudaMemcpyHostToDevice);
    CHECK(cvz_scoda_pass(e32, m, NULL, n, 2, 0, CVZ_SCODA_DETERMINISTIC, cnt, lab, NULL, NULL) ==
          CVZ_OK);
    int64_t lh[6];
    cudaMemcpy(lh, lab, sizeof(lh), cudaMemcpyDeviceToHost);
    /* every resolved label is one of its own members (C/community.py:123-161) */
    for (int i = 0; i < 6; ++i) CHECK(lh[lh[i]] == lh[i]);
    CHECK(lh[0] == lh[1]); /* the first edge merges (test_community.py:80-84) */
    /* C/layout.py:235-243 pair repulsion: bodies 2 apart, masses 1 -> 80/2 = 40 */
    double pos_h[4] = {-1.0, 0.0, 1.0, 0.0}, mass_h[2] = {1.0, 1.0}, out_h[4];
    double *pos, *mass, *out;
    cudaMalloc((void **)&pos, sizeof(pos_h));
    cudaMalloc((void **)&mass, sizeof(mass_h));
    cudaMalloc((void **)&out, sizeof(out_h));
    cudaMemcpy(pos, pos_h, sizeof(pos_h), cudaMemcpyHostToDevice);
    cudaMemcpy(mass, mass_h, sizeof(mass_h), cudaMemcpyHostToDevice);
    CHECK(cvz_repulsion(pos, mass, 2, 80.0, 0.5, out, NULL) == CVZ_OK);
    cudaMemcpy(out_h, out, sizeof(out_h), cudaMemcpyDeviceToHost);
    CHECK(out_h[0] == -40.0 && out_h[2] == 40.0 && out_h[1] == 0.0);
    CHECK(cvz_launch_count() > 0);
    cudaFree(e_d);
    cudaFree(e32);
    cudaFree(scal);
    cudaFree(deg);
    cudaFree(stats);
    cudaFree(lab);
    cudaFree(cnt);
    cudaFree(pos);
    cudaFree(mass);
    cudaFree(out);
}
#endif

int main(int argc, char **argv) {
    host_checks();
#ifdef WITH_CUDA
    if (argc > 1 && strcmp(argv[1], "--gpu") == 0) gpu_checks();
#else
    (void)argc;
    (void)argv;
#endif
    if (fails) {
        fprintf(stderr, "%d check(s) failed\n", fails);
        return 1;
    }
    printf("c-abi smoke ok\n");
    return 0;
}
