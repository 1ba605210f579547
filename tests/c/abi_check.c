/* abi_check.c -- a plain C11 program compiled against include/duhl.h and linked with
 * libduhl.so (tests/test_abi.py).  Without a GPU (argv[1] = "0") it checks that
 * duhl_create fails cleanly with DUHL_E_CUDA and that the host-only calls work; with
 * a B200 (argv[1] = "1") it solves the P1 worked example (A = I2,
 * b = (1, 1), lambda = 1/4, so alpha* = (1/2, 1/2), P:758 / P:852) through duhl_solve
 * with a per-round callback, and reads the state and the working set back. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "duhl.h"

static int rounds_seen = 0;
static void on_round(const duhl_round_record* rec, void* user) {
    (void)user;
    if (rec->round == rounds_seen) ++rounds_seen;
}

#define REQUIRE(c)                                                  \
    do {                                                            \
        if (!(c)) {                                                 \
            fprintf(stderr, "abi_check: %s failed (line %d)\n", #c, __LINE__); \
            return 1;                                               \
        }                                                           \
    } while (0)

int main(int argc, char** argv) {
    const int gpu = argc > 1 && atoi(argv[1]) != 0;
    duhl_config cfg;
    duhl_default_config(&cfg);
    REQUIRE(cfg.cert_every == 10 && cfg.scd_exact == 1 && cfg.refresh_fraction == 0.05);
    duhl_group* g = NULL;
    REQUIRE(duhl_group_create(2, &g) == DUHL_OK && g != NULL);
    REQUIRE(duhl_group_destroy(g) == DUHL_OK);
    REQUIRE(duhl_group_create(0, &g) == DUHL_E_INVALID);

    const float a[4] = {1.0f, 0.0f, 0.0f, 1.0f}; /* column-major A = I2 */
    const double b[2] = {1.0, 1.0};
    duhl_matrix A = {2, 2, a, 2};
    duhl_ctx* ctx = NULL;
    REQUIRE(duhl_create(&A, b, -1.0, DUHL_LASSO, &cfg, &ctx) == DUHL_E_INVALID && ctx == NULL);
    cfg.cert_every = 1;
    duhl_status st = duhl_create(&A, b, 0.25, DUHL_LASSO, &cfg, &ctx);
    if (!gpu) {
        REQUIRE(st == DUHL_E_CUDA && ctx == NULL);
        printf("abi_check ok (no GPU: duhl_create -> DUHL_E_CUDA)\n");
        return 0;
    }
    REQUIRE(st == DUHL_OK && ctx != NULL);
    REQUIRE(duhl_set_trace_callback(ctx, on_round, NULL) == DUHL_OK);
    int64_t rounds = 0;
    double gap = -1.0;
    st = duhl_solve(ctx, 1e-12, 20, 1, DUHL_SEL_GAP, NULL, 0, &rounds, &gap);
    REQUIRE(st == DUHL_OK && gap <= 1e-12 && rounds >= 1 && rounds_seen == rounds);
    double alpha[2], v[2], z[2];
    REQUIRE(duhl_get_state(ctx, alpha, v, z) == DUHL_OK);
    REQUIRE(fabs(alpha[0] - 0.5) < 1e-12 && fabs(alpha[1] - 0.5) < 1e-12);
    double G, O, D;
    REQUIRE(duhl_duality_gap(ctx, &G, &O, &D) == DUHL_OK && fabs(O - 0.375) < 1e-12);
    int64_t P[2], m = 0;
    REQUIRE(duhl_get_working_set(ctx, P, 2, &m) == DUHL_OK && m == 2 && P[0] == 0 && P[1] == 1);
    REQUIRE(duhl_get_working_set(ctx, P, 1, &m) == DUHL_E_INVALID);
    int64_t launches = 0, h2d = 0, zc = 0, upd = 0, d2h = 0;
    REQUIRE(duhl_get_counters(ctx, &launches, &h2d, &zc, &upd, &d2h) == DUHL_OK && launches > 0 && d2h > 0);
    REQUIRE(duhl_destroy(ctx) == DUHL_OK);
    printf("abi_check ok (P1 solved in %lld rounds, O* = %.6f)\n", (long long)rounds, O);
    return 0;
}
