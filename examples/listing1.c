/* Listing 1 of the paper through the C-ABI, from plain C:
 *   #pragma acc data copyout(x[0:N]) present(y)
 *   #pragma acc parallel loop
 *   for (int i = 0; i < N; i++) x[i] = y[i] * y[i];
 * distributed over `n` logical devices (argv[1], default 2; all on GPU 0
 * unless JACC_DISTINCT is set), then a Jacobi-2D timestep with a HALO merge
 * and a dot reduction.  Prints "x = 1 4 9", the dot and "ok". */
#include <stdio.h>
#include <stdlib.h>

#include "jacc.h"

#define CHECK(call)                                                              \
    do {                                                                         \
        jacc_status st_ = (call);                                                \
        if (st_ != JACC_OK) {                                                    \
            fprintf(stderr, "%s -> %s\n", #call, jacc_error_string(st_));        \
            return 1;                                                            \
        }                                                                        \
    } while (0)

int main(int argc, char **argv) {
    int n = argc > 1 ? atoi(argv[1]) : 2;
    int ids[JACC_MAX_DEVICES];
    for (int d = 0; d < n; d++) ids[d] = getenv("JACC_DISTINCT") ? d : 0;
    CHECK(jacc_init(n, ids));

    float y[3] = {1, 2, 3}, x[3] = {0, 0, 0};
    int64_t e3 = 3;
    CHECK(jacc_data_create(y, sizeof y, sizeof(float), 1, &e3));
    CHECK(jacc_data_create(x, sizeof x, sizeof(float), 1, &e3));
    CHECK(jacc_update_device(y, 0, sizeof y));
    jacc_range r = {1, {0, 0, 0}, {3, 0, 0}};
    jacc_arg sq[2] = {{JACC_ARG_ARRAY_IN, y, 0, 0}, {JACC_ARG_ARRAY_OUT, x, 0, 0}};
    CHECK(jacc_launch(JACC_LOOP_SQUARE_F32, &r, sq, 2, -1));
    CHECK(jacc_update_host(x, 0, sizeof x));
    printf("x = %g %g %g\n", x[0], x[1], x[2]);

    enum { N = 64 };
    static double A[N][N], B[N][N];
    for (int i = 0; i < N; i++)
        for (int j = 0; j < N; j++) A[i][j] = B[i][j] = 3.0 * i + 7.0 * j + 11.0;  /* harmonic */
    int64_t e2[2] = {N, N};
    CHECK(jacc_set_merge_policy(JACC_MERGE_HALO));
    CHECK(jacc_data_create(A, sizeof A, sizeof(double), 2, e2));
    CHECK(jacc_data_create(B, sizeof B, sizeof(double), 2, e2));
    CHECK(jacc_update_device(A, 0, sizeof A));
    CHECK(jacc_update_device(B, 0, sizeof B));
    jacc_arg ab[2] = {{JACC_ARG_ARRAY_IN, A, 0, 0}, {JACC_ARG_ARRAY_OUT, B, 0, 0}};
    jacc_arg ba[2] = {{JACC_ARG_ARRAY_IN, B, 0, 0}, {JACC_ARG_ARRAY_OUT, A, 0, 0}};
    CHECK(jacc_launch(JACC_LOOP_JACOBI2D_F64, NULL, ab, 2, 0));
    CHECK(jacc_launch(JACC_LOOP_JACOBI2D_F64, NULL, ba, 2, 0));
    CHECK(jacc_update_host(A, 0, sizeof A));
    int bad = 0;
    for (int i = 0; i < N; i++)
        for (int j = 0; j < N; j++) bad += A[i][j] != 3.0 * i + 7.0 * j + 11.0;

    double s = 0.5;
    int64_t en = (int64_t)N * N;
    jacc_range rd = {1, {0, 0, 0}, {en, 0, 0}};
    jacc_arg dot[3] = {{JACC_ARG_ARRAY_IN, A, 0, 0}, {JACC_ARG_ARRAY_IN, B, 0, 0},
                       {JACC_ARG_REDUCE_SUM_F64, &s, 0, 0}};
    CHECK(jacc_launch(JACC_LOOP_DOT_F64, &rd, dot, 3, -1));
    printf("dot = %.17g\n", s);
    CHECK(jacc_finalize());
    printf(bad == 0 && x[0] == 1 && x[1] == 4 && x[2] == 9 ? "ok\n" : "FAIL\n");
    return bad != 0;
}
