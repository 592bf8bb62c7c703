/* abi_client.c -- a plain C user of include/qsim.h (no Python, no torch):
 * Bell/GHZ + adder + permutation checks through the C-ABI only.
 * Exit code 0 = all checks passed. */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "qsim.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        qsim_status s_ = (call);                                                     \
        if (s_ != QSIM_OK) {                                                         \
            fprintf(stderr, "%s -> %s (%s)\n", #call, qsim_status_str(s_), qsim_last_error(ctx)); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(void)
{
    const double r = 1.0 / sqrt(2.0);
    const qsim_c128 H[4] = {{r, 0}, {r, 0}, {r, 0}, {-r, 0}};
    const qsim_c128 X[4] = {{0, 0}, {1, 0}, {1, 0}, {0, 0}};
    qsim_ctx ctx = NULL;
    const int n = 14;
    CHECK(qsim_create(n, 1, &ctx));
    /* GHZ: H(0), CNOT(0 -> i) for every i */
    CHECK(qsim_init_basis(ctx, 0));
    CHECK(qsim_apply_1q(ctx, 0, H));
    for (int i = 1; i < n; i++) {
        int c = 0;
        CHECK(qsim_apply_controlled(ctx, &c, 1, i, X));
    }
    qsim_c128 a[2];
    CHECK(qsim_get_amplitudes(ctx, 0, 1, &a[0]));
    CHECK(qsim_get_amplitudes(ctx, (1ULL << n) - 1, 1, &a[1]));
    if (fabs(a[0].re - r) > 1e-15 || fabs(a[1].re - r) > 1e-15) {
        fprintf(stderr, "GHZ amplitudes wrong: %g %g\n", a[0].re, a[1].re);
        return 2;
    }
    double ex[14];
    CHECK(qsim_expectations(ctx, ex));
    for (int i = 0; i < n; i++)
        if (fabs(ex[i] - 0.5) > 1e-14) return 3;
    /* controlled permutation: |c=1, w> -> |c=1, w+3 mod 8> on qubits 3,4,5 */
    uint32_t perm[8];
    for (int w = 0; w < 8; w++) perm[w] = (uint32_t)((w + 3) % 8);
    int tg[3] = {3, 4, 5}, ct[1] = {0};
    CHECK(qsim_init_basis(ctx, 1 | (2 << 3)));            /* c = 1, w = 2 */
    CHECK(qsim_apply_perm(ctx, ct, 1, tg, 3, perm));
    double p[8];
    CHECK(qsim_probabilities(ctx, tg, 3, p));
    if (fabs(p[5] - 1.0) > 1e-15) return 4;
    /* errors are reported, state untouched */
    const qsim_c128 bad[4] = {{1, 0}, {1, 0}, {0, 0}, {1, 0}};
    if (qsim_apply_1q(ctx, 0, bad) != QSIM_ERR_NOT_UNITARY) return 5;
    if (qsim_apply_1q(ctx, n, H) != QSIM_ERR_QUBIT_RANGE) return 6;
    CHECK(qsim_probabilities(ctx, tg, 3, p));
    if (fabs(p[5] - 1.0) > 1e-15) return 7;
    qsim_stats st;
    CHECK(qsim_get_stats(ctx, &st));
    printf("abi_client ok: gates=%llu passes=%llu kernels=%llu\n", (unsigned long long)st.gates,
           (unsigned long long)st.passes, (unsigned long long)st.kernel_launches);
    CHECK(qsim_destroy(ctx));
    /* the SPMD shorthand with one rank: a LOCAL context */
    qsim_ctx c1 = NULL;
    if (qsim_create_rank(10, 3, 0, NULL, NULL, 0, NULL, 0, NULL, &c1) != QSIM_ERR_ARG) return 8;
    CHECK(qsim_create_rank(10, 1, 0, NULL, NULL, 0, NULL, 0, NULL, &c1));
    CHECK(qsim_init_basis(c1, 0));
    for (int q = 0; q < 10; q++) CHECK(qsim_apply_1q(c1, q, H));
    double nrm;
    CHECK(qsim_probabilities(c1, NULL, 0, &nrm));
    CHECK(qsim_get_amplitudes(c1, 1023, 1, &a[0]));
    if (fabs(nrm - 1.0) > 1e-14 || fabs(a[0].re - 1.0 / 32.0) > 1e-15) return 9;
    CHECK(qsim_destroy(c1));
    /* whole-register sampling of a 26-qubit GHZ state (k = n > 24: the
     * two-level sampler): every shot is all zeros or all ones, both occur */
    qsim_ctx c2 = NULL;
    const int n2 = 26;
    CHECK(qsim_create(n2, 1, &c2));
    CHECK(qsim_init_basis(c2, 0));
    CHECK(qsim_apply_1q(c2, 0, H));
    for (int i = 1; i < n2; i++) {
        int c = 0;
        CHECK(qsim_apply_controlled(c2, &c, 1, i, X));
    }
    int all[26];
    for (int i = 0; i < n2; i++) all[i] = i;
    uint64_t shots[64];
    CHECK(qsim_measure(c2, all, n2, 7, 64, shots));
    int zeros = 0, ones = 0;
    for (int s = 0; s < 64; s++) {
        if (shots[s] == 0) zeros++;
        else if (shots[s] == (1ULL << n2) - 1) ones++;
        else return 10;
    }
    if (!zeros || !ones) return 11;
    CHECK(qsim_destroy(c2));
    /* roofline denominators of this device */
    double f64 = 0, gbs = 0;
    if (qsim_probe_peaks(&f64, &gbs) != QSIM_OK || f64 < 1.0 || gbs < 100.0) return 12;
    printf("abi_client two-level ok: zeros=%d ones=%d fp64=%.1f TF copy=%.0f GB/s\n", zeros, ones, f64, gbs);
    return 0;
}
