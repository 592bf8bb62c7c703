/*
 * qsim_oracle.c -- plain sequential-definition CPU state-vector simulator.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product path in
 * paper_quant_ph_0608239_b200/ (DESIGN.md §4).
 *
 * What it computes: psi <- U_G ... U_1 psi_0 exactly as the paper's update
 * rules state them, one gate at a time, on ONE array of 2^n complex128
 * amplitudes (re, im interleaved), qubit 0 = least-significant index bit
 * (PAPER.md P:150-183).  No tiling, sharding, fusion, reordering or qubit
 * permutation.  OpenMP parallelises only the independent
 * outer loops; the arithmetic per amplitude is the textbook formula.
 *
 * Pins (tests/test_oracle_pins.py): dense Kronecker operators (n <= 6), the
 * paper's worked examples (Eqs. Hadamard..Toffoli), H-on-all,
 * the QFT closed form, the QFT adder, the corrected Shor closed form p_k(r)
 * and Table III, fsum for the probability sums, and the sampler
 * rule on hand-made distributions.  Every function below is pinned.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define RE(p, i) (p)[2 * (i)]
#define IM(p, i) (p)[2 * (i) + 1]

/* INITIAL STATE x (Appendix A): |x> */
void or_init_basis(double *psi, int n, uint64_t x)
{
    uint64_t D = 1ULL << n;
    memset(psi, 0, 2 * D * sizeof(double));
    RE(psi, x) = 1.0;
}

/*
 * Controlled 2x2 gate.  u = [u00r,u00i,u01r,u01i,u10r,u10i,u11r,u11i].
 * For every index i with bit t = 0 and all control bits = 1, with j = i|2^t:
 *   a'_i = u00 a_i + u01 a_j,   a'_j = u10 a_i + u11 a_j.
 * nc = 0 gives Eqs. NUM2-NUM5 for any U; nc = 1 gives CNOT
 * (NUM6), controlled phase (COMM5) and controlled-V
 * (NUM7); nc = 2 gives Toffoli (NUM8).
 */
void or_apply_controlled(double *psi, int n, const int *ctrl, int nc, int t, const double *u)
{
    uint64_t D = 1ULL << n, tb = 1ULL << t, cm = 0;
    for (int k = 0; k < nc; k++) cm |= 1ULL << ctrl[k];
    #pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)D; ii++) {
        uint64_t i = (uint64_t)ii;
        if (i & tb) continue;
        if ((i & cm) != cm) continue;
        uint64_t j = i | tb;
        double ar = RE(psi, i), ai = IM(psi, i), br = RE(psi, j), bi = IM(psi, j);
        RE(psi, i) = u[0] * ar - u[1] * ai + u[2] * br - u[3] * bi;
        IM(psi, i) = u[0] * ai + u[1] * ar + u[2] * bi + u[3] * br;
        RE(psi, j) = u[4] * ar - u[5] * ai + u[6] * br - u[7] * bi;
        IM(psi, j) = u[4] * ai + u[5] * ar + u[6] * bi + u[7] * br;
    }
}

void or_apply_1q(double *psi, int n, int q, const double *u)
{
    or_apply_controlled(psi, n, NULL, 0, q, u);
}

/* scatter the bits of w onto the positions pos[0..k-1] */
static uint64_t scatter(uint64_t w, const int *pos, int k)
{
    uint64_t r = 0;
    for (int b = 0; b < k; b++)
        if ((w >> b) & 1) r |= 1ULL << pos[b];
    return r;
}

/*
 * Controlled permutation of a target register (the "conditional operation"
 * of Shor step 2; reading 7): for every base index b whose
 * target bits are 0 and control bits are 1,
 *   a'[b | scatter_T(perm[w])] = a[b | scatter_T(w)]   for all w < 2^nt.
 * Returns -1 if perm is not a bijection of [0, 2^nt).
 */
int or_apply_perm(double *psi, int n, const int *ctrl, int nc, const int *tg, int nt,
                  const uint32_t *perm)
{
    uint64_t D = 1ULL << n, W = 1ULL << nt, tm = 0, cm = 0;
    for (int k = 0; k < nt; k++) tm |= 1ULL << tg[k];
    for (int k = 0; k < nc; k++) cm |= 1ULL << ctrl[k];
    char *seen = calloc(W, 1);
    for (uint64_t w = 0; w < W; w++) {
        if (perm[w] >= W || seen[perm[w]]) { free(seen); return -1; }
        seen[perm[w]] = 1;
    }
    free(seen);
    #pragma omp parallel
    {
        double *v = malloc(2 * W * sizeof(double));
        #pragma omp for schedule(static)
        for (int64_t bb = 0; bb < (int64_t)D; bb++) {
            uint64_t b = (uint64_t)bb;
            if (b & tm) continue;
            if ((b & cm) != cm) continue;
            for (uint64_t w = 0; w < W; w++) {
                uint64_t i = b | scatter(w, tg, nt);
                v[2 * w] = RE(psi, i);
                v[2 * w + 1] = IM(psi, i);
            }
            for (uint64_t w = 0; w < W; w++) {
                uint64_t i = b | scatter(perm[w], tg, nt);
                RE(psi, i) = v[2 * w];
                IM(psi, i) = v[2 * w + 1];
            }
        }
        free(v);
    }
    return 0;
}

/* SWAP of qubits a and b: exchange the two bit values of every index. */
void or_swap(double *psi, int n, int a, int b)
{
    uint64_t D = 1ULL << n, ab = 1ULL << a, bbit = 1ULL << b;
    #pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < (int64_t)D; ii++) {
        uint64_t i = (uint64_t)ii;
        if ((i & ab) && !(i & bbit)) {
            uint64_t j = i ^ ab ^ bbit;
            double r = RE(psi, i), m = IM(psi, i);
            RE(psi, i) = RE(psi, j); IM(psi, i) = IM(psi, j);
            RE(psi, j) = r; IM(psi, j) = m;
        }
    }
}

/* pairwise (recursive-halving) sum of |a_i|^2 over i = base | scatter(j, rest)
 * for j in [lo, hi); leaves of 8 summed left to right. */
static double pw_sum(const double *psi, uint64_t base, const int *rest, int nr,
                     uint64_t lo, uint64_t hi)
{
    if (hi - lo <= 8) {
        double s = 0.0;
        for (uint64_t j = lo; j < hi; j++) {
            uint64_t i = base | scatter(j, rest, nr);
            s += RE(psi, i) * RE(psi, i) + IM(psi, i) * IM(psi, i);
        }
        return s;
    }
    uint64_t mid = lo + (hi - lo) / 2;
    return pw_sum(psi, base, rest, nr, lo, mid) + pw_sum(psi, base, rest, nr, mid, hi);
}

/*
 * Marginal probabilities over the listed qubits (Born rule):
 *   p[beta] = sum_{i : bits_Q(i) = beta} |a_i|^2, bit b of beta <-> qubit qs[b].
 * k = 0 gives the norm (Eq. STAT1).  Pairwise summation in fixed
 * index order.
 */
void or_probabilities(const double *psi, int n, const int *qs, int k, double *out)
{
    int rest[64], nr = 0;
    uint64_t qm = 0;
    for (int b = 0; b < k; b++) qm |= 1ULL << qs[b];
    for (int p = 0; p < n; p++)
        if (!((qm >> p) & 1)) rest[nr++] = p;
    uint64_t B = 1ULL << k, J = 1ULL << nr;
    if (B >= 64) {
        #pragma omp parallel for schedule(dynamic, 16)
        for (int64_t beta = 0; beta < (int64_t)B; beta++)
            out[beta] = pw_sum(psi, scatter((uint64_t)beta, qs, k), rest, nr, 0, J);
    } else {
        /* split each bin's pairwise tree at its top 6 levels: identical result */
        int split = nr < 6 ? nr : 6;
        uint64_t S = 1ULL << split, blk = J >> split;
        double *part = malloc(B * S * sizeof(double));
        #pragma omp parallel for collapse(2) schedule(static)
        for (int64_t beta = 0; beta < (int64_t)B; beta++)
            for (int64_t s = 0; s < (int64_t)S; s++)
                part[beta * S + s] = pw_sum(psi, scatter((uint64_t)beta, qs, k), rest, nr,
                                            (uint64_t)s * blk, (uint64_t)(s + 1) * blk);
        for (uint64_t beta = 0; beta < B; beta++) {
            uint64_t w = S;
            double *p = part + beta * S;
            while (w > 1) {
                for (uint64_t s = 0; s < w / 2; s++) p[s] = p[2 * s] + p[2 * s + 1];
                w /= 2;
            }
            out[beta] = p[0];
        }
        free(part);
    }
}

/* <Q_i> = sum_k p_k k_i (Eq. Shor7) for every qubit i. */
void or_expectations(const double *psi, int n, double *out)
{
    for (int q = 0; q < n; q++) {
        double p[2];
        or_probabilities(psi, n, &q, 1, p);
        out[q] = p[1];
    }
}

/* SplitMix64 finaliser (reading 14) */
static uint64_t or_sm64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/*
 * Non-collapsing sampling by inverse CDF (reading 14):
 *   C(beta) = p[0] + ... + p[beta] summed left to right;
 *   u_s = (sm64(seed + (s+1)*G) >> 11) * 2^-53 * C(B-1);
 *   outcome_s = min{beta : C(beta) > u_s};
 *   tie[s] = 1 if u_s lies within 1e-12 of a CDF boundary adjacent to it.
 */
void or_sample(const double *p, int k, uint64_t seed, uint64_t nshots, uint64_t *out, uint8_t *tie)
{
    uint64_t B = 1ULL << k;
    double *C = malloc(B * sizeof(double));
    double acc = 0.0;
    for (uint64_t b = 0; b < B; b++) { acc += p[b]; C[b] = acc; }
    for (uint64_t s = 0; s < nshots; s++) {
        uint64_t r = or_sm64(seed + (s + 1) * 0x9E3779B97F4A7C15ULL);
        double u = (double)(r >> 11) * (1.0 / 9007199254740992.0) * C[B - 1];
        uint64_t beta = 0;
        while (beta < B - 1 && !(C[beta] > u)) beta++;
        out[s] = beta;
        int t = fabs(C[beta] - u) < 1e-12;
        if (beta > 0 && fabs(u - C[beta - 1]) < 1e-12) t = 1;
        if (tie) tie[s] = (uint8_t)t;
    }
    free(C);
}

int or_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
