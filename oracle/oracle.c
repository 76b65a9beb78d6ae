/*
 * oracle.c -- fp64 CPU ORACLE for arXiv 2106.00003 (Hamze, "Parallelized Computation and
 * Backpropagation Under Angle-Parametrized Orthogonal Matrices").
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2106_00003_b200/) never imports, links or executes anything here, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Everything is the plain definition, in fp64, in the paper's order and notation:
 *   - schedule: the circle method simulated literally on a list (Fig. 1
 *     PAPER.md:378-455; odd n: PAPER.md:457-464);
 *   - forward: Algorithm 1 over the round-robin sequence E, i.e.
 *     U = prod_{e in E} G^e(theta_e) with G^{e_N} applied first;
 *   - backward: textbook reverse-mode differentiation of Algorithm 1 with a stored tape of
 *     every rotation's inputs (chain rule on y_i = c a_i - s a_j, y_j = s a_i + c a_j).
 *     Deliberately NOT the activation replay the GPU uses.
 *   - Algorithm 3 literally, as a cross-oracle for the U-build gradient.
 * Columns of X are independent in Y = U X (each column is Alg. 1 applied to that column), so
 * columns may be processed in any grouping; no element sees any reordering of its own
 * arithmetic. cos/sin are fp64 libm of the fp32 theta promoted to fp64 (reading R11).
 * Masked angles and bye pairs are bypassed.
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC (no FMA contraction,
 * so results are bitwise reproducible across builds).
 *
 * Pins: see tests/test_oracle_pins.py (paper Eq. (5), SPEC n=4 example, paper §5 n=8/m=4
 * list, closed forms, invariants, dense explicit products, finite differences).
 *
 * Layout options: every schedule-consuming function takes
 *   perm  -- the circle method's initial sequence ("Beginning with an arbitrary
 *            permutation of the coordinate sequence"), a permutation of
 *            0..n_eff-1 (odd n: it includes the bye index n); NULL = identity (Fig. 1);
 *   refl  -- reflection (det -1) by "negating an arbitrary fixed column following the
 *            construction": U' = U with column refl negated; -1 = none.
 *            Y = U' X = U (D X) with D = diag(.., -1 at refl, ..); U'^T X = D (U^T X).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int n_eff_of(int n) { return (n % 2) ? n + 1 : n; }

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int64_t oracle_num_angles(int n) { return n < 2 ? -1 : (int64_t)n * (n - 1) / 2; }

/*
 * Circle method, literally (PAPER.md:370-377 and Fig. 1): start from the sequence
 * (0, 1, ..., n_eff-1); the block is obtained by pairing the elements at equal distance from
 * the two ends; the next sequence holds the first element fixed and shifts the remaining
 * n_eff-1 elements by one modulo n_eff-1 -- the direction is the one Fig. 1 shows:
 * (0,1,2,3,4,5) -> (0,5,1,2,3,4).
 * Odd n: augment with index n; pairs with j == n are bypassed and get no
 * angle (flat = -1).
 * Outputs: pairs[R][S][2] with i < j ("(i,j) with i<j"), and flat[R][S] = index
 * of the angle in theta (block-major: b_1 first, pairs in listed order), or -1.
 * Either output may be NULL. Returns the number of real pairs (n(n-1)/2), or -1.
 */
int64_t oracle_schedule(int n, const int32_t *perm, int32_t *pairs, int64_t *flat) {
    if (n < 2) return -1;
    int ne = n_eff_of(n);
    int R = ne - 1, S = ne / 2;
    if (perm) { /* must be a permutation of 0..ne-1 */
        char *seen = (char *)calloc(ne, 1);
        int ok = 1;
        for (int p = 0; p < ne; p++) {
            if (perm[p] < 0 || perm[p] >= ne || seen[perm[p]]) ok = 0;
            else seen[perm[p]] = 1;
        }
        free(seen);
        if (!ok) return -1;
    }
    int *seq = (int *)malloc(sizeof(int) * ne);
    int *nxt = (int *)malloc(sizeof(int) * ne);
    for (int p = 0; p < ne; p++) seq[p] = perm ? perm[p] : p;
    int64_t f = 0;
    for (int r = 0; r < R; r++) {
        for (int k = 0; k < S; k++) {
            int a = seq[k], b = seq[ne - 1 - k];
            int i = a < b ? a : b, j = a < b ? b : a;
            if (pairs) { pairs[((int64_t)r * S + k) * 2] = i; pairs[((int64_t)r * S + k) * 2 + 1] = j; }
            int64_t idx = (j == n) ? -1 : f++;   /* j == n only for the odd-n bye (n_eff = n+1) */
            if (flat) flat[(int64_t)r * S + k] = idx;
        }
        /* hold seq[0], rotate the last ne-1 elements right by one: (0,1,2,3,4,5)->(0,5,1,2,3,4) */
        nxt[0] = seq[0];
        if (ne > 1) nxt[1] = seq[ne - 1];
        for (int p = 2; p < ne; p++) nxt[p] = seq[p - 1];
        memcpy(seq, nxt, sizeof(int) * ne);
    }
    free(seq); free(nxt);
    return f;
}

/* The sequence E as a flat list of the real pairs in angle order. */
static int32_t *build_E(int n, const int32_t *perm, int64_t *N_out) {
    int ne = n_eff_of(n);
    int R = ne - 1, S = ne / 2;
    int32_t *pairs = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)R * S);
    int64_t *flat = (int64_t *)malloc(sizeof(int64_t) * (size_t)R * S);
    int64_t N = oracle_schedule(n, perm, pairs, flat);
    if (N < 0) { free(pairs); free(flat); return NULL; }
    int32_t *E = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)N);
    for (int64_t q = 0; q < (int64_t)R * S; q++) {
        if (flat[q] < 0) continue;
        E[2 * flat[q]] = pairs[2 * q];
        E[2 * flat[q] + 1] = pairs[2 * q + 1];
    }
    free(pairs); free(flat);
    *N_out = N;
    return E;
}

/*
 * Algorithm 1 for a generic pair sequence E[Np][2], in place on the n x m
 * row-major fp64 matrix A (row stride lda):
 *   for e in reversed(E): (i,j) <- e; r_i <- cos*A_i - sin*A_j; r_j <- sin*A_i + cos*A_j.
 * transpose = 1 applies U^T = G^{e_N T} ... G^{e_1 T}: e in E order, each G^T (angle -theta).
 * mask[e] == 0 bypasses e. theta is fp32; cos/sin are fp64 of it.
 */
int oracle_apply_sequence(int n, int64_t m, int64_t Np, const int32_t *E, const float *theta,
                          const uint8_t *mask, double *A, int64_t lda, int transpose) {
    if (n < 1 || m < 0 || Np < 0 || lda < m) return -1;
    for (int64_t q = 0; q < Np; q++) {
        int64_t e = transpose ? q : (Np - 1 - q);
        if (mask && !mask[e]) continue;
        int i = E[2 * e], j = E[2 * e + 1];
        double th = (double)theta[e];
        double c = cos(th), s = sin(th);
        if (transpose) s = -s;
        double *Ai = A + (int64_t)i * lda, *Aj = A + (int64_t)j * lda;
        for (int64_t l = 0; l < m; l++) {
            double ri = c * Ai[l] - s * Aj[l];
            double rj = s * Ai[l] + c * Aj[l];
            Ai[l] = ri;
            Aj[l] = rj;
        }
    }
    return 0;
}

/*
 * Y = U(theta) X (transpose=0) or U^T X (transpose=1) with E the circle-method round-robin
 * sequence. Columns are split into fixed blocks; each block runs Algorithm 1 on its columns.
 * Reflection: the block's row refl is negated before Algorithm 1 (transpose: after).
 */
int oracle_apply(int n, int64_t m, const int32_t *perm, int refl, const float *theta, const uint8_t *mask,
                 const double *X, double *Y, int transpose) {
    if (n < 2 || m < 0 || refl < -1 || refl >= n) return -1;
    int64_t N;
    int32_t *E = build_E(n, perm, &N);
    if (!E) return -1;
    const int64_t CB = 64;
    int64_t nb = (m + CB - 1) / CB;
    int rc = 0;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < nb; b++) {
        int64_t c0 = b * CB, w = (m - c0 < CB) ? (m - c0) : CB;
        double *blk = (double *)malloc(sizeof(double) * (size_t)n * w);
        for (int r = 0; r < n; r++)
            for (int64_t l = 0; l < w; l++) blk[(int64_t)r * w + l] = X[(int64_t)r * m + c0 + l];
        if (refl >= 0 && !transpose)
            for (int64_t l = 0; l < w; l++) blk[(int64_t)refl * w + l] = -blk[(int64_t)refl * w + l];
        if (oracle_apply_sequence(n, w, N, E, theta, mask, blk, w, transpose)) rc = -1;
        if (refl >= 0 && transpose)
            for (int64_t l = 0; l < w; l++) blk[(int64_t)refl * w + l] = -blk[(int64_t)refl * w + l];
        for (int r = 0; r < n; r++)
            for (int64_t l = 0; l < w; l++) Y[(int64_t)r * m + c0 + l] = blk[(int64_t)r * w + l];
        free(blk);
    }
    free(E);
    return rc;
}

/* U = U(theta): Algorithm 1 / 2 starting from U <- I_n. */
int oracle_build_U(int n, const int32_t *perm, int refl, const float *theta, const uint8_t *mask, double *U) {
    if (n < 2) return -1;
    double *I = (double *)calloc((size_t)n * n, sizeof(double));
    for (int r = 0; r < n; r++) I[(int64_t)r * n + r] = 1.0;
    int rc = oracle_apply(n, n, perm, refl, theta, mask, I, U, 0);
    free(I);
    return rc;
}

/*
 * Backward of Y = U(theta) X for a loss L with dY = dL/dY (both n x m row-major):
 *   dtheta[e] = sum over columns of dL/dtheta_e, dX = dL/dX.
 * Per column: run Algorithm 1 storing, for every rotation, its inputs (a_i, a_j) (the tape);
 * then sweep the rotations in reverse application order applying the chain rule to
 *   y_i = c a_i - s a_j,  y_j = s a_i + c a_j:
 *   dL/dtheta += g_i * (-s a_i - c a_j) + g_j * (c a_i - s a_j)
 *   g_i' = c g_i + s g_j,  g_j' = -s g_i + c g_j           (gradient w.r.t. a_i, a_j).
 * Masked angles are not parameters: their dtheta is exactly 0.
 * dtheta is summed in fp64 over columns in increasing column order within each thread's
 * fixed contiguous column range; thread partials are combined in thread order.
 * dX may be NULL. Reflection: the forward starts from D X and dX = D (gradient w.r.t. D X).
 */
int oracle_backward(int n, int64_t m, const int32_t *perm, int refl, const float *theta, const uint8_t *mask,
                    const double *X, const double *dY, double *dX, double *dtheta) {
    if (n < 2 || m < 0 || refl < -1 || refl >= n) return -1;
    int64_t N;
    int32_t *E = build_E(n, perm, &N);
    if (!E) return -1;
    double *cs = (double *)malloc(sizeof(double) * 2 * (size_t)N);
    for (int64_t e = 0; e < N; e++) {
        double th = (double)theta[e];
        cs[2 * e] = cos(th);
        cs[2 * e + 1] = sin(th);
    }
    int nt = oracle_num_threads();
    double *part = (double *)calloc((size_t)nt * N, sizeof(double));
#pragma omp parallel num_threads(nt)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        int64_t c0 = m * t / nt, c1 = m * (t + 1) / nt;
        double *acc = part + (int64_t)t * N;
        double *x = (double *)malloc(sizeof(double) * n);
        double *g = (double *)malloc(sizeof(double) * n);
        double *tape = (double *)malloc(sizeof(double) * 2 * (size_t)N);
        for (int64_t col = c0; col < c1; col++) {
            for (int r = 0; r < n; r++) x[r] = X[(int64_t)r * m + col];
            if (refl >= 0) x[refl] = -x[refl];
            /* forward, Algorithm 1 order: e = e_N, ..., e_1 */
            for (int64_t e = N - 1; e >= 0; e--) {
                if (mask && !mask[e]) continue;
                int i = E[2 * e], j = E[2 * e + 1];
                double c = cs[2 * e], s = cs[2 * e + 1];
                double ai = x[i], aj = x[j];
                tape[2 * e] = ai;
                tape[2 * e + 1] = aj;
                x[i] = c * ai - s * aj;
                x[j] = s * ai + c * aj;
            }
            for (int r = 0; r < n; r++) g[r] = dY[(int64_t)r * m + col];
            /* reverse sweep: e = e_1, ..., e_N */
            for (int64_t e = 0; e < N; e++) {
                if (mask && !mask[e]) continue;
                int i = E[2 * e], j = E[2 * e + 1];
                double c = cs[2 * e], s = cs[2 * e + 1];
                double ai = tape[2 * e], aj = tape[2 * e + 1];
                double gi = g[i], gj = g[j];
                acc[e] += gi * (-s * ai - c * aj) + gj * (c * ai - s * aj);
                g[i] = c * gi + s * gj;
                g[j] = -s * gi + c * gj;
            }
            if (refl >= 0) g[refl] = -g[refl];
            if (dX)
                for (int r = 0; r < n; r++) dX[(int64_t)r * m + col] = g[r];
        }
        free(x); free(g); free(tape);
    }
    for (int64_t e = 0; e < N; e++) {
        double sacc = 0.0;
        for (int t = 0; t < nt; t++) sacc += part[(int64_t)t * N + e];
        dtheta[e] = (mask && !mask[e]) ? 0.0 : sacc;
    }
    free(part); free(cs); free(E);
    return 0;
}

/*
 * Algorithm 3 "Parallel JVP", literally, sequentially:
 *   U^fwd <- U, M <- Gamma^T, A <- n/2 x n (the "N/2 x N" at PAPER.md:802 is
 *   read as n/2 x n, reading R7);
 *   for b in reversed(B):
 *     U^fwd columns i,j <- c U_:i - s U_:j, s U_:i + c U_:j
 *     M rows i,j        <- c M_i: - s M_j:, s M_i: + c M_j:
 *     A_{m(e) l} <- M_il u_lj - M_jl u_li   (u_lj = U^fwd[l][j])
 *     d <- A 1;  dL/dtheta_e <- d_{m(e)}
 * m(e) = slot index of e in its block. Bye (j == n) and masked pairs are bypassed.
 */
int oracle_alg3(int n, const int32_t *perm, const float *theta, const uint8_t *mask, const double *U,
                const double *Gamma, double *dtheta) {
    if (n < 2) return -1;
    int ne = n_eff_of(n);
    int R = ne - 1, S = ne / 2;
    int32_t *pairs = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)R * S);
    int64_t *flat = (int64_t *)malloc(sizeof(int64_t) * (size_t)R * S);
    int64_t N = oracle_schedule(n, perm, pairs, flat);
    if (N < 0) { free(pairs); free(flat); return -1; }
    double *Uf = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *M = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *A = (double *)malloc(sizeof(double) * (size_t)S * n);
    memcpy(Uf, U, sizeof(double) * (size_t)n * n);
    for (int r = 0; r < n; r++)
        for (int l = 0; l < n; l++) M[(int64_t)r * n + l] = Gamma[(int64_t)l * n + r];
    for (int64_t e = 0; e < N; e++) dtheta[e] = 0.0;
    for (int b = R - 1; b >= 0; b--) {          /* b in reversed(B) */
        for (int k = 0; k < S; k++) {           /* parallel U^fwd column update */
            int i = pairs[2 * ((int64_t)b * S + k)], j = pairs[2 * ((int64_t)b * S + k) + 1];
            int64_t f = flat[(int64_t)b * S + k];
            if (f < 0 || (mask && !mask[f])) continue;
            double th = (double)theta[f], c = cos(th), s = sin(th);
            for (int l = 0; l < n; l++) {
                double ui = Uf[(int64_t)l * n + i], uj = Uf[(int64_t)l * n + j];
                Uf[(int64_t)l * n + i] = c * ui - s * uj;
                Uf[(int64_t)l * n + j] = s * ui + c * uj;
            }
        }
        for (int k = 0; k < S; k++) {           /* parallel M row update */
            int i = pairs[2 * ((int64_t)b * S + k)], j = pairs[2 * ((int64_t)b * S + k) + 1];
            int64_t f = flat[(int64_t)b * S + k];
            if (f < 0 || (mask && !mask[f])) continue;
            double th = (double)theta[f], c = cos(th), s = sin(th);
            for (int l = 0; l < n; l++) {
                double mi = M[(int64_t)i * n + l], mj = M[(int64_t)j * n + l];
                M[(int64_t)i * n + l] = c * mi - s * mj;
                M[(int64_t)j * n + l] = s * mi + c * mj;
            }
        }
        for (int k = 0; k < S; k++) {           /* parallel A assignment, m(e) = k */
            int i = pairs[2 * ((int64_t)b * S + k)], j = pairs[2 * ((int64_t)b * S + k) + 1];
            int64_t f = flat[(int64_t)b * S + k];
            if (f < 0 || (mask && !mask[f])) continue;
            for (int l = 0; l < n; l++)
                A[(int64_t)k * n + l] = M[(int64_t)i * n + l] * Uf[(int64_t)l * n + j]
                                      - M[(int64_t)j * n + l] * Uf[(int64_t)l * n + i];
        }
        for (int k = 0; k < S; k++) {           /* d <- A 1, scatter */
            int64_t f = flat[(int64_t)b * S + k];
            if (f < 0 || (mask && !mask[f])) continue;
            double d = 0.0;
            for (int l = 0; l < n; l++) d += A[(int64_t)k * n + l];
            dtheta[f] = d;
        }
    }
    free(pairs); free(flat); free(Uf); free(M); free(A);
    return 0;
}

/* ======================================================================================
 * Unitary U(n) (Appendix A). Complex matrices are interleaved (re, im)
 * fp64, row-major. G^e(theta, phi) multiplies column i of the real Givens matrix by e^{i phi}
 * (PAPER.md:199-201): G_ii = e^{i phi} cos, G_ij = -sin, G_ji = e^{i phi} sin, G_jj = cos --
 * Algorithm 4's row update; the entry table at PAPER.md:973 also puts the
 * phase on G_jj, which contradicts Alg. 4, dG/dtheta and the two-entry dG/dphi
 * (PAPER.md:1030); we follow Alg. 4 (reading R15).
 * Loss convention for a real loss L of complex U/Y (reading R16):
 *   Gamma = dL/dRe(Y) + i dL/dIm(Y),  dL/dalpha = Re sum conj(Gamma) * dY/dalpha.
 * ====================================================================================== */

/* Algorithm 4 for the round-robin E on a copy of the complex n x m X:
 * for e in reversed(E): r_i <- e^{i phi} cos U_i - sin U_j ; r_j <- e^{i phi} sin U_i + cos U_j.
 * adjoint = 1 applies U^dagger = G^{e_N dagger} ... G^{e_1 dagger}: e in E order with
 * G^dagger = [[e^{-i phi} c, e^{-i phi} s], [-s, c]]. */
int oracle_u_apply(int n, int64_t m, const int32_t *perm, int refl, const float *theta, const float *phi,
                   const uint8_t *mask, const double *X, double *Y, int adjoint) {
    if (n < 2 || m < 0 || refl < -1 || refl >= n) return -1;
    int64_t N;
    int32_t *E = build_E(n, perm, &N);
    if (!E) return -1;
    memcpy(Y, X, sizeof(double) * 2 * (size_t)n * m);
#pragma omp parallel for schedule(static)
    for (int64_t col = 0; col < m; col++) {
        double *yc = Y + ((int64_t)(refl >= 0 ? refl : 0) * m + col) * 2;
        if (refl >= 0 && !adjoint) { yc[0] = -yc[0]; yc[1] = -yc[1]; }
        for (int64_t q = 0; q < N; q++) {
            int64_t e = adjoint ? q : (N - 1 - q);
            if (mask && !mask[e]) continue;
            int i = E[2 * e], j = E[2 * e + 1];
            double c = cos((double)theta[e]), s = sin((double)theta[e]);
            double pc = cos((double)phi[e]), ps = sin((double)phi[e]);
            double *yi = Y + ((int64_t)i * m + col) * 2, *yj = Y + ((int64_t)j * m + col) * 2;
            double ar = yi[0], ai = yi[1], br = yj[0], bi = yj[1];
            if (!adjoint) {
                double er = pc * ar - ps * ai, ei = pc * ai + ps * ar; /* e^{i phi} a */
                yi[0] = c * er - s * br;
                yi[1] = c * ei - s * bi;
                yj[0] = s * er + c * br;
                yj[1] = s * ei + c * bi;
            } else {
                double tr = c * ar + s * br, ti = c * ai + s * bi; /* row i of G^T applied */
                yi[0] = pc * tr + ps * ti;                         /* e^{-i phi} (t) */
                yi[1] = pc * ti - ps * tr;
                yj[0] = -s * ar + c * br;
                yj[1] = -s * ai + c * bi;
            }
        }
        if (refl >= 0 && adjoint) { yc[0] = -yc[0]; yc[1] = -yc[1]; }
    }
    free(E);
    return 0;
}

/* Backward of Y = U(theta, phi) X for a real loss with upstream Gamma (complex n x m):
 * dtheta[e], dphi[e] = Re sum_cols conj(Gamma-propagated) * dY/d(.), and dX = U^dagger Gamma.
 * Per column: run Algorithm 4 storing each rotation's complex inputs (a_i, a_j) (the tape);
 * reverse sweep with the chain rule on y_i = e^{i phi}(c a_i) - s a_j, y_j = e^{i phi}(s a_i) + c a_j:
 *   dy_i/dtheta = -e^{i phi} s a_i - c a_j,  dy_j/dtheta = e^{i phi} c a_i - s a_j,
 *   dy_i/dphi = i e^{i phi} c a_i,           dy_j/dphi = i e^{i phi} s a_i,
 *   g_a_i = conj(e^{i phi}) (c g_i + s g_j),  g_a_j = -s g_i + c g_j   (adjoint of the 2x2 map). */
int oracle_u_backward(int n, int64_t m, const int32_t *perm, int refl, const float *theta, const float *phi,
                      const uint8_t *mask, const double *X, const double *G, double *dX, double *dtheta,
                      double *dphi) {
    if (n < 2 || m < 0 || refl < -1 || refl >= n) return -1;
    int64_t N;
    int32_t *E = build_E(n, perm, &N);
    if (!E) return -1;
    int nt = oracle_num_threads();
    double *pt = (double *)calloc((size_t)nt * N, sizeof(double));
    double *pp = (double *)calloc((size_t)nt * N, sizeof(double));
#pragma omp parallel num_threads(nt)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        int64_t c0 = m * t / nt, c1 = m * (t + 1) / nt;
        double *at = pt + (int64_t)t * N, *ap = pp + (int64_t)t * N;
        double *x = (double *)malloc(sizeof(double) * 2 * n);
        double *g = (double *)malloc(sizeof(double) * 2 * n);
        double *tape = (double *)malloc(sizeof(double) * 4 * (size_t)N);
        for (int64_t col = c0; col < c1; col++) {
            for (int r = 0; r < n; r++) {
                x[2 * r] = X[((int64_t)r * m + col) * 2];
                x[2 * r + 1] = X[((int64_t)r * m + col) * 2 + 1];
            }
            if (refl >= 0) { x[2 * refl] = -x[2 * refl]; x[2 * refl + 1] = -x[2 * refl + 1]; }
            for (int64_t e = N - 1; e >= 0; e--) {
                if (mask && !mask[e]) continue;
                int i = E[2 * e], j = E[2 * e + 1];
                double c = cos((double)theta[e]), s = sin((double)theta[e]);
                double pc = cos((double)phi[e]), ps = sin((double)phi[e]);
                double ar = x[2 * i], ai = x[2 * i + 1], br = x[2 * j], bi = x[2 * j + 1];
                tape[4 * e] = ar; tape[4 * e + 1] = ai; tape[4 * e + 2] = br; tape[4 * e + 3] = bi;
                double er = pc * ar - ps * ai, ei = pc * ai + ps * ar;
                x[2 * i] = c * er - s * br;
                x[2 * i + 1] = c * ei - s * bi;
                x[2 * j] = s * er + c * br;
                x[2 * j + 1] = s * ei + c * bi;
            }
            for (int r = 0; r < n; r++) {
                g[2 * r] = G[((int64_t)r * m + col) * 2];
                g[2 * r + 1] = G[((int64_t)r * m + col) * 2 + 1];
            }
            for (int64_t e = 0; e < N; e++) {
                if (mask && !mask[e]) continue;
                int i = E[2 * e], j = E[2 * e + 1];
                double c = cos((double)theta[e]), s = sin((double)theta[e]);
                double pc = cos((double)phi[e]), ps = sin((double)phi[e]);
                double ar = tape[4 * e], ai = tape[4 * e + 1], br = tape[4 * e + 2], bi = tape[4 * e + 3];
                double er = pc * ar - ps * ai, ei = pc * ai + ps * ar; /* e^{i phi} a_i */
                double gir = g[2 * i], gii = g[2 * i + 1], gjr = g[2 * j], gji = g[2 * j + 1];
                /* dy/dtheta */
                double yti_r = -s * er - c * br, yti_i = -s * ei - c * bi;
                double ytj_r = c * er - s * br, ytj_i = c * ei - s * bi;
                at[e] += gir * yti_r + gii * yti_i + gjr * ytj_r + gji * ytj_i; /* Re conj(g) dy */
                /* dy/dphi = i e^{i phi} (c a_i, s a_i) */
                double ypi_r = -c * ei, ypi_i = c * er;
                double ypj_r = -s * ei, ypj_i = s * er;
                ap[e] += gir * ypi_r + gii * ypi_i + gjr * ypj_r + gji * ypj_i;
                /* adjoint of the 2x2 map */
                double hr = c * gir + s * gjr, hi = c * gii + s * gji;
                g[2 * i] = pc * hr + ps * hi;
                g[2 * i + 1] = pc * hi - ps * hr;
                g[2 * j] = -s * gir + c * gjr;
                g[2 * j + 1] = -s * gii + c * gji;
            }
            if (refl >= 0) { g[2 * refl] = -g[2 * refl]; g[2 * refl + 1] = -g[2 * refl + 1]; }
            if (dX)
                for (int r = 0; r < n; r++) {
                    dX[((int64_t)r * m + col) * 2] = g[2 * r];
                    dX[((int64_t)r * m + col) * 2 + 1] = g[2 * r + 1];
                }
        }
        free(x); free(g); free(tape);
    }
    for (int64_t e = 0; e < N; e++) {
        double st = 0.0, sp = 0.0;
        for (int t = 0; t < nt; t++) { st += pt[(int64_t)t * N + e]; sp += pp[(int64_t)t * N + e]; }
        dtheta[e] = (mask && !mask[e]) ? 0.0 : st;
        dphi[e] = (mask && !mask[e]) ? 0.0 : sp;
    }
    free(pt); free(pp); free(E);
    return 0;
}
