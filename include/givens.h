/*
 * givens.h -- C ABI of the B200 (sm_100a) Givens library: the data-parallel hot path of
 * arXiv 2106.00003 (Hamze, "Parallelized Computation and Backpropagation Under
 * Angle-Parametrized Orthogonal Matrices").
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * n        matrix dimension, n >= 2. n_eff = n rounded up to even; odd n uses the bye
 *          (phantom) index n ("bypass ... if j = n").
 * N        number of angles = n(n-1)/2.
 * E, theta the round-robin sequence built by the circle method (Fig. 1
 *          PAPER.md:378-455): R = n_eff-1 blocks b_1..b_R of S = n_eff/2 disjoint pairs;
 *          block b_{r+1} (r = 0..R-1) pairs positions k and n_eff-1-k (slot k = 0..S-1) of the
 *          sequence s_r with s_r[0] = 0, s_r[p] = 1 + ((p-1-r) mod (n_eff-1)); each pair is
 *          (i,j) = (min, max). theta / dtheta have length N in BLOCK-MAJOR FLAT ORDER: block
 *          b_1 first, slots in increasing k, bye pairs skipped (reading R3).
 *          U = prod_{e in E} G^e(theta_e) with G^{e_N} applied first, G^e as
 *          in PAPER.md:171-181 (G_ii = G_jj = cos, G_ij = -sin, G_ji = +sin, i < j).
 * mask     optional uint8[N] (device pointer or NULL): 1 = free angle, 0 = pinned to zero.
 *          Pinned angles are bypassed (PAPER.md:869-872 generalised to any angle subset): their
 *          theta value is never read (NaN is fine) and their dtheta is written as exactly 0.
 * layout   every matrix is fp32 row-major with a leading dimension (elements) >= its row
 *          length; X, Y, dY, dX are n x m, U is n x n. All data pointers are DEVICE pointers
 *          (cudaMalloc / torch CUDA tensors), caller-owned; nothing is retained after return.
 * ws       device workspace of at least givens_workspace_bytes(op, n, m) bytes, 256-byte
 *          aligned, caller-owned; it may be reused across calls on the same stream. ws = NULL
 *          is allowed: the call then allocates its workspace stream-ordered on `stream`
 *          (cudaMallocAsync from the device's default pool) and frees it (cudaFreeAsync) before
 *          returning; GIVENS_ENOMEM if that allocation fails. Every call is self-contained by
 *          default: it computes its coefficient tables from theta/mask itself. Only
 *          givens_backward with GIVENS_FLAG_REUSE_TABLES consumes the tables a preceding
 *          givens_apply / givens_build_U (same stream) left in ws; the library remembers, per
 *          workspace address, the (device, n, theta, mask, perm, reflect_col) pointers the tables
 *          were built from and refuses a mismatch with GIVENS_EINVAL (it cannot see a theta
 *          rewritten in place at the same address: do not pass the flag then).
 * stream   cudaStream_t (as void*), NULL = legacy default stream. Every call is
 *          stream-ordered and asynchronous: it enqueues kernels and returns; results are
 *          visible after the stream is synchronised. No call allocates device memory unless
 *          ws == NULL.
 * empty    m = 0 is valid: X, Y, dY, dX may then be NULL; dtheta (dphi) is written as zeros.
 * errors   0 on success; negative givens_status_t otherwise, with a thread-local message
 *          from givens_last_error(). Parameter errors are detected before anything is
 *          enqueued. Asynchronous CUDA faults surface at the next synchronising call.
 * threads  all functions are thread-safe (global state: the thread-local error string, a
 *          per-device attribute cache and the mutex-guarded workspace table tags).
 */
#ifndef GIVENS_H_
#define GIVENS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GIVENS_OK = 0,
    GIVENS_EINVAL = -1,       /* bad argument (size, pointer, leading dimension, workspace) */
    GIVENS_ECUDA = -2,        /* a CUDA launch / attribute call failed */
    GIVENS_EUNSUPPORTED = -3, /* valid arguments but no kernel configuration for this n yet */
    GIVENS_ENOMEM = -4        /* ws == NULL and the stream-ordered workspace allocation failed */
} givens_status_t;

enum { GIVENS_OP_APPLY = 0, GIVENS_OP_BUILD_U = 1, GIVENS_OP_BACKWARD = 2,
       GIVENS_OP_U_APPLY = 3, GIVENS_OP_U_BUILD_U = 4, GIVENS_OP_U_BACKWARD = 5 };
/* backward flags: GIVENS_FLAG_RECOMPUTE (the default behaviour, accepted for clarity) rebuilds the
 * coefficient tables from theta/mask; GIVENS_FLAG_REUSE_TABLES reads those a forward call left in
 * ws (checked against the workspace's tag, see `ws` above). */
enum { GIVENS_FLAG_RECOMPUTE = 1, GIVENS_FLAG_REUSE_TABLES = 2 };

/* Thread-local description of the last failure ("" if none). */
const char *givens_last_error(void);

/* Library version string. */
const char *givens_version(void);

/* n(n-1)/2, or -1 if n < 2. */
int64_t givens_num_angles(int32_t n);

/* 1 if the GPU path supports dimension n (a kernel configuration exists), else 0. */
int givens_supported(int32_t n);

/*
 * Host-side, pure: the circle-method schedule by its closed form (Fig. 1).
 * pairs_host: int32[R][S][2] (i < j; bye pairs of odd n have j == n), flat_host: int64[R][S]
 * (flat angle index, -1 for the bye). Either may be NULL. Returns 0 or GIVENS_EINVAL.
 */
int givens_schedule(int32_t n, int32_t *pairs_host, int64_t *flat_host);

/*
 * Host-side, pure: mask[N] from an excluded-dimension set excluded_dims_host[n] (1 =
 * excluded): pair (i,j) is pinned iff both i and j are excluded. The paper's §5 restriction
 * is excluded = {m_keep, ..., n-1}.
 */
int givens_mask_from_dims(int32_t n, const uint8_t *excluded_dims_host, uint8_t *mask_host);

/* Forget what this library remembers about the coefficient tables in ws (the reuse tag, see `ws`
 * above): call it when a workspace is (re)allocated, so that a caching allocator handing out an
 * old workspace address can never make GIVENS_FLAG_REUSE_TABLES accept stale tables. Host-only. */
void givens_workspace_reset(const void *ws);

/* Workspace bytes for op (GIVENS_OP_*) at (n, m) (m = complex columns for the GIVENS_OP_U_*
 * ops). Returns 0 for invalid arguments. */
size_t givens_workspace_bytes(int op, int32_t n, int64_t m);

/*
 * Y = U(theta) X (transpose = 0) or Y = U(theta)^T X (transpose = 1): Algorithm 2
 * applied to the columns of X instead of I. Y may alias X (same pointer
 * and leading dimension). Fills the coefficient tables in ws (reused by givens_backward).
 */
int givens_apply(int32_t n, int64_t m, const float *theta, const uint8_t *mask,
                 const float *X, int64_t ldx, float *Y, int64_t ldy, int transpose,
                 void *ws, size_t ws_bytes, void *stream);

/* U = U(theta), n x n (Algorithm 2 from U <- I_n). Fills ws tables. */
int givens_build_U(int32_t n, const float *theta, const uint8_t *mask, float *U, int64_t ldu,
                   void *ws, size_t ws_bytes, void *stream);

/*
 * Backward of Y = U(theta) X given Y and dY = dL/dY (n x m):
 *   dtheta[N] = dL/dtheta (overwritten, never accumulated; masked entries exactly 0),
 *   dX = U^T dY (optional, NULL to skip; may alias dY).
 * Activations are replayed from Y by inverse rotation (U^fwd recursion),
 * each dtheta_e is reduced over the m columns with a fixed-order, atomic-free two-stage sum
 * (PAPER.md:768-781), so the result is bitwise deterministic for a given (n, m, device).
 * With X = I, Y = U, dY = Gamma this is the paper's Algorithm 3.
 * flags: 0 (or GIVENS_FLAG_RECOMPUTE) builds the coefficient tables from theta/mask;
 * GIVENS_FLAG_REUSE_TABLES reuses a forward's tables in ws (EINVAL if ws holds none for these inputs).
 */
int givens_backward(int32_t n, int64_t m, const float *theta, const uint8_t *mask,
                    const float *Y, int64_t ldy, const float *dY, int64_t lddy,
                    float *dX, int64_t lddx, float *dtheta, int flags,
                    void *ws, size_t ws_bytes, void *stream);

/*
 * Debug / test: run the kernels' data movement for dimension n with row ids as data and no
 * rotation, and record, for every block b_{r+1} and slot k, the row ids the kernel pairs:
 * out_dev int32[R][S][2] (device), reported as (min, max). direction 0 walks the blocks in
 * forward order (b_R first, as givens_apply), 1 in backward order (b_1 first, as
 * givens_backward). Bit-exact against the schedule (pins the on-device indexing).
 */
int givens_index_trace(int32_t n, int direction, int32_t *out_dev, void *stream);

/* ------------------------------------------------------------------------------------------
 * Unitary U(n) variant (Appendix A). theta, phi: fp32[N] in the same flat
 * order; G^e(theta, phi) = R(theta) diag(e^{i phi}, 1) on (i, j), i.e. Algorithm 4's row update
 * (r_i = e^{i phi} cos U_i - sin U_j, r_j = e^{i phi} sin U_i + cos U_j;
 * DESIGN.md reading R15). Complex matrices are interleaved (re, im) fp32 pairs (complex64),
 * row-major, leading dimensions in complex elements. Same workspace / stream / error rules as
 * above, with the GIVENS_OP_U_* workspace ops. givens_u_supported(n) is 1 for 2 <= n <= 32768:
 * n whose real ring configuration fits the unitary tables run on a register ring (one complex
 * column per packed register pair), the rest (W = 32 rings, S = 2048, and the n without a ring)
 * on the generic any-n kernel.
 * ------------------------------------------------------------------------------------------ */
int givens_u_supported(int32_t n);

/* Y = U(theta, phi) X (adjoint = 0) or U^dagger X (adjoint = 1); X, Y complex n x m. */
int givens_u_apply(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask,
                   const float *X, int64_t ldx, float *Y, int64_t ldy, int adjoint,
                   void *ws, size_t ws_bytes, void *stream);

/* U = U(theta, phi), complex n x n (Algorithm 4 from U <- I_n). */
int givens_u_build_U(int32_t n, const float *theta, const float *phi, const uint8_t *mask, float *U,
                     int64_t ldu, void *ws, size_t ws_bytes, void *stream);

/*
 * Backward for a real loss of Y = U X: dY = dL/dRe(Y) + i dL/dIm(Y) (complex n x m).
 * dtheta[N], dphi[N] = dL/dtheta, dL/dphi (overwritten; masked entries 0), dX = U^dagger dY
 * (optional). Replay by the adjoint rotations; per block the theta term uses Q_e and the phi term
 * P_e, both reduced over the m columns deterministically.
 */
int givens_u_backward(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask,
                      const float *Y, int64_t ldy, const float *dY, int64_t lddy, float *dX, int64_t lddx,
                      float *dtheta, float *dphi, int flags, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * Layout options.
 * perm         the circle method's initial sequence ("Beginning with an
 *              arbitrary permutation of the coordinate sequence"): a
 *              permutation of 0..n_eff-1 (odd n: it contains the bye index n), NULL = identity
 *              (Fig. 1). Block b_{r+1} then pairs perm[s_r[k]] with perm[s_r[n_eff-1-k]]; theta
 *              stays in block-major flat order over the resulting pairs (byes skipped). In the
 *              _ex compute calls perm is a DEVICE pointer (int32[n_eff]) and must be valid --
 *              check it on the host with givens_check_perm (the kernels do not). In
 *              givens_schedule_ex / givens_mask_from_dims_ex it is a HOST pointer and is checked.
 * reflect_col  -1, or a column c in [0, n): the reflection class (det -1) "by ... negating an
 *              arbitrary fixed column following the construction":
 *              U' = U diag(.., -1 at c, ..). apply: Y = U' X; transpose: U'^T X; backward:
 *              dtheta of L(U' X), dX = U'^T dY. Costs nothing in the kernels (it is one more
 *              sign in the per-row sign bookkeeping).
 * A givens_backward_ex with GIVENS_FLAG_REUSE_TABLES must use the workspace of a forward call
 * with the same (n, theta, mask, perm, reflect_col) (checked). The calls without _ex are the _ex calls
 * with perm = NULL, reflect_col = -1.
 * ------------------------------------------------------------------------------------------ */

/* 0 if perm_host (int32[n_eff], host) is a permutation of 0..n_eff-1 (NULL counts as valid),
 * else GIVENS_EINVAL with the offending entry in givens_last_error(). */
int givens_check_perm(int32_t n, const int32_t *perm_host);

/* givens_schedule / givens_mask_from_dims for the start sequence perm_host (host, checked). */
int givens_schedule_ex(int32_t n, const int32_t *perm_host, int32_t *pairs_host, int64_t *flat_host);
int givens_mask_from_dims_ex(int32_t n, const int32_t *perm_host, const uint8_t *excluded_dims_host,
                             uint8_t *mask_host);

int givens_apply_ex(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx,
                    float *Y, int64_t ldy, int transpose, const int32_t *perm, int32_t reflect_col, void *ws,
                    size_t ws_bytes, void *stream);
int givens_build_U_ex(int32_t n, const float *theta, const uint8_t *mask, float *U, int64_t ldu,
                      const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes, void *stream);
int givens_backward_ex(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *Y, int64_t ldy,
                       const float *dY, int64_t lddy, float *dX, int64_t lddx, float *dtheta, int flags,
                       const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes, void *stream);
int givens_u_apply_ex(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask,
                      const float *X, int64_t ldx, float *Y, int64_t ldy, int adjoint, const int32_t *perm,
                      int32_t reflect_col, void *ws, size_t ws_bytes, void *stream);
int givens_u_build_U_ex(int32_t n, const float *theta, const float *phi, const uint8_t *mask, float *U,
                        int64_t ldu, const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes,
                        void *stream);
int givens_u_backward_ex(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask,
                         const float *Y, int64_t ldy, const float *dY, int64_t lddy, float *dX, int64_t lddx,
                         float *dtheta, float *dphi, int flags, const int32_t *perm, int32_t reflect_col,
                         void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * Fast (square-root-free) Givens: the same Y = U(theta) X (and U) as
 * givens_apply / givens_build_U, computed with two FMAs per rotation-column on scaled values
 * x = d z, the per-row scales d and the choice between the two factorings (|cos| >= |sin|) made by
 * the precompute. Only for one-lane columns (n_eff in {8, 16, 32, 64}: the factoring choice is then
 * uniform across a warp), identity layout; GIVENS_EUNSUPPORTED for other n. Workspace: the
 * GIVENS_OP_APPLY (resp. GIVENS_OP_BUILD_U) size; the tables it leaves are not reusable by a backward.
 * A measured variant, not the default path.
 * ------------------------------------------------------------------------------------------ */
int givens_fast_apply(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx,
                      float *Y, int64_t ldy, void *ws, size_t ws_bytes, void *stream);
int givens_fast_build_U(int32_t n, const float *theta, const uint8_t *mask, float *U, int64_t ldu, void *ws,
                        size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * GEMM path: the paper's own framing of the workload --
 * build U(theta) once (Alg. 2 from I on the register ring), then Y = U X (or U^T X) as a dense
 * GEMM on the tensor cores in 3xTF32 (hi/lo split of both operands, three TF32 products,
 * relative error ~2^-21), and for the backward dX = U^T dY, Gamma = dL/dU =
 * dY X^T = (dY Y^T) U and dtheta = Algorithm 3 on Gamma (computed by the
 * replay backward with X = I). Same argument meanings, layout options and results as
 * givens_apply_ex / givens_backward_ex (within the fp32 tolerances), but: the workspace is
 * givens_gemm_workspace_bytes(n, m) (U, M, Gamma, K-chunk partials and two staging buffers), the
 * GEMMs run on the library's own tcgen05 kernel (TMA operand tiles, the hi/lo split inside the
 * kernel's pipeline, TMEM accumulators; GIVENS_EUNSUPPORTED if the driver has no tensor-map
 * encoder), operands whose base or leading dimension the TMA cannot describe (16-byte alignment,
 * ld a multiple of 4) are staged through the workspace, and nothing may alias.
 * givens_gemm_backward with GIVENS_FLAG_REUSE_TABLES reuses the U a givens_gemm_apply with the same
 * inputs left in ws (checked as above); ws = NULL allocates stream-ordered as above.
 * ------------------------------------------------------------------------------------------ */
size_t givens_gemm_workspace_bytes(int32_t n, int64_t m);
int givens_gemm_apply(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx,
                      float *Y, int64_t ldy, int transpose, const int32_t *perm, int32_t reflect_col, void *ws,
                      size_t ws_bytes, void *stream);
int givens_gemm_backward(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *Y, int64_t ldy,
                         const float *dY, int64_t lddy, float *dX, int64_t lddx, float *dtheta, int flags,
                         const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GIVENS_H_ */
