// ring.cuh -- register-resident circle-method ring for sm_100a.
//
// Layout: a column of X (n_eff rows) lives in the registers of a
// group of L lanes. Lane t of the group owns the W consecutive slots k = tW .. tW+W-1 of the
// S = n_eff/2 slots of the circle method; for slot k it holds T[q] = the value at position k
// of the current dimension sequence s_r and B[q] = the value at position n_eff-1-k (q = k-tW).
// Slot k of block b_{r+1} rotates exactly that pair ("pairing coordinates at
// the same distance from the endpoints"), so every rotation is thread-local.
//
// Moving from block to block is Fig. 1's shift ("shifting modulo n-1 the
// last n-1 elements ... holding the first element fixed"). Positions 1..n_eff-1 form a ring:
// in slot space top(k) -> top(k+1), bottom(k) -> bottom(k-1), top(S-1) -> bottom(S-1),
// bottom(0) -> top(1), top(0) fixed (s_r -> s_{r+1}; the forward walks it backwards). Only two
// values per lane cross a lane boundary per block, via warp shuffles; everything else is
// register renaming once the step loop is unrolled W times.
#pragma once
#include <cuda_runtime.h>

namespace gk {

// ---- packed fp32x2 helpers (FFMA2 on sm_100a: two columns per instruction) ----------------
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

__device__ __forceinline__ float fma_v(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ float2 fma_v(float a, float2 b, float2 c) { return __ffma2_rn(f2(a), b, c); }
__device__ __forceinline__ float2 fma_v(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

__device__ __forceinline__ float mul_v(float a, float b) { return a * b; }
template <typename V> __device__ __forceinline__ V f2v(float a);
template <> __device__ __forceinline__ float f2v<float>(float a) { return a; }
template <> __device__ __forceinline__ float2 f2v<float2>(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 mul_v(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float neg_v(float a) { return -a; }
__device__ __forceinline__ float2 neg_v(float2 a) { return make_float2(-a.x, -a.y); }

// acc += db*zt - dt*zb summed over the packed columns, in scalar FFMAs (4 pipe cycles per
// packed pair instead of FMUL2 + FFMA2 + FADD = 5)
__device__ __forceinline__ float cross_acc(float acc, float db, float zt, float dt, float zb) {
    return fmaf(-dt, zb, fmaf(db, zt, acc));
}
__device__ __forceinline__ float cross_acc(float acc, float2 db, float2 zt, float2 dt, float2 zb) {
    // packed: FMUL2 + FFMA2 + one FADD (scalar FFMAs with three distinct registers issue at half rate)
    float2 s2 = __ffma2_rn(neg_v(dt), zb, __fmul2_rn(db, zt));
    return acc + (s2.x + s2.y);
}
// the first term of a sum: no "0 + x" (an FADD the compiler must keep, 0 + -0 = +0)
__device__ __forceinline__ float cross_first(float db, float zt, float dt, float zb) {
    return fmaf(-dt, zb, db * zt);
}
__device__ __forceinline__ float cross_first(float2 db, float2 zt, float2 dt, float2 zb) {
    float2 s2 = __ffma2_rn(neg_v(dt), zb, __fmul2_rn(db, zt));
    return s2.x + s2.y;
}

// dphi accumulation of the unitary backward: acc + Re(i conj(v) w) = acc + v.im w.re - v.re w.im
__device__ __forceinline__ float phi_acc(float acc, float2 v, float2 w) {
    return fmaf(-v.x, w.y, fmaf(v.y, w.x, acc));
}
__device__ __forceinline__ float phi_acc(float acc, float, float) { return acc; }

__device__ __forceinline__ float shfl_up_v(float v, int w) { return __shfl_up_sync(0xffffffffu, v, 1, w); }
__device__ __forceinline__ float2 shfl_up_v(float2 v, int w) {
    return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1, w), __shfl_up_sync(0xffffffffu, v.y, 1, w));
}
__device__ __forceinline__ float shfl_dn_v(float v, int w) { return __shfl_down_sync(0xffffffffu, v, 1, w); }
__device__ __forceinline__ float2 shfl_dn_v(float2 v, int w) {
    return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1, w), __shfl_down_sync(0xffffffffu, v.y, 1, w));
}
__device__ __forceinline__ float sel_v(bool p, float a, float b) { return p ? a : b; }
__device__ __forceinline__ float2 sel_v(bool p, float2 a, float2 b) {
    return make_float2(p ? a.x : b.x, p ? a.y : b.y);
}

// ---- one rotation of the pair (top x, bottom y) by angle psi in three shears -------------
// R(psi) = [[1,-tan(psi/2)],[0,1]] [[1,0],[sin psi,1]] [[1,-tan(psi/2)],[0,1]]; the table holds
// tq = tan(psi/2), sq = sin psi with |psi| <= pi/2 after the pi-reduction.
// Forward applies R(psi): x -= tq y; y += sq x; x -= tq y.       (3 FFMA per column)
// Inverse (= transpose) R(-psi): x += tq y; y -= sq x; x += tq y.
template <typename V>
__device__ __forceinline__ void rot_fwd(V &x, V &y, float tq, float sq) {
    x = fma_v(-tq, y, x);
    y = fma_v(sq, x, y);
    x = fma_v(-tq, y, x);
}
template <typename V>
__device__ __forceinline__ void rot_inv(V &x, V &y, float tq, float sq) {
    x = fma_v(tq, y, x);
    y = fma_v(-sq, x, y);
    x = fma_v(tq, y, x);
}
// The backward rotates Z and D by the same coefficients: issue their shears pairwise so the
// second FFMA2 of each pair re-reads the coefficient from the operand reuse cache (an FFMA2 with
// two register pairs and a fresh scalar reads three registers from one bank).
template <typename V>
__device__ __forceinline__ void rot_inv2(V &x, V &y, V &u, V &v, float tq, float sq) {
    x = fma_v(tq, y, x);
    u = fma_v(tq, v, u);
    y = fma_v(-sq, x, y);
    v = fma_v(-sq, u, v);
    x = fma_v(tq, y, x);
    u = fma_v(tq, v, u);
}

// Two slots' replays interleaved: four independent chains per shear stage.
template <typename V>
__device__ __forceinline__ void rot_inv2x2(V &x0, V &y0, V &u0, V &v0, V &x1, V &y1, V &u1, V &v1, float t0,
                                           float s0, float t1, float s1) {
    x0 = fma_v(t0, y0, x0);
    u0 = fma_v(t0, v0, u0);
    x1 = fma_v(t1, y1, x1);
    u1 = fma_v(t1, v1, u1);
    y0 = fma_v(-s0, x0, y0);
    v0 = fma_v(-s0, u0, v0);
    y1 = fma_v(-s1, x1, y1);
    v1 = fma_v(-s1, u1, v1);
    x0 = fma_v(t0, y0, x0);
    u0 = fma_v(t0, v0, u0);
    x1 = fma_v(t1, y1, x1);
    u1 = fma_v(t1, v1, u1);
}

// ---- the ring shift ------------------------------------------------------------------------
// s_r -> s_{r+1} (backward / transpose direction): positions p -> p+1 on the ring 1..n_eff-1.
template <int W, typename V>
__device__ __forceinline__ void shift_up(V (&T)[W], V (&B)[W], bool first, bool last, int L) {
    if constexpr (W == 1) {
        return;  // n = 2: the ring has a single position
    } else {
        V from_prev = shfl_up_v(T[W - 1], L);  // lane t-1's top(tW-1) -> my top(tW)
        V from_next = shfl_dn_v(B[0], L);      // lane t+1's bottom(tW+W) -> my bottom(tW+W-1)
        V b_last = sel_v(last, T[W - 1], from_next);  // top(S-1) -> bottom(S-1)
        V b0 = B[0];
        V t0 = T[0];
#pragma unroll
        for (int q = W - 1; q >= 1; q--) T[q] = T[q - 1];
        T[0] = sel_v(first, t0, from_prev);      // top(0) fixed
        T[1] = sel_v(first, b0, T[1]);           // bottom(0) -> top(1)
#pragma unroll
        for (int q = 0; q < W - 1; q++) B[q] = B[q + 1];
        B[W - 1] = b_last;
    }
}

// s_r -> s_{r-1} (forward direction): positions p -> p-1 on the ring.
template <int W, typename V>
__device__ __forceinline__ void shift_down(V (&T)[W], V (&B)[W], bool first, bool last, int L) {
    if constexpr (W == 1) {
        return;
    } else {
        V from_next = shfl_dn_v(T[0], L);      // lane t+1's top(tW+W) -> my top(tW+W-1)
        V from_prev = shfl_up_v(B[W - 1], L);  // lane t-1's bottom(tW-1) -> my bottom(tW)
        V t_last = sel_v(last, B[W - 1], from_next);  // bottom(S-1) -> top(S-1)
        V b_first = sel_v(first, T[1], from_prev);    // top(1) -> bottom(0)
        V t0 = T[0];
#pragma unroll
        for (int q = 0; q < W - 1; q++) T[q] = T[q + 1];
        T[W - 1] = t_last;
        T[0] = sel_v(first, t0, T[0]);           // top(0) fixed
#pragma unroll
        for (int q = W - 1; q >= 1; q--) B[q] = B[q - 1];
        B[0] = b_first;
    }
}


// The same two shifts with the cross-lane values supplied by the caller, for column groups that
// span several warps (the values crossing a warp boundary come through shared memory).
// forward direction: from_next = lane t+1's T[0], from_prev = lane t-1's B[W-1]
template <int W, typename V>
__device__ __forceinline__ void shift_down_with(V (&T)[W], V (&B)[W], bool first, bool last, V from_next,
                                                V from_prev) {
    V t_last = sel_v(last, B[W - 1], from_next);
    V b_first = sel_v(first, T[1], from_prev);
    V t0 = T[0];
#pragma unroll
    for (int q = 0; q < W - 1; q++) T[q] = T[q + 1];
    T[W - 1] = t_last;
    T[0] = sel_v(first, t0, T[0]);
#pragma unroll
    for (int q = W - 1; q >= 1; q--) B[q] = B[q - 1];
    B[0] = b_first;
}
// backward direction: from_prev = lane t-1's T[W-1], from_next = lane t+1's B[0]
template <int W, typename V>
__device__ __forceinline__ void shift_up_with(V (&T)[W], V (&B)[W], bool first, bool last, V from_prev,
                                              V from_next) {
    V b_last = sel_v(last, T[W - 1], from_next);
    V b0 = B[0];
    V t0 = T[0];
#pragma unroll
    for (int q = W - 1; q >= 1; q--) T[q] = T[q - 1];
    T[0] = sel_v(first, t0, from_prev);
    T[1] = sel_v(first, b0, T[1]);
#pragma unroll
    for (int q = 0; q < W - 1; q++) B[q] = B[q + 1];
    B[W - 1] = b_last;
}

// Row held at position p of s_0 (identity) and of s_{R-1} = (0, 2, 3, ..., n_eff-1, 1).
__device__ __forceinline__ int row_s0(int p) { return p; }
__device__ __forceinline__ int row_sRm1(int p, int ne) { return p == 0 ? 0 : (p == ne - 1 ? 1 : p + 1); }

}  // namespace gk
