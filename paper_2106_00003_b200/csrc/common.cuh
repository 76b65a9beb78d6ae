// common.cuh -- device-side pieces shared by the C-ABI translation unit (givens.cu) and the
// per-configuration ring-kernel instantiations (ring_inst.cu): the closed-form schedule, PTX
// helpers (mbarrier, TMA bulk copies), and the register-ring kernel template k_ring<W,L,MODE>.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

#include "ring.cuh"

namespace gk {

// ------------------------------------------------------------------ schedule (closed form)
// Circle method (Fig. 1): s_r[0] = 0, s_r[p] = 1 + ((p-1-r) mod (n_eff-1));
// block b_{r+1} pairs positions k and n_eff-1-k. Odd n: bye index n sits at
// position r (r >= 1) or n_eff-1 (r = 0), i.e. in slot 0 at r = 0 and min(r, n_eff-1-r) else.
__host__ __device__ inline int seq_at(int r, int p, int ne) {
    int R = ne - 1;
    if (p == 0) return 0;
    int v = (p - 1 - r) % R;
    if (v < 0) v += R;
    return 1 + v;
}
__host__ __device__ inline int bye_slot(int r, int ne) {
    if (r == 0) return 0;
    return r < ne - 1 - r ? r : ne - 1 - r;
}
// flat angle index of (block r, slot k) in block-major order skipping byes; -1 for the bye.
__host__ __device__ inline int64_t flat_of(int r, int k, int n, int ne) {
    int S = ne / 2;
    if (n == ne) return (int64_t)r * S + k;
    int kb = bye_slot(r, ne);
    if (k == kb) return -1;
    return (int64_t)r * (S - 1) + k - (k > kb ? 1 : 0);
}
// position of label i in s_r
__host__ __device__ inline int pos_of(int i, int r, int ne) {
    if (i == 0) return 0;
    int R = ne - 1;
    return 1 + ((i - 1 + r) % R);
}
// Start permutation: the ring works on labels 0..n_eff-1 (the
// positions of the identity start sequence); label l is row perm[l]. Odd n: the bye is the label
// bl with perm[bl] = n. flat index of (block r, slot k) with the bye at label bl.
__host__ __device__ inline int64_t flat_of_bl(int r, int k, int n, int ne, int bl) {
    int S = ne / 2;
    if (n == ne) return (int64_t)r * S + k;
    int p = pos_of(bl, r, ne);
    int kb = p < ne - 1 - p ? p : ne - 1 - p;
    if (k == kb) return -1;
    return (int64_t)r * (S - 1) + k - (k > kb ? 1 : 0);
}
// workspace layout block (k_layout): lay[0..ne) = row of each label, lay[ne] = bye label (odd n),
// lay[ne + 1] = label of the reflected column (-1: none)

#ifndef GK_BWD_WARPS
#define GK_BWD_WARPS 8
#endif
constexpr int kNW = GK_BWD_WARPS;
#ifndef RS_LC
#define RS_LC 1  // reduce-scatter of the per-slot sums across column groups sharing a warp
#endif  // warps per CTA of the backward ring kernel
#ifndef GK_FWD_WARPS
#define GK_FWD_WARPS 8
#endif
constexpr int kNWF = GK_FWD_WARPS;  // warps per CTA of the forward / transpose ring kernels
// base modes; M_UNI marks the unitary U(n) variant (Appendix A): complex columns stored as
// interleaved (re, im) pairs, i.e. two real columns per complex column
// M_IDLE (launch-time only) selects the instantiation with idle lanes (La < L, runtime La); without
// it La == L is a compile-time constant (fewer registers and address computations)
// M_NARROW (launch-time only): 4-warp CTAs with at most 2 columns per thread, for batches too
// small to give every SM a slab at the normal width (U-build and Alg. 3 at n <= 2048, C2)
// M_NK4 (launch-time only, with M_NARROW, W = 8 rings): 4 columns per thread instead of 2 -- the same
// slab width as the W = 16 narrow launch with half the slots per lane, a quarter of the unrolled body
// (the W = 16 narrow backward does not fit the instruction cache at one warp per SMSP) and each
// coefficient shared by two packed column pairs (C2: backward 130 -> 101 us)
// M_FG (forward / U-build on one-lane columns only): fast (square-root-free) Givens --
// two FFMAs per rotation-column on scaled values z = x / d, the per-row scales d tracked by the
// precompute (k_fg_tables), the factoring (unit coefficient on one input or the other) chosen per slot
// by |cos| >= |sin|; warp-uniform in this layout because every lane holds a whole column
enum Mode { M_FWD = 0, M_BUILDU = 1, M_TRANS = 2, M_BWD = 3, M_UNI = 4, M_IDLE = 8, M_NARROW = 16, M_NK4 = 32,
            M_FG = 64 };
constexpr int kNWN = 4;  // warps per CTA of the narrow variant
#ifndef GK_HALF_BODY
#define GK_HALF_BODY -1  // -1: per-kernel choice (k_ring); else bit mask (1 unitary bwd, 2 unitary fwd, 4 real bwd, 8 real fwd): W/2-step bodies
#endif
#ifndef GK_QUARTER_BODY
#define GK_QUARTER_BODY 2  // bit mask as GK_HALF_BODY: W/4-step bodies (the unitary apply: 11.88 -> 11.71 ms; the
                           // others measured neutral or slower: C5 shard backward 35.26 -> 36.2 ms, C4 gradient
                           // 20.96 -> 21.26 ms, unitary backward 38.63 -> 38.75 ms)
#endif
#ifndef GK_UNI_ONE_SITE
#define GK_UNI_ONE_SITE 1  // unitary backward: one reduction call site per group (u_backward 63.3 -> 62.5 ms)
#endif
#ifndef GK_DEFER_BWD
#define GK_DEFER_BWD 1  // the backward's warp-boundary exchange "arrive early, wait late" (bit 0: four-warp, bit 1: two-warp columns)
#endif
#ifndef GK_BFIRST
#define GK_BFIRST 1  // two-warp-column backward: ring-boundary slot quads first in every step (see k_ring)
#endif
#ifndef GK_PDL
#define GK_PDL 1  // programmatic dependent launches of k_coef, the ring kernels and the stage-2 reduction
#endif
#ifndef GK_XPRED
#define GK_XPRED 3  // multi-warp columns: branch-free warp-boundary publish / read (bit 0: the named-barrier
                    // exchange of two-warp columns; bit 1: also the deferred exchange of four-warp columns,
                    // C4 U-build 7.06 -> 6.52 ms, gradient 20.81 -> 20.15 ms)
                    // (C5 shard forward 10.93 -> 9.63 ms, backward 35.26 -> 33.56 ms; n = 2048 U-build
                    // 0.855 -> 0.750 ms, gradient 2.746 -> 2.632 ms: the per-step divergent regions around the
                    // lane-0 / lane-31 stores and loads had cost 8.5% branch_resolving stall samples)
#endif
#ifndef GK_NO_PARTIAL
#define GK_NO_PARTIAL 0  // timing ablation only (wrong dtheta): skip the bulk stores / reduce-adds of the partial rows
#endif
#ifndef GK_BWD_IL
#define GK_BWD_IL 1  // interleave the replays of a slot pair in the real backward (C3 bwd 15.78 -> 15.60 ms)
#endif

__host__ __device__ constexpr int ring_warps(int mode) {
    return (mode & M_NARROW) ? kNWN : ((mode & 3) == 3 ? kNW : kNWF);
}

__host__ __device__ constexpr int kcols(int W, int mode) {
    // real columns per thread, so that the column state is ~128 registers (2 W K forward, 4 W K
    // backward); two packed fp32 columns per FFMA2 (one complex column in the unitary variant)
    const int k = ((mode & 3) == M_BWD) ? (32 / W > 8 ? 8 : 32 / W) : (64 / W > 8 ? 8 : 64 / W);
    const int cap = (mode & M_NK4) ? 4 : 2;
    return ((mode & M_NARROW) && k > cap) ? cap : k;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// structured (C++-level) spin so the compiler sees the loop and re-converges the warp after it
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    while (!mbar_try(b, parity)) {
    }
}

// Programmatic dependent launch: a kernel launched with the programmatic-stream-serialization
// attribute may start before its predecessor on the stream has finished; it must not touch memory the
// predecessor writes (or reads) before pdl_wait(), which returns once the predecessor has completed and
// its writes are visible. pdl_trigger() lets the successor launch as soon as every CTA of this grid has
// issued it. Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// predicated shared-memory store (no divergent branch around it)
__device__ __forceinline__ void st_shared_if(bool p, float *a, float v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.f32 [%1], %2;\n}" ::"r"((uint32_t)p),
                 "r"(smem_u32(a)), "f"(v)
                 : "memory");
}
__device__ __forceinline__ void st_shared_if(bool p, float2 *a, float2 v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.v2.f32 [%1], {%2, %3};\n}" ::"r"((uint32_t)p),
                 "r"(smem_u32(a)), "f"(v.x), "f"(v.y)
                 : "memory");
}

// compile-time unrolling: f(std::integral_constant<int, I>{}) for I = 0..N-1, as straight-line code
template <typename F, int... I>
__device__ __forceinline__ void unroll_impl(F &&f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void unroll(F &&f) {
    unroll_impl(f, std::make_integer_sequence<int, N>{});
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------------ the register-ring kernel
struct RingArgs {
    int n, ne;
    int La;           // active lanes per column group (== L except for idle-lane configurations)
    int64_t m;
    const float *X;   // FWD/TRANS: input; BWD: Y
    int64_t ldx;
    const float *dY;  // BWD only
    int64_t lddy;
    float *Y;         // FWD/BUILDU/TRANS: output; BWD: dX (nullable)
    int64_t ldy;
    const uint8_t *coef;     // (t, s) per slot, lane-chunked rows
    const uint8_t *coef_ph;  // unitary: (p_t, q_t, p_b, q_b) phase factors per slot
    const uint8_t *coef_ab;  // unitary backward: (alpha, beta) dphi weights per slot
    const uint8_t *sfin;     // final sign per label
    const int32_t *lrow;     // row of each label under a start permutation (>= n: the odd-n bye);
                             // NULL = identity (no dependent global loads at slab load/store)
    float *partial;   // BWD: per CTA, per reduction group, NW warp blocks (see red_geom)
    int64_t nslabs;
    int vec_ok;       // 1 if all row starts are 16-byte aligned for K-wide vector access
    const uint32_t *fgmask;  // M_FG: per table row, bit q = slot q uses the second factoring
    const float *sfg;        // M_FG: final scale of each label (the store multiplies by it)
};

template <int K>
struct ColIO;
// whole-slab fast path (every column in range, K-aligned rows): unconditional vector accesses, so
// a slab load is one batch of independent LDGs instead of a chain of branch regions that each wait
// for their load
template <int K>
struct FastIO {
    using IO = ColIO<K>;
    using V = typename IO::V;
    static constexpr int KP = IO::KP;
    __device__ static void load(const float *p, V (&v)[KP]) {
        if constexpr (K == 1) {
            v[0] = __ldg(p);
        } else if constexpr (K == 2) {
            v[0] = __ldg(reinterpret_cast<const float2 *>(p));
        } else {
#pragma unroll
            for (int h = 0; h < K / 4; h++) {
                const float4 a = __ldg(reinterpret_cast<const float4 *>(p) + h);
                v[2 * h] = make_float2(a.x, a.y);
                v[2 * h + 1] = make_float2(a.z, a.w);
            }
        }
    }
    __device__ static void store(float *p, const V (&v)[KP]) {
        if constexpr (K == 1) {
            *p = v[0];
        } else if constexpr (K == 2) {
            *reinterpret_cast<float2 *>(p) = v[0];
        } else {
#pragma unroll
            for (int h = 0; h < K / 4; h++)
                reinterpret_cast<float4 *>(p)[h] = make_float4(v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y);
        }
    }
};
template <>
struct ColIO<1> {
    using V = float;
    static constexpr int KP = 1;
    __device__ static void load(const float *row, int64_t c0, int64_t m, int, V (&v)[1]) {
        v[0] = c0 < m ? __ldg(row + c0) : 0.f;
    }
    __device__ static void store(float *row, int64_t c0, int64_t m, int, const V (&v)[1]) {
        if (c0 < m) row[c0] = v[0];
    }
};
template <>
struct ColIO<2> {
    using V = float2;
    static constexpr int KP = 1;
    __device__ static void load(const float *row, int64_t c0, int64_t m, int vec, V (&v)[1]) {
        if (vec && c0 + 2 <= m) {
            v[0] = __ldg(reinterpret_cast<const float2 *>(row + c0));
        } else {
            v[0].x = c0 < m ? __ldg(row + c0) : 0.f;
            v[0].y = c0 + 1 < m ? __ldg(row + c0 + 1) : 0.f;
        }
    }
    __device__ static void store(float *row, int64_t c0, int64_t m, int vec, const V (&v)[1]) {
        if (vec && c0 + 2 <= m) {
            *reinterpret_cast<float2 *>(row + c0) = v[0];
        } else {
            if (c0 < m) row[c0] = v[0].x;
            if (c0 + 1 < m) row[c0 + 1] = v[0].y;
        }
    }
};
template <>
struct ColIO<4> {
    using V = float2;
    static constexpr int KP = 2;
    __device__ static void load(const float *row, int64_t c0, int64_t m, int vec, V (&v)[2]) {
        if (vec && c0 + 4 <= m) {
            float4 a = __ldg(reinterpret_cast<const float4 *>(row + c0));
            v[0] = make_float2(a.x, a.y);
            v[1] = make_float2(a.z, a.w);
        } else {
            v[0].x = c0 < m ? __ldg(row + c0) : 0.f;
            v[0].y = c0 + 1 < m ? __ldg(row + c0 + 1) : 0.f;
            v[1].x = c0 + 2 < m ? __ldg(row + c0 + 2) : 0.f;
            v[1].y = c0 + 3 < m ? __ldg(row + c0 + 3) : 0.f;
        }
    }
    __device__ static void store(float *row, int64_t c0, int64_t m, int vec, const V (&v)[2]) {
        if (vec && c0 + 4 <= m) {
            *reinterpret_cast<float4 *>(row + c0) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
        } else {
            if (c0 < m) row[c0] = v[0].x;
            if (c0 + 1 < m) row[c0 + 1] = v[0].y;
            if (c0 + 2 < m) row[c0 + 2] = v[1].x;
            if (c0 + 3 < m) row[c0 + 3] = v[1].y;
        }
    }
};

template <>
struct ColIO<8> {
    using V = float2;
    static constexpr int KP = 4;
    __device__ static void load(const float *row, int64_t c0, int64_t m, int vec, V (&v)[4]) {
        if (vec && c0 + 8 <= m) {
            float4 a = __ldg(reinterpret_cast<const float4 *>(row + c0));
            float4 b = __ldg(reinterpret_cast<const float4 *>(row + c0 + 4));
            v[0] = make_float2(a.x, a.y); v[1] = make_float2(a.z, a.w);
            v[2] = make_float2(b.x, b.y); v[3] = make_float2(b.z, b.w);
        } else {
#pragma unroll
            for (int p = 0; p < 4; p++) {
                v[p].x = c0 + 2 * p < m ? __ldg(row + c0 + 2 * p) : 0.f;
                v[p].y = c0 + 2 * p + 1 < m ? __ldg(row + c0 + 2 * p + 1) : 0.f;
            }
        }
    }
    __device__ static void store(float *row, int64_t c0, int64_t m, int vec, const V (&v)[4]) {
        if (vec && c0 + 8 <= m) {
            *reinterpret_cast<float4 *>(row + c0) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
            *reinterpret_cast<float4 *>(row + c0 + 4) = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
        } else {
#pragma unroll
            for (int p = 0; p < 4; p++) {
                if (c0 + 2 * p < m) row[c0 + 2 * p] = v[p].x;
                if (c0 + 2 * p + 1 < m) row[c0 + 2 * p + 1] = v[p].y;
            }
        }
    }
};

template <typename V>
__device__ __forceinline__ V vneg_if(V v, bool neg) { return neg ? neg_v(v) : v; }

__device__ __forceinline__ void bulk_s2g_reduce_add(float *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g_store(float *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// dtheta-partial geometry of the backward ring (shared by the kernel, the host's workspace sizing
// and the stage-2 reduction): RG steps per reduction group, NSUM warps per chunk, OUTCH chunks
// reduced per warp; per CTA the partial holds, for every group, NW blocks of RG x OUTCH float4.
struct RedGeom {
    int LW, H, NCHW, NSUM, OUTCH, RG, NW;
};
__host__ __device__ constexpr RedGeom red_geom(int W, int L, int vals = 1, int NW = kNW) {
    int LW = L < 32 ? L : 32, H = L / LW, NCHW = (W / 4) * LW * vals, NSUM = NW / H;
    // 4-step groups wherever the ring fits next to two coefficient stages (two-warp columns
    // included: n = 2048 bwd 37.3 -> 36.8 ms on 32768 columns); 2-step groups for four-warp columns
    // (4-step ones would leave one-step coefficient stages: 169.6 -> 220.9 ms), the unitary variant
    // and wide rows
    int RG = (NCHW >= 256 || (H > 2 && NCHW >= 128) || NW > 8 || vals > 1) ? 2 : 4;
    return RedGeom{LW, H, NCHW, NSUM, (NCHW + NSUM - 1) / NSUM, RG, NW};
}

// Compile-time geometry of one ring configuration: W slots per lane, L lanes per column group
// (L < 32: several groups per warp; L = 32 H: a group spans H warps).
template <int W, int L, int MODE>
struct RingGeom {
    static constexpr int S = W * L;                 // slots = n_eff / 2 (instantiated maximum)
    static constexpr int LW = L < 32 ? L : 32;      // lanes of a group inside one warp
    static constexpr int H = L / LW;                // warps per column group
    static constexpr int LC = 32 / LW;              // column groups per warp
    static constexpr int BM = MODE & 3;             // base mode
    static constexpr bool UNI = (MODE & M_UNI) != 0;
    static constexpr int NW = ring_warps(MODE);      // warps per CTA
    static constexpr int NGRP = NW * LC / H;        // column groups per CTA
    static constexpr int K = kcols(W, MODE);        // real columns per thread
    static constexpr bool GRAD = (BM == M_BWD);
    static constexpr int KP = (K + 1) / 2;          // packed register pairs per slot
    // table bytes per slot staged per block: (t, s) 8 B; unitary adds the phases (16 B) and, in
    // the backward, the dphi weights (alpha, beta) (8 B)
    // (forward / adjoint apply: the phases as two FFMA2-ready pairs per side, 32 B)
    static constexpr int PHB = UNI ? (GRAD ? 16 : 32) : 0;  // phase bytes per slot
    static constexpr int RB = 8 + PHB + ((UNI && GRAD) ? 8 : 0);
    // backward sums (dtheta, and dphi in the unitary variant): per-warp ring of NG groups of RG
    // steps, reduced one group later
    static constexpr int VALS = UNI ? 2 : 1;
    static constexpr int RG = red_geom(W, L, VALS, NW).RG;  // steps per reduction group
    static constexpr int NG = 2;                    // groups in flight
    static constexpr int D = RG * NG;               // ring depth in steps
    static constexpr int NCHW1 = (W / 4) * LW;      // dtheta chunks held by one warp
    static constexpr int NCHW = NCHW1 * VALS;       // all chunks of a warp's ring row
    static constexpr int NSUM = NW / H;             // warps contributing to each chunk
    static constexpr int OUTCH = (NCHW + NSUM - 1) / NSUM;  // chunks reduced per warp (max)
    static constexpr int XV = GRAD ? 2 * KP : KP;   // packed values crossing a warp boundary per direction
    static constexpr size_t XB = H > 1 ? (size_t)2 * NW * 2 * XV * 8 : 0;  // warp-boundary exchange
    static constexpr size_t REDB = GRAD ? (size_t)NW * D * NCHW * 16 + (size_t)NW * NG * RG * OUTCH * 16 : 0;
    // Coefficient stages. Each stage boundary costs a wait and a release, so stages are as large as
    // shared memory allows: the real apply stages up to one unrolled body of W table rows (<= 64 KB
    // each, 192 KB in flight; 4.61 -> 4.41 ms at C3 against 8-row stages); the real backward takes
    // what its dtheta ring leaves (<= 128 KB, two or more stages; C3: two of 32 KB instead of four of 16 KB,
    // 7.95 -> 7.86 ms, n = 2048: 42.6 -> 40.7 ms on 32768 columns); the unitary variant keeps W/2-row
    // stages of <= 40 KB for the apply (the backward's tables are 32 B per slot: 16 KB per step at
    // S = 512, so 16 KB stages meant a boundary every step).
    static constexpr int GRAD_BUDGET_() {
        const long free_ = 225 * 1024 - 256 - (long)XB - (long)REDB;
        return (int)(free_ < 131072 ? free_ : 131072);
    }
    static constexpr int STAGE_BUDGET = GRAD ? GRAD_BUDGET_() : (UNI ? 163840 : 196608);
    static constexpr int sps_pick() {
        int v = (GRAD || UNI) ? W / 2 : W;
        const int lim = GRAD ? STAGE_BUDGET / 2 : (UNI ? 40960 : 65536);
        while (v > 1 && v * S * RB > lim) v /= 2;
        return v;
    }
    static constexpr int SPS = sps_pick();
    static constexpr int STAGEB = SPS * S * RB;
    static constexpr int NSTAGE_ = STAGE_BUDGET / STAGEB;
    static constexpr int NSTAGE = NSTAGE_ > 8 ? 8 : (NSTAGE_ < 2 ? 2 : NSTAGE_);
    static constexpr size_t OFF_STAGE = 256;
    static constexpr size_t OFF_X = OFF_STAGE + (size_t)NSTAGE * STAGEB;
    static constexpr size_t OFF_RED = OFF_X + XB;
    static constexpr size_t OFF_OUT = OFF_RED + (GRAD ? (size_t)NW * D * NCHW * 16 : 0);
    static constexpr size_t SMEM = OFF_OUT + (GRAD ? (size_t)NW * NG * RG * OUTCH * 16 : 0);
};

// complex multiply of a packed (re, im) value by (p + i q), and by its conjugate (p - i q)
__device__ __forceinline__ float2 cmul(float2 z, float p, float q) {
    return __ffma2_rn(make_float2(z.y, z.y), make_float2(-q, p), __fmul2_rn(make_float2(z.x, z.x), make_float2(p, q)));
}
__device__ __forceinline__ float2 cmulc(float2 z, float p, float q) {
    return __ffma2_rn(make_float2(z.y, z.y), make_float2(q, p), __fmul2_rn(make_float2(z.x, z.x), make_float2(p, -q)));
}
__device__ __forceinline__ float cmul(float z, float, float) { return z; }
__device__ __forceinline__ float cmulc(float z, float, float) { return z; }
// the same with the factor pre-arranged as (a, b, c, d): z -> (z.x a + z.y c, z.x b + z.y d), i.e.
// e = (p, q, -q, p) multiplies by p + i q and (p, -q, q, p) by its conjugate -- one FMUL2 + one
// FFMA2 on register pairs as loaded
__device__ __forceinline__ float2 cmul4(float2 z, float4 e) {
    return __ffma2_rn(make_float2(z.y, z.y), make_float2(e.z, e.w), __fmul2_rn(make_float2(z.x, z.x), make_float2(e.x, e.y)));
}
__device__ __forceinline__ float cmul4(float z, float4) { return z; }

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Hot-path kernel. One CTA of kNW warps owns a slab of C = NGRP * K columns; every column
// lives in the registers of L lanes (ring.cuh). All 2S steps (pad + the n_eff-1 blocks) run
// on-chip; the coefficient table streams through shared memory in TMA bulk stages; values that
// cross a warp boundary of a multi-warp column group go through shared memory under a named
// barrier; the backward's per-slot column sums go to a per-warp shared-memory ring in groups of
// RG steps, are reduced across the warps holding the same slots one group later (each warp owns
// a chunk range) and leave the SM as TMA bulk reduce-adds into this CTA's private partial rows
// (fixed order, no atomics => deterministic).
template <int W, int L, int MODE>
__global__ void __launch_bounds__(RingGeom<W, L, MODE>::NW * 32, 1) k_ring(const RingArgs a) {
    using G = RingGeom<W, L, MODE>;
    using IO = ColIO<G::K>;
    using V = typename IO::V;
    constexpr int KP = IO::KP;
    constexpr int K = G::K;
    constexpr int LW = G::LW, H = G::H, LC = G::LC, SPS = G::SPS, NSTAGE = G::NSTAGE;
    // active geometry: L lanes are instantiated, the last warp of a group may leave lanes idle
    // (S = W * La with La in (L - 32, L]); buffers are sized for the instantiated maximum
    constexpr bool IDLE = (MODE & M_IDLE) != 0 && !(H == 1 && LC > 1);
    const int La = IDLE ? a.La : L;
    const int S = W * La, STEPS = 2 * S;
    const int rowb = S * 8;                       // bytes per (t, s) table row
    const uint32_t stage_bytes = (uint32_t)(SPS * S * G::RB);
    constexpr int RG = G::RG, NG = G::NG, D = G::D, NCHW = G::NCHW, NSUM = G::NSUM, OUTCH = G::OUTCH;
    constexpr int XV = G::XV;
    constexpr int NW = G::NW;
    constexpr int BM = G::BM;
    constexpr bool UNI = G::UNI;
    constexpr int NCHW1 = G::NCHW1;
    constexpr bool UP = (BM == M_TRANS || BM == M_BWD);  // walk b_1 -> b_R (inverse rotations)
    constexpr bool GRAD = G::GRAD;
    static_assert(W % SPS == 0 && W % RG == 0 && W % 4 == 0 && W % 2 == 0, "geometry");
    static_assert(H == 1 || LW == 32, "multi-warp groups use whole warps");
    // Multi-warp column groups without a gradient exchange their warp-boundary values "arrive early,
    // wait late": each warp publishes its two boundary values at the end of a step and arrives on its
    // group's mbarrier without waiting; the lanes that need a neighbour's value leave the shifted
    // register pending; the next step rotates its middle slot pairs first and only then waits for the
    // group's phase and patches the two pending registers (slots 0 and W-1, whose pairs go last). The
    // exchange latency overlaps W - 2 slots of arithmetic instead of stalling every warp of the group
    // at a named barrier. Double-buffered by step parity: a warp publishes step s + 1 only after it has
    // read step s, and the writer of step s + 2 has waited for step s + 1, so no buffer is overwritten
    // before it is read. Measured (one B200, same call): four-warp columns (n = 4096 U-build) 7.21 ->
    // 6.99 ms; two-warp columns got slower (C5 shard forward 10.94 -> 11.63 ms), so they keep the
    // named barrier.
    // (the backward too, under GK_DEFER_BWD: bit 0 four-warp columns, bit 1 two-warp columns; its
    // boundary values include D, and its slot order keeps the quads whole for the dtheta ring stores)
    constexpr bool DEFER = !GRAD ? (H >= 4) : (!UNI && (((GK_DEFER_BWD & 1) && H >= 4) || ((GK_DEFER_BWD & 2) && H == 2)));
    constexpr int UBH = W / 2;
    // W/2-step unrolled bodies: half the instruction footprint, for a register move of the ring at every
    // loop edge (the renaming is half way round). Chosen per kernel from one-box A/B runs of the whole
    // library (GK_HALF_BODY=15 against 0): the unitary backward 62.4 -> 38.7 ms and apply 12.9 -> 11.9 ms
    // (no_instruction was 2.8 stalls per issue), the n = 1024 U-build gradient (W = 16 narrow) 488 -> 403 us,
    // C4 gradient 21.6 -> 20.9 ms, C5 shard backward 35.9 -> 35.3 ms; slower for the one-warp-column wide
    // backward (C3 15.62 -> 15.82 ms), the real forwards (C5 shard 10.93 -> 11.3 ms) and the W = 8
    // narrow backward (n = 256 gradient 67.0 -> 69.4 us), which keep W-step bodies
    constexpr bool HALF_PICK = GK_HALF_BODY >= 0
                                   ? ((UNI && GRAD && (GK_HALF_BODY & 1)) || (UNI && !GRAD && (GK_HALF_BODY & 2)) ||
                                      (!UNI && GRAD && (GK_HALF_BODY & 4)) || (!UNI && !GRAD && (GK_HALF_BODY & 8)))
                                   : (UNI || (GRAD && (H >= 2 || ((MODE & M_NARROW) && W == 16))));
    constexpr bool HALF = HALF_PICK && UBH % G::SPS == 0 && (!GRAD || UBH % G::RG == 0) && UBH % 2 == 0;
    // W/4-step bodies (GK_QUARTER_BODY, same bit mask as GK_HALF_BODY; where the stage and ring group
    // sizes divide W/4)
    constexpr int UBQ = W / 4;
    constexpr bool QUARTER = ((UNI && GRAD && (GK_QUARTER_BODY & 1)) || (UNI && !GRAD && (GK_QUARTER_BODY & 2)) ||
                              (!UNI && GRAD && (GK_QUARTER_BODY & 4)) || (!UNI && !GRAD && (GK_QUARTER_BODY & 8))) &&
                             UBQ % G::SPS == 0 && (!GRAD || UBQ % G::RG == 0) && UBQ % 2 == 0;
    constexpr int UB = QUARTER ? UBQ : (HALF ? UBH : W);  // steps per unrolled body
    constexpr bool FG = (MODE & M_FG) != 0;
    // (measured, one box: two-warp-column backward C5 shard 37.2 -> 35.8 ms, n = 2048 U-build gradient
    // 2.78 -> 2.76 ms; slower for one-warp columns (C3 backward 15.58 -> 15.78 ms), the forwards and
    // four-warp columns, which keep the natural order)
    constexpr bool BFIRST = GK_BFIRST != 0 && H == 2 && GRAD;
    static_assert(!FG || (L == 1 && !UNI && !GRAD && !UP), "fast Givens: forward / U-build on one-lane columns");

    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint32_t *released = reinterpret_cast<uint32_t *>(full + NSTAGE);  // per-buffer warp release counts
    uint64_t *rfull = full + NSTAGE + (NSTAGE + 1) / 2;
    uint64_t *rempty = rfull + NG;
    uint64_t *xb = rempty + NG;  // DEFER: one barrier per column group, the warp-boundary exchange
    uint8_t *stagebuf = smem + G::OFF_STAGE;
    V *xbuf = reinterpret_cast<V *>(smem + G::OFF_X);                 // [2][NW][2][XV]
    float4 *red = reinterpret_cast<float4 *>(smem + G::OFF_RED);   // [NW][D][NCHW]
    float4 *outb = reinterpret_cast<float4 *>(smem + G::OFF_OUT);  // [NW][NG][RG][OUTCH]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = warp % H;                       // which warp of its column group
    const int cw = warp / H;                      // warp-group index in the CTA
    const int g = lane / LW;                      // column group inside the warp (LC > 1)
    const int tl = lane % LW;                     // lane inside the group's warp slice
    const int t = h * LW + tl;                    // lane inside the column group
    const bool first = (t == 0), last = (t == La - 1);
    const bool active = t < La;
    const int tc = active ? t : La - 1;          // idle lanes read a valid coefficient slot
    const int ne = a.ne, n = a.n;
    const int64_t C = (int64_t)G::NGRP * K;
    const int my_slabs = (int)((a.nslabs - blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int total_stages = my_slabs * (STEPS / SPS);
    // chunk range (of this warp's half h) of the per-step sums this warp reduces
    const int ch0 = (cw * NCHW) / NSUM, ch1 = ((cw + 1) * NCHW) / NSUM;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; i++) {
            mbar_init(&full[i], 1);
            released[i] = 0;
        }
        for (int i = 0; i < NG; i++) {
            mbar_init(&rfull[i], NW);
            mbar_init(&rempty[i], NW);
        }
        if constexpr (DEFER)
            for (int i = 0; i < NW / H; i++) mbar_init(&xb[i], H);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    __syncthreads();
    // launched with programmatic stream serialization (launch_wlm): the barrier setup above overlaps the
    // predecessor's tail; every global access (tables, signs, X, outputs) comes after this wait
    pdl_trigger();
    pdl_wait();
    if constexpr (GRAD) {
        // pre-arm: every ring group starts out "empty" (phase 0 completes here), so the first
        // use of each group waits on parity 0 without a special case
        if (lane == 0)
            for (int i = 0; i < NG; i++) mbar_arrive(&rempty[i]);
    }

    // table rows of slab-local stage j: forward reads rho = 2S - u (descending), backward rho = u;
    // a stage holds SPS rows of each staged table part: (t, s) [, phases [, (alpha, beta)]]
    auto stage_rho0 = [&](int gst) -> int {
        int j = gst % (STEPS / SPS);
        return UP ? j * SPS : (STEPS - (j + 1) * SPS + 1);
    };
    auto issue_stage = [&](int gst, int b) {
        const int rho0 = stage_rho0(gst);
        uint8_t *dst = stagebuf + (size_t)b * G::STAGEB;
        mbar_expect_tx(&full[b], stage_bytes);
        bulk_g2s(dst, a.coef + (int64_t)rho0 * rowb, (uint32_t)(SPS * rowb), &full[b]);
        if constexpr (UNI) {
            constexpr int PR = G::PHB / 8;  // phase bytes per slot in units of the (t, s) row
            bulk_g2s(dst + SPS * rowb, a.coef_ph + (int64_t)rho0 * PR * rowb, (uint32_t)(SPS * PR * rowb), &full[b]);
            if constexpr (GRAD)
                bulk_g2s(dst + SPS * 3 * rowb, a.coef_ab + (int64_t)rho0 * rowb, (uint32_t)(SPS * rowb), &full[b]);
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE && s < total_stages; s++) issue_stage(s, s);
    }

    // dtheta stage 1: reduce ring group gg (steps gg*RG .. gg*RG+RG-1 of this CTA) over the NSUM
    // warps holding the same slots, for this warp's chunk range, and push it to the partial rows.
    auto reduce_group = [&](int gg) {
        const int bi = gg % NG;
        mbar_wait(&rfull[bi], (uint32_t)((gg / NG) & 1));
        if (lane == 0) bulk_wait_read<NG - 1>();  // the bulk ops that last read outb[bi] are done
        __syncwarp();
        float4 *ob = outb + ((size_t)warp * NG + bi) * RG * OUTCH;
        const float4 *rsrc = red + ((size_t)h * D + bi * RG) * NCHW + ch0;  // warp h of group 0
        constexpr bool EVEN = (NCHW % NSUM) == 0;  // every warp owns exactly OUTCH chunks
        const int nch = EVEN ? OUTCH : ch1 - ch0;
        auto sum_item = [&](int r, int c) {
            const float4 *src = rsrc + (size_t)r * NCHW + c;
            float2 lo = make_float2(src[0].x, src[0].y), hi = make_float2(src[0].z, src[0].w);
#pragma unroll
            for (int w = 1; w < NSUM; w++) {
                const float4 v = src[(size_t)w * H * D * NCHW];
                lo = __fadd2_rn(lo, make_float2(v.x, v.y));
                hi = __fadd2_rn(hi, make_float2(v.z, v.w));
            }
            ob[r * OUTCH + c] = make_float4(lo.x, lo.y, hi.x, hi.y);
        };
        // pairwise tree over the NSUM warps (fixed order, depth log2 NSUM), all loads of an item
        // issued before the first add
        auto tree_item = [&](int r, int c) {
            const float4 *src = rsrc + (size_t)r * NCHW + c;
            float4 v[NSUM];
#pragma unroll
            for (int w = 0; w < NSUM; w++) v[w] = src[(size_t)w * H * D * NCHW];
#pragma unroll
            for (int st = 1; st < NSUM; st <<= 1) {
#pragma unroll
                for (int w = 0; w + st < NSUM; w += 2 * st) {
                    const float2 lo = __fadd2_rn(make_float2(v[w].x, v[w].y), make_float2(v[w + st].x, v[w + st].y));
                    const float2 hi = __fadd2_rn(make_float2(v[w].z, v[w].w), make_float2(v[w + st].z, v[w + st].w));
                    v[w] = make_float4(lo.x, lo.y, hi.x, hi.y);
                }
            }
            ob[r * OUTCH + c] = v[0];
        };
        // two items per pass when the items split into pairs: 2 NSUM loads in flight before the first
        // add (C3 bwd 15.65 -> 15.53 ms)
        auto tree_pair = [&](int i0, int i1) {
            const float4 *s0 = rsrc + (size_t)(i0 / OUTCH) * NCHW + (i0 % OUTCH);
            const float4 *s1 = rsrc + (size_t)(i1 / OUTCH) * NCHW + (i1 % OUTCH);
            float4 v[NSUM], u[NSUM];
#pragma unroll
            for (int w = 0; w < NSUM; w++) {
                v[w] = s0[(size_t)w * H * D * NCHW];
                u[w] = s1[(size_t)w * H * D * NCHW];
            }
#pragma unroll
            for (int st = 1; st < NSUM; st <<= 1) {
#pragma unroll
                for (int w = 0; w + st < NSUM; w += 2 * st) {
                    float2 lo = __fadd2_rn(make_float2(v[w].x, v[w].y), make_float2(v[w + st].x, v[w + st].y));
                    float2 hi = __fadd2_rn(make_float2(v[w].z, v[w].w), make_float2(v[w + st].z, v[w + st].w));
                    v[w] = make_float4(lo.x, lo.y, hi.x, hi.y);
                    lo = __fadd2_rn(make_float2(u[w].x, u[w].y), make_float2(u[w + st].x, u[w + st].y));
                    hi = __fadd2_rn(make_float2(u[w].z, u[w].w), make_float2(u[w + st].z, u[w + st].w));
                    u[w] = make_float4(lo.x, lo.y, hi.x, hi.y);
                }
            }
            ob[i0] = v[0];  // ob is [RG][OUTCH]: item it sits at it
            ob[i1] = u[0];
        };
        if constexpr (EVEN && !UNI && (RG * OUTCH) % 64 == 0) {
#pragma unroll
            for (int j = 0; j < RG * OUTCH / 64; j++) tree_pair(lane + 64 * j, lane + 64 * j + 32);
        } else if constexpr (EVEN) {
            constexpr int ITEMS = RG * OUTCH;
#pragma unroll
            for (int j = 0; j < (ITEMS + 31) / 32; j++) {
                const int it = lane + 32 * j;
                if (ITEMS % 32 == 0 || it < ITEMS) {
                    if constexpr (UNI) sum_item(it / OUTCH, it % OUTCH);  // (registers: the tree spills there)
                    else tree_item(it / OUTCH, it % OUTCH);
                }
            }
        } else {
            for (int it = lane; it < RG * nch; it += 32) sum_item(it / nch, it % nch);
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&rempty[bi]);
            if (nch > 0) {
                fence_proxy_async_smem();
                // one bulk op per warp and group: this warp's RG x OUTCH block of the group
                const int gs0 = gg * RG;
                const int rho0 = gs0 % STEPS;
                float *dst = a.partial + (((int64_t)blockIdx.x * (STEPS / RG) + rho0 / RG) * NW + warp) * (RG * OUTCH * 4);
                if (GK_NO_PARTIAL) {
                } else if (gs0 < STEPS) bulk_s2g_store(dst, ob, (uint32_t)(RG * OUTCH * 16));
                else bulk_s2g_reduce_add(dst, ob, (uint32_t)(RG * OUTCH * 16));
                bulk_commit();
                // successive slabs add into the same partial rows: keep them ordered
                if (rho0 + RG == STEPS) bulk_wait_all();
            }
        }
        __syncwarp();
    };

    // final signs (sigma) of the labels this lane holds in the s_{R-1} layout -- the
    // forward's store layout and the backward's / transpose's load layout: bit q top, bit W+q bottom
    // (the unitary variant keeps per-slab sfin loads and the general slab path: its register
    // budget is tighter, and the mask measured slower there)
    uint64_t smask = 0;
#pragma unroll
    for (int q = 0; q < (UNI ? 0 : W); q++) {
        const int k = t * W + q;
        const int lt = row_sRm1(k, ne), lb = row_sRm1(ne - 1 - k, ne);
        if (active) {
            const int rt = a.lrow ? a.lrow[lt] : lt, rb = a.lrow ? a.lrow[lb] : lb;
            if (rt < n && a.sfin[lt]) smask |= 1ull << q;
            if (rb < n && a.sfin[lb]) smask |= 1ull << (W + q);
        }
    }
    auto sneg_t = [&](int q) { return ((smask >> q) & 1ull) != 0; };
    auto sneg_b = [&](int q) { return ((smask >> (W + q)) & 1ull) != 0; };
    auto sgn_t = [&](int q, int lt, int rt) -> bool {
        if constexpr (UNI) return rt < n && a.sfin[lt]; else return sneg_t(q);
    };
    auto sgn_b = [&](int q, int lb, int rb) -> bool {
        if constexpr (UNI) return rb < n && a.sfin[lb]; else return sneg_b(q);
    };

    int gst = 0;    // coefficient stages consumed by this CTA
    int grp = 0;    // dtheta ring groups completed by this CTA
    V ZT[KP][W], ZB[KP][W];
    V DT[GRAD ? KP : 1][GRAD ? W : 1], DB[GRAD ? KP : 1][GRAD ? W : 1];
    int xn = 0;          // DEFER: boundary exchanges this warp has published
    bool xpend = false;  // DEFER: the last shift left two boundary registers pending
    // DEFER: fill the registers the last shift took from a neighbour warp (its values of the step whose
    // buffers have parity ppar): forward (shift_down) lane 31's T[W-1] and lane 0's B[0]; backward
    // direction (shift_up, the transpose apply) lane 0's T[0] and lane 31's B[W-1]
    auto xpatch = [&](int ppar) {
        if constexpr (GK_XPRED & 2) {
            // branch-free: clamped broadcast loads, the two boundary lanes select
            const V *xp = xbuf + ((size_t)(ppar * NW + (h > 0 ? warp - 1 : warp)) * 2) * XV;
            const V *xq = xbuf + ((size_t)(ppar * NW + (h < H - 1 ? warp + 1 : warp)) * 2) * XV;
            const bool fp = lane == 0 && h > 0, fq = lane == 31 && h < H - 1;
#pragma unroll
            for (int p = 0; p < KP; p++) {
                const V a0 = xp[XV + p], b0 = xq[p];
                if (UP) {
                    ZT[p][0] = sel_v(fp, a0, ZT[p][0]);
                    ZB[p][W - 1] = sel_v(fq, b0, ZB[p][W - 1]);
                } else {
                    ZB[p][0] = sel_v(fp, a0, ZB[p][0]);
                    ZT[p][W - 1] = sel_v(fq, b0, ZT[p][W - 1]);
                }
                if constexpr (GRAD) {
                    const V a1 = xp[XV + KP + p], b1 = xq[KP + p];
                    DT[p][0] = sel_v(fp, a1, DT[p][0]);
                    DB[p][W - 1] = sel_v(fq, b1, DB[p][W - 1]);
                }
            }
            return;
        }
        const V *xprev = xbuf + ((size_t)(ppar * NW + warp - 1) * 2) * XV;
        const V *xnext = xbuf + ((size_t)(ppar * NW + warp + 1) * 2) * XV;
        if (lane == 0 && h > 0) {
#pragma unroll
            for (int p = 0; p < KP; p++) {
                if (UP) ZT[p][0] = xprev[XV + p];
                else ZB[p][0] = xprev[XV + p];
                if constexpr (GRAD) DT[p][0] = xprev[XV + KP + p];
            }
        }
        if (lane == 31 && h < H - 1) {
#pragma unroll
            for (int p = 0; p < KP; p++) {
                if (UP) ZB[p][W - 1] = xnext[p];
                else ZT[p][W - 1] = xnext[p];
                if constexpr (GRAD) DB[p][W - 1] = xnext[KP + p];
            }
        }
    };

    for (int64_t slab = blockIdx.x; slab < a.nslabs; slab += gridDim.x) {
        const int64_t col0 = slab * C + (int64_t)(cw * LC + g) * K;
        // uniform over the CTA: every column of the slab in range, vector-aligned rows, identity layout
        const bool fast = !UNI && a.vec_ok && a.lrow == nullptr && (slab + 1) * C <= a.m;
        // ---------------- load the slab into the start layout (s_0 forward, s_{R-1} backward)
        if (BM != M_BUILDU && fast) {
            // rows >= n (the odd-n bye, idle lanes) read row 0 and are zeroed after the load
#pragma unroll
            for (int q = 0; q < W; q++) {
                const int k = t * W + q;
                int rt = UP ? row_sRm1(k, ne) : row_s0(k), rb = UP ? row_sRm1(ne - 1 - k, ne) : row_s0(ne - 1 - k);
                if (!active) rt = rb = n;
                const bool zt = rt >= n, zb = rb >= n;
                V vt[KP], vb[KP];
                FastIO<K>::load(a.X + (int64_t)(zt ? 0 : rt) * a.ldx + col0, vt);
                FastIO<K>::load(a.X + (int64_t)(zb ? 0 : rb) * a.ldx + col0, vb);
                const bool nt = UP && sneg_t(q), nb = UP && sneg_b(q);
#pragma unroll
                for (int p = 0; p < KP; p++) {
                    ZT[p][q] = zt ? V{} : vneg_if(vt[p], nt);
                    ZB[p][q] = zb ? V{} : vneg_if(vb[p], nb);
                }
                if constexpr (GRAD) {
                    FastIO<K>::load(a.dY + (int64_t)(zt ? 0 : rt) * a.lddy + col0, vt);
                    FastIO<K>::load(a.dY + (int64_t)(zb ? 0 : rb) * a.lddy + col0, vb);
#pragma unroll
                    for (int p = 0; p < KP; p++) {
                        DT[p][q] = zt ? V{} : vneg_if(vt[p], nt);
                        DB[p][q] = zb ? V{} : vneg_if(vb[p], nb);
                    }
                }
            }
        } else
#pragma unroll
        for (int q = 0; q < W; q++) {
            const int k = t * W + q;
            const int pt = k, pb = ne - 1 - k;
            int lt, lb;  // labels
            if (UP) { lt = row_sRm1(pt, ne); lb = row_sRm1(pb, ne); }
            else    { lt = row_s0(pt);       lb = row_s0(pb); }
            int rt = n, rb = n;  // rows; idle lanes hold zeros and never store
            if (active) { rt = a.lrow ? a.lrow[lt] : lt; rb = a.lrow ? a.lrow[lb] : lb; }
            V vt[KP], vb[KP];
            if constexpr (BM == M_BUILDU && UNI) {
#pragma unroll
                for (int p = 0; p < KP; p++) {  // one complex column per pack: 1 + 0i on the diagonal
                    const int64_t c = (col0 >> 1) + p;
                    vt[p] = make_float2((rt < n && c == rt) ? 1.f : 0.f, 0.f);
                    vb[p] = make_float2((rb < n && c == rb) ? 1.f : 0.f, 0.f);
                }
            } else if constexpr (BM == M_BUILDU) {
#pragma unroll
                for (int p = 0; p < KP; p++) {
                    const int64_t c = col0 + 2 * p;
                    vt[p] = make_float2((rt < n && c == rt) ? 1.f : 0.f, (rt < n && c + 1 == rt) ? 1.f : 0.f);
                    vb[p] = make_float2((rb < n && c == rb) ? 1.f : 0.f, (rb < n && c + 1 == rb) ? 1.f : 0.f);
                }
            } else {
                if (rt < n) IO::load(a.X + (int64_t)rt * a.ldx, col0, a.m, a.vec_ok, vt);
                else for (int p = 0; p < KP; p++) vt[p] = V{};
                if (rb < n) IO::load(a.X + (int64_t)rb * a.ldx, col0, a.m, a.vec_ok, vb);
                else for (int p = 0; p < KP; p++) vb[p] = V{};
            }
            if (UP) {
                const bool nt = sgn_t(q, lt, rt), nb = sgn_b(q, lb, rb);
#pragma unroll
                for (int p = 0; p < KP; p++) { vt[p] = vneg_if(vt[p], nt); vb[p] = vneg_if(vb[p], nb); }
            }
#pragma unroll
            for (int p = 0; p < KP; p++) { ZT[p][q] = vt[p]; ZB[p][q] = vb[p]; }
            if constexpr (GRAD) {
                if (rt < n) IO::load(a.dY + (int64_t)rt * a.lddy, col0, a.m, a.vec_ok, vt);
                else for (int p = 0; p < KP; p++) vt[p] = V{};
                if (rb < n) IO::load(a.dY + (int64_t)rb * a.lddy, col0, a.m, a.vec_ok, vb);
                else for (int p = 0; p < KP; p++) vb[p] = V{};
                const bool nt = sgn_t(q, lt, rt), nb = sgn_b(q, lb, rb);
#pragma unroll
                for (int p = 0; p < KP; p++) {
                    DT[p][q] = vneg_if(vt[p], nt);
                    DB[p][q] = vneg_if(vb[p], nb);
                }
            }
        }

        // ---------------- all 2S steps, UB steps per unrolled body (register renaming of the ring:
        // a body of W steps returns every ring register to its place; UB = W/2 leaves the renaming
        // half way round, and the compiler moves the ring registers at the loop edge)
#pragma unroll 1
        for (int body = 0; body < STEPS / UB; body++) {
            unroll<UB>([&](auto ic) {
                constexpr int uu = decltype(ic)::value;
                constexpr int su = uu % SPS;
                if constexpr (su == 0) {
                    mbar_wait(&full[gst % NSTAGE], (uint32_t)((gst / NSTAGE) & 1));
                    __syncwarp();
                }
                const int srow = UP ? su : (SPS - 1 - su);
                uint32_t fgm = 0;  // M_FG: this step's factoring bits (one table row, warp-uniform)
                if constexpr (FG) fgm = __ldg(a.fgmask + stage_rho0(gst) + srow);
                const uint8_t *sbase = stagebuf + (gst % NSTAGE) * G::STAGEB;
                const float4 *row4 = reinterpret_cast<const float4 *>(sbase + srow * rowb);
                const float4 *ph4 = reinterpret_cast<const float4 *>(sbase + SPS * rowb + srow * (G::PHB / 8) * rowb);
                const float4 *ab4 = reinterpret_cast<const float4 *>(sbase + SPS * 3 * rowb + srow * rowb);
                constexpr int r = uu % RG;
                int bi = 0;
                float4 *ring_dst = nullptr;
                if constexpr (GRAD) {
                    bi = grp % NG;
                    if constexpr (r == 0) {  // the ring group we are about to fill is free
                        mbar_wait(&rempty[bi], (uint32_t)((grp / NG) & 1));
                        __syncwarp();
                    }
                    ring_dst = red + ((size_t)warp * D + bi * RG + r) * NCHW;
                }
                float acc[GRAD ? (LC > 1 ? W : 4) : 1];
                float accp[(GRAD && UNI) ? (LC > 1 ? W : 4) : 1];
#pragma unroll
                for (int jj = 0; jj < W / 2; jj++) {
                    // DEFER: middle pairs 1 .. W/2-2 first, then the two boundary pairs
                    // BFIRST: the quads (4 slots) holding the two ring-boundary slots 0 and W-1 go first, so the
                    // step's shift shuffles (of the rotated T[W-1] and B[0]) can issue half way through the
                    // step and the next step's boundary slots find them done; quads stay contiguous for the
                    // per-quad dtheta ring stores
                    constexpr int NQ = W / 4;
                    const int qd = jj / 2, qp = (!BFIRST || NQ <= 2) ? qd : (qd == 0 ? 0 : (qd == 1 ? NQ - 1 : qd - 1));
                    // DEFER backward: middle quads first, then quad 0 and quad NQ-1 (whole quads)
                    const int qg = qd < NQ - 2 ? qd + 1 : (qd == NQ - 2 ? 0 : NQ - 1);
                    const int pp = !DEFER ? 2 * qp + (jj & 1)
                                 : GRAD ? 2 * qg + (jj & 1)
                                        : (jj < W / 2 - 2 ? jj + 1 : (jj == W / 2 - 2 ? 0 : W / 2 - 1));
                    if constexpr (DEFER) {
                        if (jj == (GRAD ? W / 2 - 4 : W / 2 - 2) && xpend) {
                            constexpr int ppar = (uu + 1) & 1;  // parity of the previous step's buffers
                            mbar_wait(&xb[cw], (uint32_t)((xn - 1) & 1));
                            xpatch(ppar);
                        }
                    }
                    const float4 cf = row4[pp * La + tc];
                    float4 ab = make_float4(0.f, 0.f, 0.f, 0.f);
                    if constexpr (GRAD && UNI) ab = ab4[pp * La + tc];
                    // real backward, one packed pair per slot: both slots' cross products first, then the
                    // two slots' replays interleaved (four independent FFMA2 chains per shear)
                    constexpr bool IL = GRAD && !UNI && KP == 1 && H < 4 && GK_BWD_IL;  // (four-warp columns: 22.9 -> 23.2 ms, off)
                    if constexpr (IL) {
                        const int q0 = 2 * pp, q1 = q0 + 1;
                        acc[LC > 1 ? q0 : (q0 & 3)] = cross_first(DB[0][q0], ZT[0][q0], DT[0][q0], ZB[0][q0]);
                        acc[LC > 1 ? q1 : (q1 & 3)] = cross_first(DB[0][q1], ZT[0][q1], DT[0][q1], ZB[0][q1]);
                        rot_inv2x2(ZT[0][q0], ZB[0][q0], DT[0][q0], DB[0][q0], ZT[0][q1], ZB[0][q1], DT[0][q1], DB[0][q1],
                                   cf.x, cf.y, cf.z, cf.w);
                    } else {
#pragma unroll
                    for (int hh = 0; hh < 2; hh++) {
                        const int q = 2 * pp + hh;
                        const float tq = hh ? cf.z : cf.x, sq = hh ? cf.w : cf.y;
                        float4 ph = make_float4(1.f, 0.f, 1.f, 0.f), pha = ph, phb = ph;
                        if constexpr (UNI && GRAD) ph = ph4[q * La + tc];  // (p_t, q_t, p_b, q_b)
                        if constexpr (UNI && !GRAD) {
                            // (p, q, -q, p) forward / (p, -q, q, p) adjoint, top then bottom
                            pha = ph4[(2 * q) * La + tc];
                            phb = ph4[(2 * q + 1) * La + tc];
                        }
                        if constexpr (GRAD) {
                            // dtheta contribution before this block's inverse rotation:
                            // dz_bottom * z_top - dz_top * z_bottom (Q_e structure, PAPER.md:515-521;
                            // in the unitary variant Re(conj(dz_b) z_t - conj(dz_t) z_b), the same
                            // sum over the (re, im) halves)
                            float c = cross_first(DB[0][q], ZT[0][q], DT[0][q], ZB[0][q]);
#pragma unroll
                            for (int p = 1; p < KP; p++) c = cross_acc(c, DB[p][q], ZT[p][q], DT[p][q], ZB[p][q]);
                            acc[LC > 1 ? q : (q & 3)] = c;
                            if constexpr (UNI) {
                                // dphi: Re(i conj(v) w), w = alpha z_t + beta z_b, v = alpha dz_t + beta dz_b
                                // (P_e structure, in z-space)
                                const float al = hh ? ab.z : ab.x, be = hh ? ab.w : ab.y;
                                float cp = 0.f;
#pragma unroll
                                for (int p = 0; p < KP; p++) {
                                    const V w = fma_v(be, ZB[p][q], mul_v(f2(al), ZT[p][q]));
                                    const V v = fma_v(be, DB[p][q], mul_v(f2(al), DT[p][q]));
                                    cp = phi_acc(cp, v, w);
                                }
                                accp[LC > 1 ? q : (q & 3)] = cp;
                            }
                        }
#pragma unroll
                        for (int p = 0; p < KP; p++) {
                            if (UP) {
                                if constexpr (GRAD) rot_inv2(ZT[p][q], ZB[p][q], DT[p][q], DB[p][q], tq, sq);
                                else rot_inv(ZT[p][q], ZB[p][q], tq, sq);
                                if constexpr (UNI && GRAD) {  // G^dagger = diag(conj phases) R^T
                                    ZT[p][q] = cmulc(ZT[p][q], ph.x, ph.y);
                                    ZB[p][q] = cmulc(ZB[p][q], ph.z, ph.w);
                                    DT[p][q] = cmulc(DT[p][q], ph.x, ph.y);
                                    DB[p][q] = cmulc(DB[p][q], ph.z, ph.w);
                                } else if constexpr (UNI) {
                                    ZT[p][q] = cmul4(ZT[p][q], pha);
                                    ZB[p][q] = cmul4(ZB[p][q], phb);
                                }
                            } else {
                                if constexpr (UNI) {  // G = R diag(phases): phase first
                                    ZT[p][q] = cmul4(ZT[p][q], pha);
                                    ZB[p][q] = cmul4(ZB[p][q], phb);
                                }
                                if constexpr (FG) {
                                    // (x, y) = (top, bottom) or, with the second factoring, (bottom, top):
                                    // top' = x - a y, bottom' = y + b x (2 FFMA)
                                    const bool fb = (fgm >> q) & 1u;
                                    const V x = fb ? ZB[p][q] : ZT[p][q], y = fb ? ZT[p][q] : ZB[p][q];
                                    ZT[p][q] = fma_v(-tq, y, x);
                                    ZB[p][q] = fma_v(sq, x, y);
                                } else {
                                    rot_fwd(ZT[p][q], ZB[p][q], tq, sq);
                                }
                            }
                        }
                    }
                    }  // IL
                    if constexpr (GRAD && LC == 1) {
                        // one lane per column group and warp: the per-slot sums go straight to the ring
                        if (pp & 1) {
                            ring_dst[(pp >> 1) * LW + tl] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                            if constexpr (UNI)
                                ring_dst[NCHW1 + (pp >> 1) * LW + tl] = make_float4(accp[0], accp[1], accp[2], accp[3]);
                        }
                    }
                }
                if constexpr (GRAD) {
                    if constexpr (LC > 1 && !UNI && W / LC >= 4 && RS_LC) {
                        // several column groups per warp share the slots: reduce-scatter over the
                        // groups (log2 LC butterfly rounds, each lane keeps half of its live sums and
                        // ships the other half) instead of an all-reduce of every slot -- W (LC-1)/LC
                        // shuffles per lane and step instead of W log2 LC; group g ends up with the
                        // W/LC slots at off(g) and stores them, the ring layout is unchanged
                        int off = 0;
                        unroll<ilog2(LC)>([&](auto jc) {
                            constexpr int j = decltype(jc)::value;
                            constexpr int h = W >> (j + 1);  // live sums after this round
                            const bool hi = (lane >> (ilog2(LW) + j)) & 1;
#pragma unroll
                            for (int i = 0; i < h; i++) {
                                const float send = hi ? acc[i] : acc[h + i];
                                const float keep = hi ? acc[h + i] : acc[i];
                                acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, LW << j);
                            }
                            if (hi) off += h;
                        });
#pragma unroll
                        for (int k = 0; k < W / LC / 4; k++)
                            ring_dst[(off / 4 + k) * LW + tl] =
                                make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
                    } else if constexpr (LC > 1) {
#pragma unroll
                        for (int q = 0; q < W; q++) {
#pragma unroll
                            for (int o = LW; o < 32; o <<= 1) {
                                acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
                                if constexpr (UNI) accp[q] += __shfl_xor_sync(0xffffffffu, accp[q], o);
                            }
                        }
                        if (g == 0) {
#pragma unroll
                            for (int q4 = 0; q4 < W / 4; q4++) {
                                ring_dst[q4 * LW + tl] =
                                    make_float4(acc[4 * q4], acc[4 * q4 + 1], acc[4 * q4 + 2], acc[4 * q4 + 3]);
                                if constexpr (UNI)
                                    ring_dst[NCHW1 + q4 * LW + tl] =
                                        make_float4(accp[4 * q4], accp[4 * q4 + 1], accp[4 * q4 + 2], accp[4 * q4 + 3]);
                            }
                        }
                    }
                    // warps w and w+4 share an SMSP: the low half reduces the previous group at step
                    // LO of this one, the high half at RG/2 - 1, so one of them keeps the FMA pipe busy;
                    // LO = RG - 2 (not the group's last step) leaves the low half a step of slack
                    // before the next group's rempty wait (C3 bwd 15.74 -> 15.63 ms)
                    constexpr int LO = RG >= 4 ? RG - 2 : RG - 1;
                    // ONE_SITE: every warp reduces at step LO (one inlined copy of the reduction per group
                    // instead of two: the unitary backward's body does not fit the instruction cache)
                    constexpr bool ONE_SITE = UNI && GK_UNI_ONE_SITE;
                    if constexpr (r == LO) {
                        if ((ONE_SITE || ((warp >> 2) & 1) == 0) && grp >= 1) reduce_group(grp - 1);
                    }
                    if constexpr (r == RG - 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&rfull[bi]);
                        grp++;
                    }
                    if constexpr (r == RG / 2 - 1 && NW > 4 && !ONE_SITE) {
                        // (no high half in 4-warp CTAs: the call site would only cost instruction cache)
                        if (((warp >> 2) & 1) == 1 && grp >= 1) reduce_group(grp - 1);
                    }
                }
                // ring shift to the next block's layout (Fig. 1)
                if constexpr (H == 1) {
#pragma unroll
                    for (int p = 0; p < KP; p++) {
                        if (UP) {
                            shift_up<W>(ZT[p], ZB[p], first, last, L);
                            if constexpr (GRAD) shift_up<W>(DT[p], DB[p], first, last, L);
                        } else {
                            shift_down<W>(ZT[p], ZB[p], first, last, L);
                        }
                    }
                } else {
                    // values crossing a warp boundary: publish, named barrier of the group, read
                    constexpr int par = uu & 1;  // double buffer (W is even)
                    V *xo = xbuf + ((size_t)(par * NW + warp) * 2) * XV;  // [0]: to warp h-1, [1]: to warp h+1
                    if ((GK_XPRED & 1) && (!DEFER || (GK_XPRED & 2))) {
                        // branch-free publish: lanes 0 and 31 store through predicated STS (no divergent
                        // region per step), the same slots as below
                        const bool pub = lane == 0 || lane == 31;
#pragma unroll
                        for (int p = 0; p < KP; p++) {
                            if (UP) {
                                st_shared_if(pub, xo + (lane == 31 ? XV + p : p), lane == 31 ? ZT[p][W - 1] : ZB[p][0]);
                                if constexpr (GRAD)
                                    st_shared_if(pub, xo + (lane == 31 ? XV + KP + p : KP + p), lane == 31 ? DT[p][W - 1] : DB[p][0]);
                            } else {
                                st_shared_if(pub, xo + (lane == 0 ? p : XV + p), lane == 0 ? ZT[p][0] : ZB[p][W - 1]);
                            }
                        }
                    } else if (UP) {
                        // lane t+1 needs my T[W-1] (from_prev), lane t-1 needs my B[0] (from_next)
                        if (lane == 31) {
#pragma unroll
                            for (int p = 0; p < KP; p++) {
                                xo[XV + p] = ZT[p][W - 1];
                                if constexpr (GRAD) xo[XV + KP + p] = DT[p][W - 1];
                            }
                        }
                        if (lane == 0) {
#pragma unroll
                            for (int p = 0; p < KP; p++) {
                                xo[p] = ZB[p][0];
                                if constexpr (GRAD) xo[KP + p] = DB[p][0];
                            }
                        }
                    } else {
                        // lane t-1 needs my T[0] (its from_next), lane t+1 needs my B[W-1] (its from_prev)
                        if (lane == 0) {
#pragma unroll
                            for (int p = 0; p < KP; p++) xo[p] = ZT[p][0];
                        }
                        if (lane == 31) {
#pragma unroll
                            for (int p = 0; p < KP; p++) xo[XV + p] = ZB[p][W - 1];
                        }
                    }
                    if constexpr (DEFER) {
                        // publish and go on: the pending boundary registers are patched next step
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&xb[cw]);
                        xn++;
                        xpend = true;
                    } else {
                        named_bar(1 + cw, 32 * H);
                    }
                    const V *xprev = xbuf + ((size_t)(par * NW + warp - 1) * 2) * XV;  // warp h-1 of my group
                    const V *xnext = xbuf + ((size_t)(par * NW + warp + 1) * 2) * XV;  // warp h+1
                    const bool from_x_prev = !DEFER && (lane == 0 && h > 0);
                    const bool from_x_next = !DEFER && (lane == 31 && h < H - 1);
                    if constexpr ((GK_XPRED & 1) && !DEFER) {
                        // branch-free read: every lane loads (clamped, always valid addresses; one broadcast
                        // wavefront each) and the two boundary lanes select
                        const V *xp = xbuf + ((size_t)(par * NW + (h > 0 ? warp - 1 : warp)) * 2) * XV;
                        const V *xq = xbuf + ((size_t)(par * NW + (h < H - 1 ? warp + 1 : warp)) * 2) * XV;
#pragma unroll
                        for (int p = 0; p < KP; p++) {
                            if (UP) {
                                const V lp = xp[XV + p], ln = xq[p];
                                V fp = shfl_up_v(ZT[p][W - 1], 32), fn = shfl_dn_v(ZB[p][0], 32);
                                fp = sel_v(from_x_prev, lp, fp);
                                fn = sel_v(from_x_next, ln, fn);
                                shift_up_with<W>(ZT[p], ZB[p], first, last, fp, fn);
                                if constexpr (GRAD) {
                                    const V lq = xp[XV + KP + p], lr = xq[KP + p];
                                    V dp = shfl_up_v(DT[p][W - 1], 32), dn = shfl_dn_v(DB[p][0], 32);
                                    dp = sel_v(from_x_prev, lq, dp);
                                    dn = sel_v(from_x_next, lr, dn);
                                    shift_up_with<W>(DT[p], DB[p], first, last, dp, dn);
                                }
                            } else {
                                const V ln = xq[p], lp = xp[XV + p];
                                V fn = shfl_dn_v(ZT[p][0], 32), fp = shfl_up_v(ZB[p][W - 1], 32);
                                fn = sel_v(from_x_next, ln, fn);
                                fp = sel_v(from_x_prev, lp, fp);
                                shift_down_with<W>(ZT[p], ZB[p], first, last, fn, fp);
                            }
                        }
                    } else {
#pragma unroll
                    for (int p = 0; p < KP; p++) {
                        if (UP) {
                            V fp = shfl_up_v(ZT[p][W - 1], 32), fn = shfl_dn_v(ZB[p][0], 32);
                            if (from_x_prev) fp = xprev[XV + p];
                            if (from_x_next) fn = xnext[p];
                            shift_up_with<W>(ZT[p], ZB[p], first, last, fp, fn);
                            if constexpr (GRAD) {
                                V dp = shfl_up_v(DT[p][W - 1], 32), dn = shfl_dn_v(DB[p][0], 32);
                                if (from_x_prev) dp = xprev[XV + KP + p];
                                if (from_x_next) dn = xnext[KP + p];
                                shift_up_with<W>(DT[p], DB[p], first, last, dp, dn);
                            }
                        } else {
                            V fn = shfl_dn_v(ZT[p][0], 32), fp = shfl_up_v(ZB[p][W - 1], 32);
                            if (from_x_next) fn = xnext[p];
                            if (from_x_prev) fp = xprev[XV + p];
                            shift_down_with<W>(ZT[p], ZB[p], first, last, fn, fp);
                        }
                    }
                    }  // !GK_XPRED
                }
                if constexpr (su == SPS - 1) {
                    // release the stage buffer; the LAST warp to release it refills it with the
                    // stage NSTAGE ahead (no warp ever waits to act as the producer)
                    __syncwarp();
                    if (lane == 0) {
                        const int b = gst % NSTAGE;
                        __threadfence_block();  // this warp's reads of buffer b happen-before the release
                        if (atomicAdd(&released[b], 1u) == NW - 1) {
                            __threadfence_block();
                            released[b] = 0;
                            const int nxt = gst + NSTAGE;
                            if (nxt < total_stages) {
                                fence_proxy_async_smem();
                                issue_stage(nxt, b);
                            }
                        }
                    }
                    __syncwarp();
                    gst++;
                }
            });
        }

        if constexpr (DEFER) {
            if (xpend) {  // the last step's exchange
                mbar_wait(&xb[cw], (uint32_t)((xn - 1) & 1));
                xpatch((UB - 1) & 1);
                xpend = false;
            }
        }
        // ---------------- store from the end layout (s_{R-1} forward, s_0 backward)
        if (BM == M_BWD && a.Y == nullptr) continue;
        if constexpr (FG) {
            // y = d_final * z per row (identity layout only)
#pragma unroll
            for (int q = 0; q < W; q++) {
                const int k = t * W + q;
                const int lt = row_sRm1(k, ne), lb = row_sRm1(ne - 1 - k, ne);
                V vt[KP], vb[KP];
                const float st = lt < n ? __ldg(a.sfg + lt) : 0.f, sb = lb < n ? __ldg(a.sfg + lb) : 0.f;
#pragma unroll
                for (int p = 0; p < KP; p++) {
                    vt[p] = mul_v(f2v<V>(st), ZT[p][q]);
                    vb[p] = mul_v(f2v<V>(sb), ZB[p][q]);
                }
                if (active && lt < n) IO::store(a.Y + (int64_t)lt * a.ldy, col0, a.m, a.vec_ok, vt);
                if (active && lb < n) IO::store(a.Y + (int64_t)lb * a.ldy, col0, a.m, a.vec_ok, vb);
            }
            continue;
        }
        if (fast) {
#pragma unroll
            for (int q = 0; q < W; q++) {
                const int k = t * W + q;
                const int rt = UP ? row_s0(k) : row_sRm1(k, ne), rb = UP ? row_s0(ne - 1 - k) : row_sRm1(ne - 1 - k, ne);
                V vt[KP], vb[KP];
                const bool nt = !UP && sneg_t(q), nb = !UP && sneg_b(q);
#pragma unroll
                for (int p = 0; p < KP; p++) {
                    if constexpr (GRAD) { vt[p] = DT[p][q]; vb[p] = DB[p][q]; }
                    else { vt[p] = vneg_if(ZT[p][q], nt); vb[p] = vneg_if(ZB[p][q], nb); }
                }
                if (active && rt < n) FastIO<K>::store(a.Y + (int64_t)rt * a.ldy + col0, vt);
                if (active && rb < n) FastIO<K>::store(a.Y + (int64_t)rb * a.ldy + col0, vb);
            }
            continue;
        }
#pragma unroll
        for (int q = 0; q < W; q++) {
            const int k = t * W + q;
            const int pt = k, pb = ne - 1 - k;
            int lt, lb;
            if (UP) { lt = row_s0(pt); lb = row_s0(pb); }
            else    { lt = row_sRm1(pt, ne); lb = row_sRm1(pb, ne); }
            int rt = n, rb = n;
            if (active) { rt = a.lrow ? a.lrow[lt] : lt; rb = a.lrow ? a.lrow[lb] : lb; }
            V vt[KP], vb[KP];
#pragma unroll
            for (int p = 0; p < KP; p++) {
                if constexpr (GRAD) { vt[p] = DT[p][q]; vb[p] = DB[p][q]; }
                else { vt[p] = ZT[p][q]; vb[p] = ZB[p][q]; }
            }
            if (!UP) {
                const bool nt = sgn_t(q, lt, rt), nb = sgn_b(q, lb, rb);
#pragma unroll
                for (int p = 0; p < KP; p++) { vt[p] = vneg_if(vt[p], nt); vb[p] = vneg_if(vb[p], nb); }
            }
            if (rt < n) IO::store(a.Y + (int64_t)rt * a.ldy, col0, a.m, a.vec_ok, vt);
            if (rb < n) IO::store(a.Y + (int64_t)rb * a.ldy, col0, a.m, a.vec_ok, vb);
        }
    }
    if constexpr (GRAD) {
        if (grp >= 1) reduce_group(grp - 1);  // both halves: the last group is still pending
        if (lane == 0) bulk_wait_all();
    }
}


}  // namespace gk
