// tc_gemm.cuh -- hand-written sm_100a tensor-core GEMM in 3xTF32 for the GEMM path (SURVEY §8(f2),
// PAPER.md:209-222): D = A B^T over K with fp32 operands, ~fp32 accuracy from three TF32 products
// (a = a_hi + a_lo with a_hi exactly TF32: a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi).
//
// One CTA computes a BM x BN tile of D over its K range (split-K: blockIdx.z), warp-specialised:
//   warp 0      TMA producer: raw fp32 tiles of A and B (SWIZZLE_128B) into a stage's "hi" buffers;
//   warp 1      MMA issuer (one elected thread): per 32-wide k-block 3 x 4 tcgen05.mma.kind::tf32
//               (M = 128, N = BN, K = 8) into a TMEM accumulator; tcgen05.commit frees the stage;
//   warp 2      TMEM allocator;
//   warps 4-7   the 3xTF32 split in the pipeline: the tensor core reads an fp32 operand as TF32 by
//               truncation (the low 13 mantissa bits ignored; measured by tools/tc_trunc.cu), so the
//               raw tile already is "hi" = trunc(x); per stage they write lo = x - trunc(x) (exact in
//               fp32) into a second buffer of the same swizzled layout -- the split is elementwise,
//               so it never needs to know the swizzle -- then fence the async proxy and arrive;
//               after the mainloop they are the epilogue:
//               tcgen05.ld of the accumulator, stored to global with the M index contiguous.
// Operand layouts (both operands are described as "rows x K" = M x K for A and N x K for B):
//   K-major  : element (r, k) at p + r ld + k  -- TMA box {32 k, R rows}, canonical K-major SW128
//              (8-row x 128 B atoms, SBO = 1024 B), the k-step of 8 advances the start by 32 B;
//   MN-major : element (r, k) at p + k ld + r  -- TMA boxes {32 r, 32 k} per 32-row block. For
//              32-bit operands the only MN-major UMMA layout is SWIZZLE_128B_BASE32B (32-byte chunks
//              swizzled within 128-byte rows, 4-row x 128 B atoms; the TMA's SWIZZLE_128B_ATOM_32B
//              writes it): LBO = 4096 B between 32-row blocks, SBO = 512 B between 4-deep k atoms,
//              the k-step of 8 advances the start by 1024 B.
// Output: D[m][n] is stored at out[z * zstride + n * ldo + m] (the m index contiguous: a warp's
// 32 TMEM lanes are 32 consecutive m, so every store instruction writes 128 contiguous bytes).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace tcg {

constexpr int BM = 128, BN = 256, BK = 32, NST = 2;
constexpr int TILE_A = BM * BK * 4;            // 16 KB
constexpr int TILE_B = BN * BK * 4;            // 32 KB
constexpr int HI_BYTES = TILE_A + TILE_B;      // raw / hi part of a stage
constexpr int STAGE_BYTES = 2 * HI_BYTES;      // hi A | hi B | lo A | lo B
constexpr int NTHREADS = 256;
constexpr size_t SMEM_BYTES = 1024 + (size_t)NST * STAGE_BYTES + 256;  // 1 KB alignment slack + barriers

struct Args {
    int M, N, K;          // D is M x N, contraction over K (per split: kchunk)
    int kchunk;           // K range per blockIdx.z (multiple of BK)
    float *out;
    int64_t ldo, zstride;
    int accumulate;       // 1: out += D (K cut into sequential launches), 0: out = D
};

// the same box delivered to the same shared-memory offset (and barrier) of every CTA in ctamask
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar,
                                               uint16_t ctamask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(gk::smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(gk::smem_u32(bar)), "h"(ctamask)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(gk::smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(gk::smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor (sm_100): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), layout [61,64): SWIZZLE_128B = 2 (K-major), SWIZZLE_128B_BASE32B = 1 (MN-major tf32)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
// operand descriptor for k-step ks of a stage tile at base
template <bool MN>
__device__ __forceinline__ uint64_t odesc(uint32_t base, int ks) {
    if constexpr (MN) return sdesc(base + ks * 1024u, 4096u, 512u, 1u);
    else return sdesc(base + ks * 32u, 16u, 1024u, 2u);
}

// kind::tf32 instruction descriptor: D f32 [4,6) = 1, A/B tf32 [7,10) / [10,13) = 2, A/B major
// (0 K, 1 MN) bits 15 / 16, N >> 3 [17,23), M >> 4 [24,29)
template <bool AMN, bool BMN>
__host__ __device__ constexpr uint32_t idesc_tf32() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// arrive on the barrier at this offset in every CTA of ctamask once this thread's MMAs are done
__device__ __forceinline__ void mma_commit_mc(uint64_t *bar, uint16_t ctamask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(gk::smem_u32(bar)), "h"(ctamask)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(gk::smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// x - trunc_tf32(x): exact in fp32 (the low 13 mantissa bits of x)
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// Clusters of CL = 2 CTAs along M share their B tile: each loads half of it with a multicast TMA
// into both CTAs' stage (B's L2 -> SM traffic halves), and each CTA's MMA commit releases the stage in
// both (empty barriers count CL arrivals), so neither overwrites a stage its peer still reads.
constexpr int CL = 2;

template <bool AMN, bool BMN>
__global__ void __cluster_dims__(1, CL, 1) __launch_bounds__(NTHREADS, 1)
k_gemm3_1sm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, const Args a) {
    extern __shared__ uint8_t smem_raw[];
    // SWIZZLE_128B atoms need 1024-byte alignment
    uint8_t *smem = reinterpret_cast<uint8_t *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)NST * STAGE_BYTES);
    uint64_t *conv = full + NST;
    uint64_t *empty = conv + NST;
    uint64_t *accb = empty + NST;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accb + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // n-tiles vary fastest: the CTAs that share an A tile (the streamed operand) run at the same time,
    // so it comes from DRAM once and from L2 for the others
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
    const int kbeg = blockIdx.z * a.kchunk;
    const int kend = min(a.K, kbeg + a.kchunk);
    const int nkb = (kend - kbeg + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; s++) {
            gk::mbar_init(&full[s], 1);
            gk::mbar_init(&conv[s], 4);
            gk::mbar_init(&empty[s], CL);
        }
        gk::mbar_init(accb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        gk::fence_proxy_async_smem();
    }
    if (warp == 2) {  // TMEM: BN fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(gk::smem_u32(tmem_slot)),
                     "n"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers exist before any multicast write or remote arrive
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t crank = cluster_rank();
    constexpr uint16_t kMask = (1u << CL) - 1;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % NST, j = kb / NST;
                if (j > 0) gk::mbar_wait(&empty[s], (uint32_t)((j - 1) & 1));
                uint8_t *st = smem + (size_t)s * STAGE_BYTES;
                gk::mbar_expect_tx(&full[s], HI_BYTES);
                const int k0 = kbeg + kb * BK;
                if constexpr (AMN) {
#pragma unroll
                    for (int b = 0; b < BM / 32; b++) tma_load_2d(st + b * 4096, &tma_a, m0 + 32 * b, k0, &full[s]);
                } else {
                    tma_load_2d(st, &tma_a, k0, m0, &full[s]);
                }
                // this CTA's half of B, multicast into both CTAs of the cluster
                if constexpr (BMN) {
#pragma unroll
                    for (int b = 0; b < BN / 32 / CL; b++) {
                        const int bb = (int)crank * (BN / 32 / CL) + b;
                        tma_load_2d_mc(st + TILE_A + bb * 4096, &tma_b, n0 + 32 * bb, k0, &full[s], kMask);
                    }
                } else {
                    tma_load_2d_mc(st + TILE_A + crank * (TILE_B / CL), &tma_b, k0, n0 + (int)crank * (BN / CL),
                                   &full[s], kMask);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32<AMN, BMN>();
            const uint32_t base = gk::smem_u32(smem);
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % NST, j = kb / NST;
                gk::mbar_wait(&conv[s], (uint32_t)(j & 1));
                tc_fence_after();
                const uint32_t ahi = base + s * STAGE_BYTES, bhi = ahi + TILE_A;
                const uint32_t alo = ahi + HI_BYTES, blo = bhi + HI_BYTES;
#pragma unroll
                for (int ks = 0; ks < BK / 8; ks++) {
                    const uint64_t dah = odesc<AMN>(ahi, ks), dal = odesc<AMN>(alo, ks);
                    const uint64_t dbh = odesc<BMN>(bhi, ks), dbl = odesc<BMN>(blo, ks);
                    const uint32_t acc0 = (kb > 0 || ks > 0) ? 1u : 0u;
                    // small cross terms first, then hi x hi
#ifndef TCG_ONE_MMA
                    mma_tf32(tmem, dah, dbl, idesc, acc0);
                    mma_tf32(tmem, dal, dbh, idesc, 1u);
                    mma_tf32(tmem, dah, dbh, idesc, 1u);
#else
                    (void)dal; (void)dbl;
                    mma_tf32(tmem, dah, dbh, idesc, acc0);
#endif
                }
                mma_commit_mc(&empty[s], kMask);  // frees the stage (in both CTAs) once these MMAs have read it
            }
            mma_commit(accb);  // the accumulator is complete
        }
    } else if (warp >= 4) {
        // ---- the 3xTF32 split of every stage (warpgroup 1: threads 128..255)
        const int t = threadIdx.x - 128;
        for (int kb = 0; kb < nkb; kb++) {
            const int s = kb % NST, j = kb / NST;
            gk::mbar_wait(&full[s], (uint32_t)(j & 1));
            float4 *hi = reinterpret_cast<float4 *>(smem + (size_t)s * STAGE_BYTES);
            float4 *lo = reinterpret_cast<float4 *>(smem + (size_t)s * STAGE_BYTES + HI_BYTES);
#ifndef TCG_NO_CONVERT
#pragma unroll 4
            for (int i = t; i < HI_BYTES / 16; i += 128) {
                const float4 x = hi[i];
                lo[i] = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
            }
#else
            (void)hi; (void)lo;
#endif
            gk::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
#ifdef TCG_DEBUG
            if (t == 0 && kb == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
                const float *hf = reinterpret_cast<const float *>(hi), *lf = reinterpret_cast<const float *>(lo);
                printf("DBG conv: tmem=%08x hiA %g %g %g %g hiB %g %g loA %g %g\n", tmem, hf[0], hf[1], hf[2], hf[3],
                       hf[TILE_A / 4], hf[TILE_A / 4 + 1], lf[0], lf[1]);
            }
#endif
            __syncwarp();
            if (lane == 0) gk::mbar_arrive(&conv[s]);
        }
        // ---- epilogue: TMEM lanes 32 q .. 32 q + 31 (this warp's quarter) = rows m of the tile
        const int q = warp & 3;
        gk::mbar_wait(accb, 0);
        tc_fence_after();
        const int mrow = m0 + 32 * q + lane;
        float *outz = a.out + (int64_t)blockIdx.z * a.zstride;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
            uint32_t v[32];
            const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#ifdef TCG_DEBUG
            if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0 && c == 0)
                printf("DBG epi q=%d taddr=%08x v %g %g %g %g\n", q, taddr, __uint_as_float(v[0]), __uint_as_float(v[1]),
                       __uint_as_float(v[2]), __uint_as_float(v[3]));
#endif
            if (mrow < a.M) {
#pragma unroll
                for (int jj = 0; jj < 32; jj++) {
                    const int nn = n0 + c + jj;
                    if (nn < a.N) {
                        float *o = outz + (int64_t)nn * a.ldo + mrow;
                        *o = a.accumulate ? *o + __uint_as_float(v[jj]) : __uint_as_float(v[jj]);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while its peer may still write its smem or arrive on its barriers
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
    }
}

}  // namespace tcg

namespace tcg {

// ------------------------------------------------------------------ two-SM (cta_group::2) variant
// A CTA pair (cluster along M) computes a 256 x 256 tile: each CTA holds its own 128 rows of A and
// one 128-row half of B in shared memory (raw + lo, 64 KB per stage, three stages); the even CTA's
// single elected thread issues tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 8), which reads A and
// B from both CTAs' shared memory and accumulates each CTA's 128 rows into that CTA's TMEM. Per CTA
// the tensor core reads half the B bytes of the one-SM kernel. Both CTAs' split warps arrive on the
// leader's conversion barrier (remote arrive, cluster scope); the leader's commits multicast to both
// CTAs' stage-empty and accumulator barriers.
constexpr int BN2 = 256, TILE_B2 = (BN2 / 2) * BK * 4;             // 16 KB: this CTA's half of B
constexpr int HI2 = TILE_A + TILE_B2, STAGE2 = 2 * HI2, NST2 = 3;  // 64 KB per stage
constexpr size_t SMEM2 = 1024 + (size_t)NST2 * STAGE2 + 256;

template <bool AMN, bool BMN>
__host__ __device__ constexpr uint32_t idesc_tf32_2sm() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
           ((uint32_t)(BN2 >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32_2sm(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t *bar, uint16_t ctamask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(gk::smem_u32(bar)), "h"(ctamask)
                 : "memory");
}
// arrive on the barrier at this shared-memory offset in CTA `rank` of the cluster (release, cluster scope)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
    uint32_t raddr;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(gk::smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *b, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(gk::smem_u32(b)), "r"(parity)
            : "memory");
    }
}

// grid (2 x N tiles, M tile pairs, K splits), clusters of 2 along x: x = 2 n_tile + rank, so the CTA
// pairs of all N tiles of one M pair run together (the streamed A tile comes from DRAM once)
template <bool AMN, bool BMN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
k_gemm3(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, const Args a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)NST2 * STAGE2);
    uint64_t *conv = full + NST2;
    uint64_t *empty = conv + NST2;
    uint64_t *accb = empty + NST2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accb + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const int n0 = (blockIdx.x >> 1) * BN2, m0 = (blockIdx.y * 2 + (int)crank) * BM;  // this CTA's 128 of 256 rows
    const int kbeg = blockIdx.z * a.kchunk;
    const int kend = min(a.K, kbeg + a.kchunk);
    const int nkb = (kend - kbeg + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST2; s++) {
            gk::mbar_init(&full[s], 1);
            gk::mbar_init(&conv[s], 8);  // the split warps of both CTAs (used in the even CTA)
            gk::mbar_init(&empty[s], 1);
        }
        gk::mbar_init(accb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        gk::fence_proxy_async_smem();
    }
    if (warp == 2) {  // TMEM of each CTA of the pair: 256 fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(gk::smem_u32(tmem_slot)),
                     "n"(BN2));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % NST2, j = kb / NST2;
                if (j > 0) gk::mbar_wait(&empty[s], (uint32_t)((j - 1) & 1));
                uint8_t *st = smem + (size_t)s * STAGE2;
                gk::mbar_expect_tx(&full[s], HI2);
                const int k0 = kbeg + kb * BK;
                if constexpr (AMN) {
#pragma unroll
                    for (int b = 0; b < BM / 32; b++) tma_load_2d(st + b * 4096, &tma_a, m0 + 32 * b, k0, &full[s]);
                } else {
                    tma_load_2d(st, &tma_a, k0, m0, &full[s]);
                }
                const int nh = n0 + (int)crank * (BN2 / 2);  // this CTA's half of the N tile
                if constexpr (BMN) {
#pragma unroll
                    for (int b = 0; b < BN2 / 2 / 32; b++)
                        tma_load_2d(st + TILE_A + b * 4096, &tma_b, nh + 32 * b, k0, &full[s]);
                } else {
                    tma_load_2d(st + TILE_A, &tma_b, k0, nh, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && crank == 0) {
            constexpr uint32_t idesc = idesc_tf32_2sm<AMN, BMN>();
            const uint32_t base = gk::smem_u32(smem);
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % NST2, j = kb / NST2;
                mbar_wait_cluster(&conv[s], (uint32_t)(j & 1));
                tc_fence_after();
                const uint32_t ahi = base + s * STAGE2, bhi = ahi + TILE_A;
                const uint32_t alo = ahi + HI2, blo = bhi + HI2;
#pragma unroll
                for (int ks = 0; ks < BK / 8; ks++) {
                    const uint64_t dah = odesc<AMN>(ahi, ks), dal = odesc<AMN>(alo, ks);
                    const uint64_t dbh = odesc<BMN>(bhi, ks), dbl = odesc<BMN>(blo, ks);
                    const uint32_t acc0 = (kb > 0 || ks > 0) ? 1u : 0u;
                    mma_tf32_2sm(tmem, dah, dbl, idesc, acc0);
                    mma_tf32_2sm(tmem, dal, dbh, idesc, 1u);
                    mma_tf32_2sm(tmem, dah, dbh, idesc, 1u);
                }
                mma_commit_2sm(&empty[s], 3);  // frees stage s in both CTAs once these MMAs have read it
            }
            mma_commit_2sm(accb, 3);  // both CTAs' accumulators are complete
        }
    } else if (warp >= 4) {
        const int t = threadIdx.x - 128;
        for (int kb = 0; kb < nkb; kb++) {
            const int s = kb % NST2, j = kb / NST2;
            gk::mbar_wait(&full[s], (uint32_t)(j & 1));
            float4 *hi = reinterpret_cast<float4 *>(smem + (size_t)s * STAGE2);
            float4 *lo = reinterpret_cast<float4 *>(smem + (size_t)s * STAGE2 + HI2);
#pragma unroll 4
            for (int i = t; i < HI2 / 16; i += 128) {
                const float4 x = hi[i];
                lo[i] = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
            }
            gk::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(&conv[s], 0);  // the even CTA issues the MMAs
        }
        const int q = warp & 3;
        gk::mbar_wait(accb, 0);
        tc_fence_after();
        const int mrow = m0 + 32 * q + lane;
        float *outz = a.out + (int64_t)blockIdx.z * a.zstride;
#pragma unroll 1
        for (int c = 0; c < BN2; c += 32) {
            uint32_t v[32];
            const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (mrow < a.M) {
#pragma unroll
                for (int jj = 0; jj < 32; jj++) {
                    const int nn = n0 + c + jj;
                    if (nn < a.N) {
                        float *o = outz + (int64_t)nn * a.ldo + mrow;
                        *o = a.accumulate ? *o + __uint_as_float(v[jj]) : __uint_as_float(v[jj]);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN2));
    }
}

}  // namespace tcg

// ------------------------------------------------------------------ host side
namespace tcg {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled from the driver through the runtime (no link-time libcuda dependency)
inline EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

// TMA can describe the operand: 16-byte aligned base, leading dimension a multiple of 4 floats
inline bool tma_ok(const float *p, int64_t ld) { return ((uintptr_t)p % 16) == 0 && (ld % 4) == 0 && ld > 0; }

// operand "rows x K": mn_major -> element (r, k) at p + k ld + r, else p + r ld + k
inline bool make_map(CUtensorMap *map, const float *p, int64_t rows, int64_t K, int64_t ld, bool mn_major,
                     int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2], strides[1];
    cuuint32_t box[2], es[2] = {1, 1};
    if (mn_major) {
        dims[0] = (cuuint64_t)rows; dims[1] = (cuuint64_t)K; box[0] = 32; box[1] = 32;
    } else {
        dims[0] = (cuuint64_t)K; dims[1] = (cuuint64_t)rows; box[0] = 32; box[1] = (cuuint32_t)box_rows;
    }
    strides[0] = (cuuint64_t)ld * 4;
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Operand {
    const float *p;
    int64_t ld;
    bool mn;  // MN-major (the row index contiguous)
};

// D (M x N) = A (M x K) B (N x K)^T in 3xTF32, stored at out[z zstride + n ldo + m]; the K range is cut
// into splits of kchunk (a multiple of BK), split z written to its own output block. Returns a
// cudaError_t (cudaErrorNotSupported if the driver has no tensor-map encoder or an operand is not
// TMA-describable).
template <bool AMN, bool BMN>
inline cudaError_t gemm3_launch(const Operand &A, const Operand &B, int M, int N, int K, int kchunk, float *out,
                                int64_t ldo, int64_t zstride, int accumulate, cudaStream_t st) {
    CUtensorMap ma, mb;
    // the B map's box is half an N tile in both kernels (BN / CL = BN2 / 2 = 128 rows)
    if (!make_map(&ma, A.p, M, K, A.ld, AMN, BM) || !make_map(&mb, B.p, N, K, B.ld, BMN, BN / CL))
        return cudaErrorNotSupported;
    static const bool one_sm = [] {
        const char *e = getenv("GIVENS_TC_1SM");
        return e && atoi(e) != 0;
    }();
    Args a{M, N, K, kchunk, out, ldo, zstride, accumulate};
    const int mt = (M + BM - 1) / BM;  // M tiles, padded to whole clusters (a padding CTA loads zeros, stores nothing)
    if (one_sm) {
        static bool attr = [] {
            return cudaFuncSetAttribute(k_gemm3_1sm<AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)SMEM_BYTES) == cudaSuccess;
        }();
        if (!attr) return cudaErrorInvalidConfiguration;
        dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((mt + CL - 1) / CL * CL), (unsigned)((K + kchunk - 1) / kchunk));
        k_gemm3_1sm<AMN, BMN><<<grid, NTHREADS, SMEM_BYTES, st>>>(ma, mb, a);
        return cudaGetLastError();
    }
    static bool attr2 = [] {
        return cudaFuncSetAttribute(k_gemm3<AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM2) ==
               cudaSuccess;
    }();
    if (!attr2) return cudaErrorInvalidConfiguration;
    dim3 grid((unsigned)(2 * ((N + BN2 - 1) / BN2)), (unsigned)((mt + 1) / 2), (unsigned)((K + kchunk - 1) / kchunk));
    k_gemm3<AMN, BMN><<<grid, NTHREADS, SMEM2, st>>>(ma, mb, a);
    return cudaGetLastError();
}

inline cudaError_t gemm3(const Operand &A, const Operand &B, int M, int N, int K, int kchunk, float *out, int64_t ldo,
                         int64_t zstride, cudaStream_t st, int accumulate = 0) {
    if (A.mn && B.mn) return gemm3_launch<true, true>(A, B, M, N, K, kchunk, out, ldo, zstride, accumulate, st);
    if (A.mn) return gemm3_launch<true, false>(A, B, M, N, K, kchunk, out, ldo, zstride, accumulate, st);
    if (B.mn) return gemm3_launch<false, true>(A, B, M, N, K, kchunk, out, ldo, zstride, accumulate, st);
    return gemm3_launch<false, false>(A, B, M, N, K, kchunk, out, ldo, zstride, accumulate, st);
}

// Operand shifted by k0 along K (for sequential K chunks)
inline Operand koff(const Operand &o, int64_t k0) { return Operand{o.mn ? o.p + k0 * o.ld : o.p + k0, o.ld, o.mn}; }

}  // namespace tcg
