// ring_inst.cu -- one (W, L) configuration of the register-ring kernel, all four modes.
// Compiled once per configuration with -DRING_W=.. -DRING_L=.. (parallel build, see build.py);
// exports gk::ring_launch_<W>_<L>(mode, args, grid, stream).
#include "common.cuh"

#ifndef RING_W
#error "RING_W / RING_L must be defined"
#endif

#define GK_CAT2(a, b, c) a##b##_##c
#define GK_CAT(a, b, c) GK_CAT2(a, b, c)

namespace gk {

template <int W, int L, int MODE>
static cudaError_t launch_wlm(const RingArgs &ra, int64_t grid, cudaStream_t st) {
    // at least 120 KB: one CTA per SM (the grids are sized for that, grid_for), also when the CTAs of a
    // programmatic dependent launch become resident while the predecessor still runs (measured: without
    // the floor the 64 KB narrow C2 forward CTAs doubled up on SMs, 41 -> 57 us)
    constexpr size_t smem = RingGeom<W, L, MODE>::SMEM > 120 * 1024 ? RingGeom<W, L, MODE>::SMEM : 120 * 1024;
    static_assert(smem <= 227 * 1024, "shared memory budget");
    auto kfn = k_ring<W, L, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // programmatic dependent launch (see pdl_wait in common.cuh): the CTAs may start while the
    // precompute / the previous ring kernel drains
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(RingGeom<W, L, MODE>::NW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    // (narrow launches only: the latency regime gains -- n = 256 build 30.8 -> 26.7 us, C2 142 -> 136 us
    // -- while the four-warp-column U-build measured 6.98 -> 7.17 ms with it)
    cfg.numAttrs = (GK_PDL && (MODE & M_NARROW)) ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kfn, ra);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// configurations that also serve n with idle lanes (S = W * La, La < L; see make_cfg)
#define GK_IDLE_CAPABLE ((RING_W == 16 || RING_W == 8) && (RING_L == 32 || RING_L == 64 || RING_L == 128))

cudaError_t GK_CAT(ring_launch_, RING_W, RING_L)(int mode, const RingArgs &ra, int64_t grid, cudaStream_t st) {
    if (ra.La != RING_L) mode |= M_IDLE;
    switch (mode) {
#if RING_L <= 32  // narrow (4-warp, <= 2 columns per thread) real-valued variants for small batches;
                  // single-warp column groups only (see launch_mode in givens.cu)
        case M_FWD | M_NARROW: return launch_wlm<RING_W, RING_L, M_FWD | M_NARROW>(ra, grid, st);
        case M_BUILDU | M_NARROW: return launch_wlm<RING_W, RING_L, M_BUILDU | M_NARROW>(ra, grid, st);
        case M_TRANS | M_NARROW: return launch_wlm<RING_W, RING_L, M_TRANS | M_NARROW>(ra, grid, st);
        case M_BWD | M_NARROW: return launch_wlm<RING_W, RING_L, M_BWD | M_NARROW>(ra, grid, st);
#if RING_W == 8  // 4 columns per thread (M_NK4)
        case M_FWD | M_NARROW | M_NK4: return launch_wlm<RING_W, RING_L, M_FWD | M_NARROW | M_NK4>(ra, grid, st);
        case M_BUILDU | M_NARROW | M_NK4: return launch_wlm<RING_W, RING_L, M_BUILDU | M_NARROW | M_NK4>(ra, grid, st);
        case M_TRANS | M_NARROW | M_NK4: return launch_wlm<RING_W, RING_L, M_TRANS | M_NARROW | M_NK4>(ra, grid, st);
        case M_BWD | M_NARROW | M_NK4: return launch_wlm<RING_W, RING_L, M_BWD | M_NARROW | M_NK4>(ra, grid, st);
#endif
#if GK_IDLE_CAPABLE
        case M_FWD | M_NARROW | M_IDLE: return launch_wlm<RING_W, RING_L, M_FWD | M_NARROW | M_IDLE>(ra, grid, st);
        case M_BUILDU | M_NARROW | M_IDLE:
            return launch_wlm<RING_W, RING_L, M_BUILDU | M_NARROW | M_IDLE>(ra, grid, st);
        case M_TRANS | M_NARROW | M_IDLE: return launch_wlm<RING_W, RING_L, M_TRANS | M_NARROW | M_IDLE>(ra, grid, st);
        case M_BWD | M_NARROW | M_IDLE: return launch_wlm<RING_W, RING_L, M_BWD | M_NARROW | M_IDLE>(ra, grid, st);
#endif
#endif
#if GK_IDLE_CAPABLE
        case M_FWD | M_IDLE: return launch_wlm<RING_W, RING_L, M_FWD | M_IDLE>(ra, grid, st);
        case M_BUILDU | M_IDLE: return launch_wlm<RING_W, RING_L, M_BUILDU | M_IDLE>(ra, grid, st);
        case M_TRANS | M_IDLE: return launch_wlm<RING_W, RING_L, M_TRANS | M_IDLE>(ra, grid, st);
        case M_BWD | M_IDLE: return launch_wlm<RING_W, RING_L, M_BWD | M_IDLE>(ra, grid, st);
#if RING_W * RING_L <= 1024
        case M_FWD | M_UNI | M_IDLE: return launch_wlm<RING_W, RING_L, M_FWD | M_UNI | M_IDLE>(ra, grid, st);
        case M_BUILDU | M_UNI | M_IDLE: return launch_wlm<RING_W, RING_L, M_BUILDU | M_UNI | M_IDLE>(ra, grid, st);
        case M_TRANS | M_UNI | M_IDLE: return launch_wlm<RING_W, RING_L, M_TRANS | M_UNI | M_IDLE>(ra, grid, st);
        case M_BWD | M_UNI | M_IDLE: return launch_wlm<RING_W, RING_L, M_BWD | M_UNI | M_IDLE>(ra, grid, st);
#endif
#endif
#if RING_L == 1  // fast Givens: forward and U-build on one-lane columns
        case M_FWD | M_FG: return launch_wlm<RING_W, RING_L, M_FWD | M_FG>(ra, grid, st);
        case M_BUILDU | M_FG: return launch_wlm<RING_W, RING_L, M_BUILDU | M_FG>(ra, grid, st);
        case M_FWD | M_FG | M_NARROW: return launch_wlm<RING_W, RING_L, M_FWD | M_FG | M_NARROW>(ra, grid, st);
        case M_BUILDU | M_FG | M_NARROW: return launch_wlm<RING_W, RING_L, M_BUILDU | M_FG | M_NARROW>(ra, grid, st);
#endif
        case M_FWD: return launch_wlm<RING_W, RING_L, M_FWD>(ra, grid, st);
        case M_BUILDU: return launch_wlm<RING_W, RING_L, M_BUILDU>(ra, grid, st);
        case M_TRANS: return launch_wlm<RING_W, RING_L, M_TRANS>(ra, grid, st);
        case M_BWD: return launch_wlm<RING_W, RING_L, M_BWD>(ra, grid, st);
#if RING_W != 32 && RING_W * RING_L <= 1024  // unitary: two real columns (one complex) per thread; its
                                                // 32-byte-per-slot tables fit shared memory up to S = 1024
        case M_FWD | M_UNI: return launch_wlm<RING_W, RING_L, M_FWD | M_UNI>(ra, grid, st);
        case M_BUILDU | M_UNI: return launch_wlm<RING_W, RING_L, M_BUILDU | M_UNI>(ra, grid, st);
        case M_TRANS | M_UNI: return launch_wlm<RING_W, RING_L, M_TRANS | M_UNI>(ra, grid, st);
        case M_BWD | M_UNI: return launch_wlm<RING_W, RING_L, M_BWD | M_UNI>(ra, grid, st);
#endif
    }
    return cudaErrorInvalidValue;
}

}  // namespace gk
