// givens.cu -- sm_100a kernels and the C ABI (include/givens.h) for the data-parallel hot path
// of arXiv 2106.00003: circle-method schedule, block-parallel Givens forward on an n x m batch
// (or I to build U), and the replay backward with a deterministic dtheta reduction.
//
// Kernels (DESIGN.md §4 lists the roofline and algorithmic bytes of each):
//   k_flip / k_sigma / k_coef  per-call coefficient precompute (fp64 trig, pi-reduction, sign
//                              bookkeeping) into the ring kernels' lane-chunked table layout;
//   k_ring<W,L,MODE>           the hot path: one CTA owns a column slab, every block b_r runs
//                              on-chip from registers, coefficients stream in by TMA bulk copies;
//   k_generic<MODE>            any-n fallback (pairs derived lazily per block);
//   k_dtheta_reduce            stage 2 of the dtheta reduction (fixed CTA order, no atomics);
//   k_trace / k_trace_generic  index trace for the bit-exact schedule test.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <type_traits>
#include <utility>
#include <mutex>
#include <string>

#include "../../include/givens.h"
#include "ring.cuh"

#define GIVENS_VERSION "0.1.0"

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess) return fail(GIVENS_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

// ------------------------------------------------------------------ schedule (closed form)
// Circle method (Fig. 1): s_r[0] = 0, s_r[p] = 1 + ((p-1-r) mod (n_eff-1));
// block b_{r+1} pairs positions k and n_eff-1-k. Odd n: bye index n sits at
// position r (r >= 1) or n_eff-1 (r = 0), i.e. in slot 0 at r = 0 and min(r, n_eff-1-r) else.
__host__ __device__ __forceinline__ int seq_at(int r, int p, int ne) {
    int R = ne - 1;
    if (p == 0) return 0;
    int v = (p - 1 - r) % R;
    if (v < 0) v += R;
    return 1 + v;
}
__host__ __device__ __forceinline__ int bye_slot(int r, int ne) {
    if (r == 0) return 0;
    return r < ne - 1 - r ? r : ne - 1 - r;
}
// flat angle index of (block r, slot k) in block-major order skipping byes; -1 for the bye.
__host__ __device__ __forceinline__ int64_t flat_of(int r, int k, int n, int ne) {
    int S = ne / 2;
    if (n == ne) return (int64_t)r * S + k;
    int kb = bye_slot(r, ne);
    if (k == kb) return -1;
    return (int64_t)r * (S - 1) + k - (k > kb ? 1 : 0);
}
// position of row i in s_r
__host__ __device__ __forceinline__ int pos_of(int i, int r, int ne) {
    if (i == 0) return 0;
    int R = ne - 1;
    return 1 + ((i - 1 + r) % R);
}

// ------------------------------------------------------------------ configuration
struct Cfg {
    int ne, S, R, W, L, fast;  // fast: register ring kernel (else generic)
    int rowbytes;              // bytes per table row (S float2, padded to 16)
};

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

Cfg make_cfg(int n) {
    Cfg c;
    c.ne = n + (n & 1);
    c.S = c.ne / 2;
    c.R = c.ne - 1;
    c.fast = 0;
    c.W = c.S;
    c.L = 1;
    if (is_pow2(c.S) && c.S >= 4 && c.S <= 32) {
        c.fast = 1; c.W = c.S; c.L = 1;
    } else if (is_pow2(c.S) && c.S >= 64 && c.S <= 512) {
        c.fast = 1; c.W = 16; c.L = c.S / 16;
    } else if (c.S == 1024) {
        c.fast = 1; c.W = 32; c.L = 32;
    }
    c.rowbytes = ((c.S * 8) + 15) / 16 * 16;  // == S*8 for every ring configuration
    return c;
}

constexpr int kNW = 8;           // warps per CTA of the ring kernel
constexpr int kThreads = kNW * 32;

enum Mode { M_FWD = 0, M_BUILDU = 1, M_TRANS = 2, M_BWD = 3 };

__host__ __device__ constexpr int kcols(int W, int mode) {
    // columns per thread: two packed fp32 columns per FFMA2 where registers allow
    return (mode == M_BWD) ? (W >= 32 ? 1 : 2) : (W >= 32 ? 2 : 4);
}

int dev_sms() {
    static std::mutex mu;
    static int cache[64] = {0};
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return 148;
    std::lock_guard<std::mutex> g(mu);
    if (!cache[d]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = 148;
        cache[d] = v;
    }
    return cache[d];
}

int64_t cols_per_slab(const Cfg &c, int mode) {
    if (!c.fast) return 32;
    int Lc = 32 / c.L;
    return (int64_t)kNW * Lc * kcols(c.W, mode);
}

int64_t grid_for(const Cfg &c, int mode, int64_t m) {
    int64_t slabs = (m + cols_per_slab(c, mode) - 1) / cols_per_slab(c, mode);
    int64_t per_sm = c.fast ? 1 : 8;
    int64_t g = std::min<int64_t>(slabs, (int64_t)dev_sms() * per_sm);
    return std::max<int64_t>(g, 1);
}

struct WsLayout {
    size_t coef, amap, flip, sig, sfin, partial, scratch, total;
};

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

WsLayout ws_layout(const Cfg &c, int op, int64_t m) {
    WsLayout L;
    size_t off = 0;
    L.coef = off; off = al256(off + (size_t)(2 * c.S + 1) * c.rowbytes);
    L.amap = off; off = al256(off + (size_t)(2 * c.S + 1) * c.S * 4);
    L.flip = off; off = al256(off + (size_t)c.R * c.S);
    L.sig = off; off = al256(off + (size_t)c.R * c.ne);
    L.sfin = off; off = al256(off + (size_t)c.ne);
    L.partial = off;
    if (op == GIVENS_OP_BACKWARD) {
        int64_t g = grid_for(c, M_BWD, m);
        off = al256(off + (size_t)g * 2 * c.S * c.S * 4);
    }
    L.scratch = off;
    if (!c.fast) {
        int mode = op == GIVENS_OP_BACKWARD ? M_BWD : M_FWD;
        int64_t g = grid_for(c, mode, m);
        off = al256(off + (size_t)g * 32 * c.ne * (op == GIVENS_OP_BACKWARD ? 2 : 1) * 4);
    }
    L.total = off;
    return L;
}

}  // namespace

namespace gk {

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

// ------------------------------------------------------------------ precompute kernels
// (1) flip bit per (block, slot): |theta| > pi/2 => R(theta) = -R(theta -/+ pi).
__global__ void k_flip(int n, int ne, const float *__restrict__ theta, const uint8_t *__restrict__ mask,
                       uint8_t *__restrict__ flip) {
    int S = ne / 2, R = ne - 1;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)R * S) return;
    int r = (int)(idx / S), k = (int)(idx % S);
    int64_t f = flat_of(r, k, n, ne);
    uint8_t fl = 0;
    if (f >= 0 && (!mask || mask[f])) fl = fabs((double)theta[f]) > 1.5707963267948966 ? 1 : 0;
    flip[idx] = fl;
}

// (2) per row: parity of flips among the blocks applied before block r in forward order
// (forward applies b_R first), i.e. blocks r' > r. sig[r][row], sfin[row].
__global__ void k_sigma(int ne, const uint8_t *__restrict__ flip, uint8_t *__restrict__ sig,
                        uint8_t *__restrict__ sfin) {
    int S = ne / 2, R = ne - 1;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne) return;
    uint8_t par = 0;
    for (int r = R - 1; r >= 0; r--) {
        sig[(int64_t)r * ne + i] = par;
        int p = pos_of(i, r, ne);
        int k = p < ne - 1 - p ? p : ne - 1 - p;
        par ^= flip[(int64_t)r * S + k];
    }
    sfin[i] = par;
}

__device__ __forceinline__ int coef_pos(int k, int W, int L) {
    // float2 index of slot k inside a table row: lane t = k / W owns it; slots 2p, 2p+1 of a lane
    // form one float4 at float4-index p*L + t (conflict-free LDS.128 across the lanes).
    int t = k / W, q = k % W;
    return ((q >> 1) * L + t) * 2 + (q & 1);
}

// (3) table rows: rho = 0 pad, rho = r+1 block b_{r+1}, rho = 2S pad. Each entry (tq, sq) =
// sgn * (tan(phi/2), sin(phi)) with phi the pi-reduced angle and sgn = sigma_top * sigma_bottom *
// orientation (top row < bottom row); amap[rho][k] = flat | neg<<30 | masked<<29, or -1.
__global__ void k_coef(int n, int ne, int W, int L, int rowbytes, const float *__restrict__ theta,
                       const uint8_t *__restrict__ mask, const uint8_t *__restrict__ flip,
                       const uint8_t *__restrict__ sig, uint8_t *__restrict__ coef, int32_t *__restrict__ amap) {
    int S = ne / 2, R = ne - 1;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)(R + 2) * S) return;
    int rho = (int)(idx / S), k = (int)(idx % S);
    float2 *row = reinterpret_cast<float2 *>(coef + (int64_t)rho * rowbytes);
    int pos = coef_pos(k, W, L);
    if (rho == 0 || rho == R + 1) {
        row[pos] = make_float2(0.f, 0.f);
        amap[(int64_t)rho * S + k] = -1;
        return;
    }
    int r = rho - 1;
    int a = seq_at(r, k, ne), b = seq_at(r, ne - 1 - k, ne);
    int64_t f = flat_of(r, k, n, ne);
    bool active = f >= 0 && (!mask || mask[f]);
    double th = active ? (double)theta[f] : 0.0;
    double phi = th;
    if (fabs(th) > 1.5707963267948966) phi = th - copysign(3.141592653589793, th);
    int neg = (sig[(int64_t)r * ne + a] ^ sig[(int64_t)r * ne + b]) ^ (a > b ? 1 : 0);
    double tq = tan(0.5 * phi), sq = sin(phi);
    if (neg) { tq = -tq; sq = -sq; }
    row[pos] = make_float2((float)tq, (float)sq);
    int32_t code = -1;
    if (f >= 0) code = (int32_t)f | (neg ? (1 << 30) : 0) | (active ? 0 : (1 << 29));
    amap[(int64_t)rho * S + k] = code;
}

// ------------------------------------------------------------------ stage-2 dtheta reduction
// dtheta[flat] = sgn * sum_{cta = 0..G-1} partial[cta][rho][k] in fixed CTA order (PAPER.md:768-781
// "d <- A 1", made deterministic: no atomics). Masked angles get exactly 0.
__global__ void k_dtheta_reduce(int S, int W, int L, int G, const float *__restrict__ partial,
                                const int32_t *__restrict__ amap, float *__restrict__ dtheta) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int rows = 2 * S;
    if (idx >= (int64_t)rows * S) return;
    int32_t code = amap[idx];
    if (code < 0) return;
    int64_t f = code & 0x1FFFFFFF;
    if (code & (1 << 29)) {
        dtheta[f] = 0.f;
        return;
    }
    int rho = (int)(idx / S), k = (int)(idx % S);
    // partial rows are stored in the ring kernel's chunk order: chunk (q/4)*L + t holds slots
    // t*W + 4*(q/4) + 0..3 (natural order when L = 1, W = S)
    int t = k / W, q = k % W;
    int pos = (((q >> 2) * L + t) << 2) + (q & 3);
    float s = 0.f;
    const float *p = partial + (int64_t)rho * S + pos;
    int64_t stride = (int64_t)rows * S;
    for (int c = 0; c < G; c++) s += p[(int64_t)c * stride];
    dtheta[f] = (code & (1 << 30)) ? -s : s;
}

// ------------------------------------------------------------------ the register-ring kernel
struct RingArgs {
    int n, ne;
    int64_t m;
    const float *X;   // FWD/TRANS: input; BWD: Y
    int64_t ldx;
    const float *dY;  // BWD only
    int64_t lddy;
    float *Y;         // FWD/BUILDU/TRANS: output; BWD: dX (nullable)
    int64_t ldy;
    const uint8_t *coef;
    const uint8_t *sfin;
    float *partial;   // BWD: [grid][2S][S] in chunk order (see chunk_pos)
    int64_t nslabs;
    int vec_ok;       // 1 if all row starts are 16-byte aligned for K-wide vector access
};

template <int K>
struct ColIO;
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

// Compile-time geometry of one ring configuration (W slots per lane, L lanes per column group).
template <int W, int L, int MODE>
struct RingGeom {
    static constexpr int S = W * L;                 // slots = n_eff / 2
    static constexpr int STEPS = 2 * S;             // pad + the R = 2S-1 blocks
    static constexpr int LC = 32 / L;               // column groups per warp
    static constexpr int K = kcols(W, MODE);        // columns per thread
    // table rows per TMA stage: a power of two dividing W/2 with a stage of at most 16 KB
    static constexpr int SPS = (W / 2 * S * 8 <= 16384) ? W / 2
                             : (W / 4 * S * 8 <= 16384) ? W / 4
                             : (W / 8 * S * 8 <= 16384) ? W / 8 : 1;
    static constexpr int ROWB = S * 8;              // bytes per table row
    static constexpr int STAGEB = SPS * ROWB;
    static constexpr bool GRAD = (MODE == M_BWD);
    // stages in flight: 64 KB of table buffers next to the backward's dtheta ring, 96 KB otherwise
    static constexpr int NSTAGE_ = (GRAD ? 65536 : 98304) / STAGEB;
    static constexpr int NSTAGE = NSTAGE_ > 8 ? 8 : (NSTAGE_ < 2 ? 2 : NSTAGE_);
    // backward dtheta sums: per-warp ring of NG groups of RG steps, reduced one group later
    static constexpr int RG = (S >= 1024) ? 2 : 4;  // steps per reduction group (divides W)
    static constexpr int NG = 2;                    // groups in flight
    static constexpr int D = RG * NG;               // ring depth in steps
    static constexpr int NCH = S / 4;               // float4 chunks of a step's per-slot sums
    static constexpr int OUTCH = (NCH + kNW - 1) / kNW;  // chunks reduced per warp (max)
    static constexpr size_t OFF_STAGE = 256;
    static constexpr size_t OFF_RED = OFF_STAGE + (size_t)NSTAGE * STAGEB;
    static constexpr size_t OFF_OUT = OFF_RED + (GRAD ? (size_t)kNW * D * NCH * 16 : 0);
    static constexpr size_t SMEM_ = OFF_OUT + (GRAD ? (size_t)kNW * D * OUTCH * 16 : 0);
    static constexpr size_t SMEM = SMEM_;
};

// Hot-path kernel. One CTA of kNW warps owns a slab of C = kNW * LC * K columns; every column
// lives in the registers of L lanes (ring.cuh). All 2S steps (pad + the n_eff-1 blocks) run
// on-chip; the coefficient table streams through shared memory in TMA bulk stages; the
// backward's per-slot column sums go to a per-warp shared-memory ring in groups of RG steps; a
// group is reduced across the warps one group later (each warp owns a chunk range) and leaves
// the SM as TMA bulk reduce-adds into this CTA's private partial rows (fixed order, no
// atomics => deterministic).
template <int W, int L, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_ring(const RingArgs a) {
    using G = RingGeom<W, L, MODE>;
    using IO = ColIO<G::K>;
    using V = typename IO::V;
    constexpr int KP = IO::KP;
    constexpr int K = G::K;
    constexpr int S = G::S, STEPS = G::STEPS, LC = G::LC, SPS = G::SPS, NSTAGE = G::NSTAGE;
    constexpr int RG = G::RG, NG = G::NG, D = G::D, NCH = G::NCH, OUTCH = G::OUTCH;
    constexpr bool UP = (MODE == M_TRANS || MODE == M_BWD);  // walk b_1 -> b_R (inverse rotations)
    constexpr bool GRAD = G::GRAD;
    static_assert(W % SPS == 0 && W % RG == 0 && W % 4 == 0, "geometry");

    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint32_t *released = reinterpret_cast<uint32_t *>(full + NSTAGE);  // per-buffer warp release counts
    uint64_t *rfull = full + NSTAGE + (NSTAGE + 1) / 2;
    uint64_t *rempty = rfull + NG;
    uint8_t *stagebuf = smem + G::OFF_STAGE;
    float4 *red = reinterpret_cast<float4 *>(smem + G::OFF_RED);   // [kNW][D][NCH]
    float4 *outb = reinterpret_cast<float4 *>(smem + G::OFF_OUT);  // [kNW][NG][RG][OUTCH]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / L, t = lane % L;
    const bool first = (t == 0), last = (t == L - 1);
    const int ne = a.ne, n = a.n;
    const int64_t C = (int64_t)kNW * LC * K;
    const int my_slabs = (int)((a.nslabs - blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int total_stages = my_slabs * (STEPS / SPS);
    const int total_steps = my_slabs * STEPS;
    // chunk range of the per-step sums this warp reduces
    const int ch0 = (warp * NCH) / kNW, ch1 = ((warp + 1) * NCH) / kNW;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; i++) {
            mbar_init(&full[i], 1);
            released[i] = 0;
        }
        for (int i = 0; i < NG; i++) {
            mbar_init(&rfull[i], kNW);
            mbar_init(&rempty[i], kNW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    __syncthreads();
    if constexpr (GRAD) {
        // pre-arm: every ring group starts out "empty" (phase 0 completes here), so the first
        // use of each group waits on parity 0 without a special case
        if (lane == 0)
            for (int i = 0; i < NG; i++) mbar_arrive(&rempty[i]);
    }

    // table rows of slab-local stage j: forward reads rho = 2S - u (descending), backward rho = u
    auto stage_src = [&](int gst) -> const uint8_t * {
        int j = gst % (STEPS / SPS);
        int rho0 = UP ? j * SPS : (STEPS - (j + 1) * SPS + 1);
        return a.coef + (int64_t)rho0 * G::ROWB;
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE && s < total_stages; s++) {
            mbar_expect_tx(&full[s], G::STAGEB);
            bulk_g2s(stagebuf + (size_t)s * G::STAGEB, stage_src(s), G::STAGEB, &full[s]);
        }
    }

    // dtheta stage 1: reduce ring group gg (steps gg*RG .. gg*RG+RG-1 of this CTA) over the kNW
    // warps for this warp's chunk range and push it to this CTA's partial rows.
    auto reduce_group = [&](int gg) {
        const int bi = gg % NG;
        mbar_wait(&rfull[bi], (uint32_t)((gg / NG) & 1));
        if (lane == 0) bulk_wait_read<NG - 1>();  // the bulk ops that last read outb[bi] are done
        __syncwarp();
        const int nch = ch1 - ch0;
        float4 *ob = outb + ((size_t)warp * NG + bi) * RG * OUTCH;
        for (int it = lane; it < RG * nch; it += 32) {
            const int r = it / nch, c = it - r * nch;
            const float4 *src = red + (size_t)(bi * RG + r) * NCH + ch0 + c;
            float2 lo = make_float2(src[0].x, src[0].y), hi = make_float2(src[0].z, src[0].w);
#pragma unroll
            for (int w = 1; w < kNW; w++) {
                const float4 v = src[(size_t)w * D * NCH];
                lo = __fadd2_rn(lo, make_float2(v.x, v.y));
                hi = __fadd2_rn(hi, make_float2(v.z, v.w));
            }
            ob[r * OUTCH + c] = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&rempty[bi]);
            if (nch > 0) {
                fence_proxy_async_smem();
                for (int r = 0; r < RG; r++) {
                    const int gs = gg * RG + r;
                    const int rho = gs % STEPS;
                    float *dst = a.partial + ((int64_t)blockIdx.x * STEPS + rho) * S + ch0 * 4;
                    if (gs < STEPS) bulk_s2g_store(dst, ob + r * OUTCH, (uint32_t)nch * 16);
                    else bulk_s2g_reduce_add(dst, ob + r * OUTCH, (uint32_t)nch * 16);
                }
                bulk_commit();
                // successive slabs add into the same partial rows: keep them ordered
                if ((gg * RG + RG) % STEPS == 0) bulk_wait_all();
            }
        }
        __syncwarp();
    };

    int gst = 0;    // coefficient stages consumed by this CTA
    int grp = 0;    // dtheta ring groups completed by this CTA
    V ZT[KP][W], ZB[KP][W];
    V DT[GRAD ? KP : 1][GRAD ? W : 1], DB[GRAD ? KP : 1][GRAD ? W : 1];

    for (int64_t slab = blockIdx.x; slab < a.nslabs; slab += gridDim.x) {
        const int64_t col0 = slab * C + (int64_t)(warp * LC + g) * K;
        // ---------------- load the slab into the start layout (s_0 forward, s_{R-1} backward)
#pragma unroll
        for (int q = 0; q < W; q++) {
            const int k = t * W + q;
            const int pt = k, pb = ne - 1 - k;
            int rt, rb;
            if (UP) { rt = row_sRm1(pt, ne); rb = row_sRm1(pb, ne); }
            else    { rt = row_s0(pt);       rb = row_s0(pb); }
            V vt[KP], vb[KP];
            if constexpr (MODE == M_BUILDU) {
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
                const bool nt = rt < n && a.sfin[rt], nb = rb < n && a.sfin[rb];
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
                const bool nt = rt < n && a.sfin[rt], nb = rb < n && a.sfin[rb];
#pragma unroll
                for (int p = 0; p < KP; p++) {
                    DT[p][q] = vneg_if(vt[p], nt);
                    DB[p][q] = vneg_if(vb[p], nb);
                }
            }
        }

        // ---------------- all 2S steps, W steps per unrolled body (register renaming of the ring)
#pragma unroll 1
        for (int body = 0; body < STEPS / W; body++) {
            unroll<W>([&](auto ic) {
                constexpr int uu = decltype(ic)::value;
                constexpr int su = uu % SPS;
                if constexpr (su == 0) {
                    mbar_wait(&full[gst % NSTAGE], (uint32_t)((gst / NSTAGE) & 1));
                    __syncwarp();
                }
                const float4 *row4 = reinterpret_cast<const float4 *>(
                    stagebuf + (gst % NSTAGE) * G::STAGEB + (UP ? su : (SPS - 1 - su)) * G::ROWB);
                constexpr int r = uu % RG;
                int bi = 0;
                float4 *ring_dst = nullptr;
                if constexpr (GRAD) {
                    bi = grp % NG;
                    if constexpr (r == 0) {  // the ring group we are about to fill is free
                        mbar_wait(&rempty[bi], (uint32_t)((grp / NG) & 1));
                        __syncwarp();
                    }
                    ring_dst = red + ((size_t)warp * D + bi * RG + r) * NCH;
                }
                float acc[GRAD ? (LC > 1 ? W : 4) : 1];
#pragma unroll
                for (int pp = 0; pp < W / 2; pp++) {
                    const float4 cf = row4[pp * L + t];
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int q = 2 * pp + h;
                        const float tq = h ? cf.z : cf.x, sq = h ? cf.w : cf.y;
                        if constexpr (GRAD) {
                            // dtheta contribution before this block's inverse rotation:
                            // dz_bottom * z_top - dz_top * z_bottom (Q_e structure)
                            float c = 0.f;
#pragma unroll
                            for (int p = 0; p < KP; p++) c = cross_acc(c, DB[p][q], ZT[p][q], DT[p][q], ZB[p][q]);
                            acc[LC > 1 ? q : (q & 3)] = c;
                        }
#pragma unroll
                        for (int p = 0; p < KP; p++) {
                            if (UP) {
                                rot_inv(ZT[p][q], ZB[p][q], tq, sq);
                                if constexpr (GRAD) rot_inv(DT[p][q], DB[p][q], tq, sq);
                            } else {
                                rot_fwd(ZT[p][q], ZB[p][q], tq, sq);
                            }
                        }
                    }
                    if constexpr (GRAD && LC == 1) {
                        // one lane per column group: the per-slot sums go straight to the ring
                        if (pp & 1) ring_dst[(pp >> 1) * L + t] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                    }
                }
                if constexpr (GRAD) {
                    if constexpr (LC > 1) {
#pragma unroll
                        for (int q = 0; q < W; q++) {
#pragma unroll
                            for (int o = L; o < 32; o <<= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
                        }
                        if (g == 0) {
#pragma unroll
                            for (int q4 = 0; q4 < W / 4; q4++)
                                ring_dst[q4 * L + t] =
                                    make_float4(acc[4 * q4], acc[4 * q4 + 1], acc[4 * q4 + 2], acc[4 * q4 + 3]);
                        }
                    }
                    if constexpr (r == RG - 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&rfull[bi]);
                        // warps w and w+4 share an SMSP: the low half reduces the previous group
                        // here, the high half RG/2 steps later, so one of them keeps the FMA pipe busy
                        if (warp < 4 && grp >= 1) reduce_group(grp - 1);
                        grp++;
                    }
                    if constexpr (r == RG / 2 - 1) {
                        if (warp >= 4 && grp >= 1) reduce_group(grp - 1);
                    }
                }
                // ring shift to the next block's layout (Fig. 1)
#pragma unroll
                for (int p = 0; p < KP; p++) {
                    if (UP) {
                        shift_up<W>(ZT[p], ZB[p], first, last, L);
                        if constexpr (GRAD) shift_up<W>(DT[p], DB[p], first, last, L);
                    } else {
                        shift_down<W>(ZT[p], ZB[p], first, last, L);
                    }
                }
                if constexpr (su == SPS - 1) {
                    // release the stage buffer; the LAST warp to release it refills it with the
                    // stage NSTAGE ahead (no warp ever waits to act as the producer)
                    __syncwarp();
                    if (lane == 0) {
                        const int b = gst % NSTAGE;
                        __threadfence_block();  // this warp's reads of buffer b happen-before the release
                        if (atomicAdd(&released[b], 1u) == kNW - 1) {
                            __threadfence_block();
                            released[b] = 0;
                            const int nxt = gst + NSTAGE;
                            if (nxt < total_stages) {
                                fence_proxy_async_smem();
                                mbar_expect_tx(&full[b], G::STAGEB);
                                bulk_g2s(stagebuf + (size_t)b * G::STAGEB, stage_src(nxt), G::STAGEB, &full[b]);
                            }
                        }
                    }
                    __syncwarp();
                    gst++;
                }
            });
        }

        // ---------------- store from the end layout (s_{R-1} forward, s_0 backward)
        if (MODE == M_BWD && a.Y == nullptr) continue;
#pragma unroll
        for (int q = 0; q < W; q++) {
            const int k = t * W + q;
            const int pt = k, pb = ne - 1 - k;
            int rt, rb;
            if (UP) { rt = row_s0(pt); rb = row_s0(pb); }
            else    { rt = row_sRm1(pt, ne); rb = row_sRm1(pb, ne); }
            V vt[KP], vb[KP];
#pragma unroll
            for (int p = 0; p < KP; p++) {
                if constexpr (GRAD) { vt[p] = DT[p][q]; vb[p] = DB[p][q]; }
                else { vt[p] = ZT[p][q]; vb[p] = ZB[p][q]; }
            }
            if (!UP) {
                const bool nt = rt < n && a.sfin[rt], nb = rb < n && a.sfin[rb];
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
    (void)total_steps;
}

// ------------------------------------------------------------------ generic any-n kernel
// One warp per CTA, one column per thread; the column lives in a global scratch vector in row
// order and the pair rows of every (block, slot) are derived lazily from the closed form
// (the paper's own prototype strategy). dtheta: warp butterfly per slot, then
// lane 0 accumulates the CTA partial in fixed order.
struct GenArgs {
    int n, ne, S, rowbytes;
    int64_t m;
    const float *X; int64_t ldx;
    const float *dY; int64_t lddy;
    float *Y; int64_t ldy;
    const uint8_t *coef;
    const uint8_t *sfin;
    float *partial;
    float *scratch;  // [ne][G*32] (Z) and, for BWD, another [ne][G*32] (D)
    int64_t nslabs;
};

template <int MODE>
__global__ void __launch_bounds__(32) k_generic(const GenArgs a) {
    constexpr bool UP = (MODE == M_TRANS || MODE == M_BWD);
    constexpr bool GRAD = (MODE == M_BWD);
    const int lane = threadIdx.x;
    const int ne = a.ne, n = a.n, S = a.S, R = ne - 1;
    const int steps = 2 * S;
    const int64_t stride = (int64_t)gridDim.x * 32;
    float *Z = a.scratch + (int64_t)blockIdx.x * 32 + lane;
    float *D = Z + (int64_t)ne * stride;
    int64_t slab_i = 0;
    for (int64_t slab = blockIdx.x; slab < a.nslabs; slab += gridDim.x, slab_i++) {
        const int64_t col = slab * 32 + lane;
        const bool live = col < a.m;
        for (int i = 0; i < ne; i++) {
            float v = 0.f, d = 0.f;
            if (i < n && live) {
                if (MODE == M_BUILDU) v = (col == i) ? 1.f : 0.f;
                else v = a.X[(int64_t)i * a.ldx + col];
                if (GRAD) d = a.dY[(int64_t)i * a.lddy + col];
                if (UP && a.sfin[i]) { v = -v; d = -d; }
            }
            Z[(int64_t)i * stride] = v;
            if (GRAD) D[(int64_t)i * stride] = d;
        }
        for (int u = 0; u < steps; u++) {
            int rho = UP ? u : (steps - u);
            if (rho == 0 || rho == steps) continue;  // pad rows are the identity
            int r = rho - 1;
            const float2 *row = reinterpret_cast<const float2 *>(a.coef + (int64_t)rho * a.rowbytes);
            for (int k = 0; k < S; k++) {
                int rt = seq_at(r, k, ne), rbm = seq_at(r, ne - 1 - k, ne);
                float2 cf = row[k];  // generic tables use L = 1, W = S: natural slot order
                float x = Z[(int64_t)rt * stride], y = Z[(int64_t)rbm * stride];
                if (GRAD) {
                    float dx = D[(int64_t)rt * stride], dy = D[(int64_t)rbm * stride];
                    float v = live ? (dy * x - dx * y) : 0.f;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (lane == 0) {
                        float *pp = a.partial + ((int64_t)blockIdx.x * steps + rho) * S + k;
                        *pp = (slab_i > 0) ? (*pp + v) : v;
                    }
                    rot_inv(dx, dy, cf.x, cf.y);
                    D[(int64_t)rt * stride] = dx;
                    D[(int64_t)rbm * stride] = dy;
                }
                if (UP) rot_inv(x, y, cf.x, cf.y);
                else rot_fwd(x, y, cf.x, cf.y);
                Z[(int64_t)rt * stride] = x;
                Z[(int64_t)rbm * stride] = y;
            }
        }
        if (live && !(GRAD && a.Y == nullptr)) {
            for (int i = 0; i < n; i++) {
                float v = GRAD ? D[(int64_t)i * stride] : Z[(int64_t)i * stride];
                if (!UP && a.sfin[i]) v = -v;
                a.Y[(int64_t)i * a.ldy + col] = v;
            }
        }
    }
    if (GRAD && slab_i == 0) {
        // CTA without slabs: zero its partial so stage 2 can sum every CTA
        for (int64_t i = lane; i < (int64_t)steps * S; i += 32) a.partial[(int64_t)blockIdx.x * steps * S + i] = 0.f;
    }
}

// ------------------------------------------------------------------ index trace
template <int W>
__global__ void k_trace(int ne, int L, int up, int32_t *out) {
    const int lane = threadIdx.x;
    const int t = lane % L;          // every group runs (shuffles need the full warp)
    const bool writer = lane < L;    // group 0 records
    const bool first = t == 0, last = t == L - 1;
    const int S = ne / 2, R = ne - 1;
    float T[W], B[W];
    for (int q = 0; q < W; q++) {
        int k = t * W + q;
        T[q] = (float)(up ? row_sRm1(k, ne) : row_s0(k));
        B[q] = (float)(up ? row_sRm1(ne - 1 - k, ne) : row_s0(ne - 1 - k));
    }
    for (int body = 0; body < 2 * S / W; body++) {
#pragma unroll
        for (int uu = 0; uu < W; uu++) {
            int u = body * W + uu;
            if (u >= 1 && writer) {
                int r = up ? (u - 1) : (R - u);
                for (int q = 0; q < W; q++) {
                    int k = t * W + q;
                    int a = (int)T[q], b = (int)B[q];
                    out[((int64_t)r * S + k) * 2] = a < b ? a : b;
                    out[((int64_t)r * S + k) * 2 + 1] = a < b ? b : a;
                }
            }
            if (up) shift_up<W>(T, B, first, last, L);
            else shift_down<W>(T, B, first, last, L);
        }
    }
}

__global__ void k_trace_generic(int ne, int32_t *out) {
    const int S = ne / 2, R = ne - 1;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)R * S) return;
    int r = (int)(idx / S), k = (int)(idx % S);
    int a = seq_at(r, k, ne), b = seq_at(r, ne - 1 - k, ne);
    out[idx * 2] = a < b ? a : b;
    out[idx * 2 + 1] = a < b ? b : a;
}

}  // namespace gk

// ====================================================================== host side
namespace {

using namespace gk;

template <int W, int L, int MODE>
int launch_ring_wl(RingArgs &ra, int64_t grid, cudaStream_t st) {
    constexpr size_t smem = RingGeom<W, L, MODE>::SMEM;
    static_assert(smem <= 227 * 1024, "shared memory budget");
    auto kfn = k_ring<W, L, MODE>;
    CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kfn<<<(unsigned)grid, kThreads, smem, st>>>(ra);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

template <int MODE>
int launch_ring(const Cfg &c, RingArgs &ra, int64_t grid, cudaStream_t st) {
    if (c.L == 1) {
        switch (c.W) {
            case 4: return launch_ring_wl<4, 1, MODE>(ra, grid, st);
            case 8: return launch_ring_wl<8, 1, MODE>(ra, grid, st);
            case 16: return launch_ring_wl<16, 1, MODE>(ra, grid, st);
            case 32: return launch_ring_wl<32, 1, MODE>(ra, grid, st);
        }
    } else if (c.W == 16) {
        switch (c.L) {
            case 4: return launch_ring_wl<16, 4, MODE>(ra, grid, st);
            case 8: return launch_ring_wl<16, 8, MODE>(ra, grid, st);
            case 16: return launch_ring_wl<16, 16, MODE>(ra, grid, st);
            case 32: return launch_ring_wl<16, 32, MODE>(ra, grid, st);
        }
    } else if (c.W == 32 && c.L == 32) {
        return launch_ring_wl<32, 32, MODE>(ra, grid, st);
    }
    return fail(GIVENS_EUNSUPPORTED, "no ring kernel for W=%d L=%d", c.W, c.L);
}

int run_precompute(const Cfg &c, int n, const float *theta, const uint8_t *mask, uint8_t *ws, const WsLayout &L,
                   cudaStream_t st) {
    int64_t RS = (int64_t)c.R * c.S;
    k_flip<<<(unsigned)((RS + 255) / 256), 256, 0, st>>>(n, c.ne, theta, mask, ws + L.flip);
    CUDA_TRY(cudaGetLastError());
    k_sigma<<<(unsigned)((c.ne + 127) / 128), 128, 0, st>>>(c.ne, ws + L.flip, ws + L.sig, ws + L.sfin);
    CUDA_TRY(cudaGetLastError());
    int64_t tot = (int64_t)(c.R + 2) * c.S;
    int W = c.fast ? c.W : c.S, Lq = c.fast ? c.L : 1;
    k_coef<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, c.ne, W, Lq, c.rowbytes, theta, mask, ws + L.flip,
                                                          ws + L.sig, ws + L.coef,
                                                          reinterpret_cast<int32_t *>(ws + L.amap));
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int check_common(int32_t n, int64_t m, const void *ws, size_t ws_bytes, int op) {
    if (n < 2) return fail(GIVENS_EINVAL, "n must be >= 2 (got %d)", n);
    if (n > 32768) return fail(GIVENS_EINVAL, "n must be <= 32768 (got %d)", n);
    if (m < 0) return fail(GIVENS_EINVAL, "m must be >= 0");
    if (!ws) return fail(GIVENS_EINVAL, "workspace is NULL");
    if (((uintptr_t)ws) % 256) return fail(GIVENS_EINVAL, "workspace must be 256-byte aligned");
    size_t need = givens_workspace_bytes(op, n, m);
    if (ws_bytes < need) return fail(GIVENS_EINVAL, "workspace too small: %zu < %zu", ws_bytes, need);
    return 0;
}

int vec_ok_for(int K, std::initializer_list<std::pair<const void *, int64_t>> mats) {
    for (auto &p : mats) {
        if (!p.first) continue;
        if (((uintptr_t)p.first) % (4 * K)) return 0;
        if (p.second % K) return 0;
    }
    return 1;
}

int run_apply_mode(int mode, int32_t n, int64_t m, const float *X, int64_t ldx, const float *dY, int64_t lddy,
                   float *Y, int64_t ldy, uint8_t *ws, const WsLayout &L, const Cfg &c, cudaStream_t st) {
    if (m == 0) return 0;
    int64_t grid = grid_for(c, mode, m);
    if (c.fast) {
        RingArgs ra;
        ra.n = n; ra.ne = c.ne;
        ra.m = m; ra.X = X; ra.ldx = ldx; ra.dY = dY; ra.lddy = lddy; ra.Y = Y; ra.ldy = ldy;
        ra.coef = ws + L.coef; ra.sfin = ws + L.sfin;
        ra.partial = reinterpret_cast<float *>(ws + L.partial);
        ra.nslabs = (m + cols_per_slab(c, mode) - 1) / cols_per_slab(c, mode);
        int K = kcols(c.W, mode);
        ra.vec_ok = vec_ok_for(K, {{X, ldx}, {dY, lddy}, {Y, ldy}});
        switch (mode) {
            case M_FWD: return launch_ring<M_FWD>(c, ra, grid, st);
            case M_BUILDU: return launch_ring<M_BUILDU>(c, ra, grid, st);
            case M_TRANS: return launch_ring<M_TRANS>(c, ra, grid, st);
            case M_BWD: return launch_ring<M_BWD>(c, ra, grid, st);
        }
        return fail(GIVENS_EINVAL, "bad mode");
    }
    GenArgs ga;
    ga.n = n; ga.ne = c.ne; ga.S = c.S; ga.rowbytes = c.rowbytes; ga.m = m;
    ga.X = X; ga.ldx = ldx; ga.dY = dY; ga.lddy = lddy; ga.Y = Y; ga.ldy = ldy;
    ga.coef = ws + L.coef; ga.sfin = ws + L.sfin;
    ga.partial = reinterpret_cast<float *>(ws + L.partial);
    ga.scratch = reinterpret_cast<float *>(ws + L.scratch);
    ga.nslabs = (m + 31) / 32;
    switch (mode) {
        case M_FWD: k_generic<M_FWD><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_BUILDU: k_generic<M_BUILDU><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_TRANS: k_generic<M_TRANS><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_BWD: k_generic<M_BWD><<<(unsigned)grid, 32, 0, st>>>(ga); break;
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char *givens_last_error(void) { return g_err.c_str(); }
const char *givens_version(void) { return GIVENS_VERSION; }

int64_t givens_num_angles(int32_t n) { return n < 2 ? -1 : (int64_t)n * (n - 1) / 2; }

int givens_supported(int32_t n) { return (n >= 2 && n <= 32768) ? 1 : 0; }

int givens_schedule(int32_t n, int32_t *pairs_host, int64_t *flat_host) {
    if (n < 2) return fail(GIVENS_EINVAL, "n must be >= 2 (got %d)", n);
    int ne = n + (n & 1), S = ne / 2, R = ne - 1;
    for (int r = 0; r < R; r++)
        for (int k = 0; k < S; k++) {
            int a = seq_at(r, k, ne), b = seq_at(r, ne - 1 - k, ne);
            int64_t q = (int64_t)r * S + k;
            if (pairs_host) {
                pairs_host[2 * q] = a < b ? a : b;
                pairs_host[2 * q + 1] = a < b ? b : a;
            }
            if (flat_host) flat_host[q] = flat_of(r, k, n, ne);
        }
    return 0;
}

int givens_mask_from_dims(int32_t n, const uint8_t *excl, uint8_t *mask) {
    if (n < 2 || !excl || !mask) return fail(GIVENS_EINVAL, "bad arguments");
    int ne = n + (n & 1), S = ne / 2, R = ne - 1;
    for (int r = 0; r < R; r++)
        for (int k = 0; k < S; k++) {
            int64_t f = flat_of(r, k, n, ne);
            if (f < 0) continue;
            int a = seq_at(r, k, ne), b = seq_at(r, ne - 1 - k, ne);
            mask[f] = (excl[a] && excl[b]) ? 0 : 1;
        }
    return 0;
}

size_t givens_workspace_bytes(int op, int32_t n, int64_t m) {
    if (n < 2 || n > 32768 || m < 0 || op < 0 || op > 2) return 0;
    Cfg c = make_cfg(n);
    return ws_layout(c, op, op == GIVENS_OP_BUILD_U ? n : m).total;
}

int givens_apply(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx,
                 float *Y, int64_t ldy, int transpose, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_common(n, m, ws, ws_bytes, GIVENS_OP_APPLY);
    if (rc) return rc;
    if (!theta || !X || !Y) return fail(GIVENS_EINVAL, "theta, X and Y must be non-NULL");
    if (ldx < m || ldy < m) return fail(GIVENS_EINVAL, "leading dimension smaller than m");
    if (X == Y && ldx != ldy) return fail(GIVENS_EINVAL, "in-place apply needs ldx == ldy");
    Cfg c = make_cfg(n);
    WsLayout L = ws_layout(c, GIVENS_OP_APPLY, m);
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = (uint8_t *)ws;
    if ((rc = run_precompute(c, n, theta, mask, w, L, st))) return rc;
    return run_apply_mode(transpose ? M_TRANS : M_FWD, n, m, X, ldx, nullptr, 0, Y, ldy, w, L, c, st);
}

int givens_build_U(int32_t n, const float *theta, const uint8_t *mask, float *U, int64_t ldu, void *ws,
                   size_t ws_bytes, void *stream) {
    int rc = check_common(n, n, ws, ws_bytes, GIVENS_OP_BUILD_U);
    if (rc) return rc;
    if (!theta || !U) return fail(GIVENS_EINVAL, "theta and U must be non-NULL");
    if (ldu < n) return fail(GIVENS_EINVAL, "ldu < n");
    Cfg c = make_cfg(n);
    WsLayout L = ws_layout(c, GIVENS_OP_BUILD_U, n);
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = (uint8_t *)ws;
    if ((rc = run_precompute(c, n, theta, mask, w, L, st))) return rc;
    return run_apply_mode(M_BUILDU, n, n, nullptr, 0, nullptr, 0, U, ldu, w, L, c, st);
}

int givens_backward(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *Y, int64_t ldy,
                    const float *dY, int64_t lddy, float *dX, int64_t lddx, float *dtheta, int flags, void *ws,
                    size_t ws_bytes, void *stream) {
    int rc = check_common(n, m, ws, ws_bytes, GIVENS_OP_BACKWARD);
    if (rc) return rc;
    if (!theta || !Y || !dY || !dtheta) return fail(GIVENS_EINVAL, "theta, Y, dY and dtheta must be non-NULL");
    if (ldy < m || lddy < m || (dX && lddx < m)) return fail(GIVENS_EINVAL, "leading dimension smaller than m");
    if (dX && dX == dY && lddx != lddy) return fail(GIVENS_EINVAL, "in-place dX needs lddx == lddy");
    Cfg c = make_cfg(n);
    WsLayout L = ws_layout(c, GIVENS_OP_BACKWARD, m);
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *w = (uint8_t *)ws;
    if (flags & GIVENS_FLAG_RECOMPUTE) {
        if ((rc = run_precompute(c, n, theta, mask, w, L, st))) return rc;
    }
    int64_t N = givens_num_angles(n);
    if (m == 0) {
        CUDA_TRY(cudaMemsetAsync(dtheta, 0, (size_t)N * 4, st));
        return 0;
    }
    if ((rc = run_apply_mode(M_BWD, n, m, Y, ldy, dY, lddy, dX, lddx, w, L, c, st))) return rc;
    int64_t G = grid_for(c, M_BWD, m);
    int64_t tot = (int64_t)2 * c.S * c.S;
    k_dtheta_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        c.S, c.fast ? c.W : c.S, c.fast ? c.L : 1, (int)G, reinterpret_cast<const float *>(w + L.partial), reinterpret_cast<const int32_t *>(w + L.amap),
        dtheta);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int givens_index_trace(int32_t n, int direction, int32_t *out_dev, void *stream) {
    if (n < 2 || n > 32768 || !out_dev) return fail(GIVENS_EINVAL, "bad arguments");
    Cfg c = make_cfg(n);
    cudaStream_t st = (cudaStream_t)stream;
    int up = direction ? 1 : 0;
    if (c.fast) {
        switch (c.W) {
            case 4: k_trace<4><<<1, 32, 0, st>>>(c.ne, c.L, up, out_dev); break;
            case 8: k_trace<8><<<1, 32, 0, st>>>(c.ne, c.L, up, out_dev); break;
            case 16: k_trace<16><<<1, 32, 0, st>>>(c.ne, c.L, up, out_dev); break;
            case 32: k_trace<32><<<1, 32, 0, st>>>(c.ne, c.L, up, out_dev); break;
        }
    } else {
        int64_t RS = (int64_t)c.R * c.S;
        k_trace_generic<<<(unsigned)((RS + 255) / 256), 256, 0, st>>>(c.ne, out_dev);
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // extern "C"
