// givens.cu -- sm_100a kernels and the C ABI (include/givens.h) for the data-parallel hot path
// of arXiv 2106.00003: circle-method schedule, block-parallel Givens forward on an n x m batch
// (or I to build U), and the replay backward with a deterministic dtheta reduction.
//
// Kernels (DESIGN.md §4 lists the roofline and algorithmic bytes of each):
//   k_sigma_bits / k_coef        per-call coefficient precompute (fp64 trig, pi-reduction, sign
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
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <type_traits>
#include <utility>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/givens.h"
#include "common.cuh"

#define GIVENS_VERSION "0.1.0"

namespace gk {
#define GK_DECL(W, L) cudaError_t ring_launch_##W##_##L(int mode, const RingArgs &ra, int64_t grid, cudaStream_t st);
GK_DECL(4, 1) GK_DECL(8, 1) GK_DECL(16, 1) GK_DECL(32, 1) GK_DECL(16, 4) GK_DECL(16, 8) GK_DECL(16, 16)
GK_DECL(16, 32) GK_DECL(8, 64) GK_DECL(16, 64) GK_DECL(32, 32) GK_DECL(16, 128) GK_DECL(8, 32) GK_DECL(8, 128)
GK_DECL(8, 16)
#undef GK_DECL
}  // namespace gk

using namespace gk;

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

// ------------------------------------------------------------------ configuration
struct Cfg {
    int ne, S, R, W, L, fast;  // fast: register ring kernel (else generic); L = instantiated lanes
    int nk4 = 0;               // narrow launches use M_NK4 (4 columns per thread; W = 8 rings)
    int La;                    // active lanes per column group (S = W * La; La <= L)
    int rowbytes;              // bytes per table row (S float2, padded to 16)
};

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

int dev_sms();
int64_t cols_per_slab(const Cfg &c, int mode);

// m: the batch the configuration will serve (real columns; -1 = unknown). The real ring at S = 128 /
// 256 (n = 256 / 512) runs W = 8 slots per lane instead of 16 whenever the W = 16 launch would be
// narrow: with 2 columns per thread (twice the slabs) when the narrow W = 16 launch would leave more
// than half the SMs without a slab -- the U-build and its gradient at those n (measured: n = 256
// gradient 104 -> 72 us, n = 512 201 -> 140 us) -- else with 4 (M_NK4: the same slabs, a smaller
// body; C2 backward 130 -> 101 us). Forward and backward of one batch see the same m, hence the same
// configuration (the reuse tag checks it).
Cfg make_cfg(int n, int64_t m = -1);
Cfg make_cfg(int n, int64_t m) {
    Cfg c;
    c.ne = n + (n & 1);
    c.S = c.ne / 2;
    c.R = c.ne - 1;
    c.fast = 0;
    c.W = c.S;
    c.L = 1;
    // ring geometry S = W * L (see GK_RING_CONFIGS); GIVENS_RING_W overrides W where an
    // alternative configuration exists (tuning experiments)
    static const int wpref = [] {
        const char *e = getenv("GIVENS_RING_W");
        return e ? atoi(e) : 0;
    }();
    if (is_pow2(c.S) && c.S >= 4 && c.S <= 32) {
        c.fast = 1; c.W = c.S; c.L = 1;
    } else if (is_pow2(c.S) && c.S >= 64 && c.S <= 512) {
        c.fast = 1; c.W = 16; c.L = c.S / 16;
        if (wpref == 8 && c.S >= 128) { c.W = 8; c.L = c.S / 8; }
    } else if (c.S == 1024) {
        c.fast = 1; c.W = 16; c.L = 64;
        if (wpref == 32) { c.W = 32; c.L = 32; }
    } else if (c.S == 2048) {
        c.fast = 1; c.W = 16; c.L = 128;
    }
    c.La = c.L;
    if (!c.fast) {
        // any other S: the ring with idle lanes at the end of the last warp of each column group
        // (S = W * La, La active lanes out of L = 32, 64 or 128 instantiated ones)
        for (int w : {16, 8}) {
            if (c.S % w == 0 && c.S / w >= 2 && c.S / w <= 128) {
                c.fast = 1; c.W = w; c.La = c.S / w;
                c.L = c.La <= 32 ? 32 : (c.La <= 64 ? 64 : 128);
                break;
            }
        }
    }
    c.rowbytes = ((c.S * 8) + 15) / 16 * 16;  // == S*8 for every ring configuration
    if (m > 0 && wpref == 0 && c.fast && c.W == 16 && (c.S == 128 || c.S == 256)) {
        Cfg w8 = c;
        w8.W = 8; w8.L = w8.La = c.S / 8;
        const int64_t narrow16 = (m + cols_per_slab(c, M_FWD | M_NARROW) - 1) / cols_per_slab(c, M_FWD | M_NARROW);
        const int64_t normal16 = (m + cols_per_slab(c, M_BWD) - 1) / cols_per_slab(c, M_BWD);
        if (2 * narrow16 <= dev_sms()) return w8;
        if (normal16 < dev_sms()) {  // the W = 16 launches would be narrow (launch_mode)
            w8.nk4 = 1;
            return w8;
        }
    }
    return c;
}

// unitary variant: the ring kernels carry 16-24 more table bytes per slot, which rules out W = 32
// (registers) and W * L > 1024 (shared memory); those n take an idle-lane ring if one fits, else
// the generic kernel
Cfg make_cfg_u(int n) {
    Cfg c = make_cfg(n);
    if (c.fast && (c.W == 32 || c.W * c.L > 1024)) {
        c.fast = 0; c.W = c.S; c.L = 1; c.La = 1;
        for (int w : {16, 8}) {
            if (c.S % w == 0 && c.S / w >= 2 && c.S / w <= 128) {
                int La = c.S / w, L = La <= 32 ? 32 : (La <= 64 ? 64 : 128);
                if (w * L > 1024) continue;
                c.fast = 1; c.W = w; c.La = La; c.L = L;
                break;
            }
        }
    }
    return c;
}

Cfg cfg_for_op(int n, int op, int64_t m) { return op >= 3 ? make_cfg_u(n) : make_cfg(n, m); }

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
    int LW = c.L < 32 ? c.L : 32, H = c.L / LW, LC = 32 / LW;
    return (int64_t)ring_warps(mode) * LC / H * kcols(c.W, mode);
}

// the launch mode for m columns: the narrow variant when the normal width leaves SMs without a
// slab (real ring kernels with single-warp column groups only: with H > 1 warps per group the
// per-step exchange barrier would be amortised over half the columns -- measured 2x slower)
int launch_mode(const Cfg &c, int mode, int64_t m) {
    if (!c.fast || (mode & M_UNI) || (mode & M_NARROW)) return mode;
    const int H = c.L < 32 ? 1 : c.L / 32;
    if (H > 1) return mode;
    const int64_t slabs = (m + cols_per_slab(c, mode) - 1) / cols_per_slab(c, mode);
    const int nm = mode | M_NARROW | (c.nk4 ? M_NK4 : 0);
    const int64_t slabs_n = (m + cols_per_slab(c, nm) - 1) / cols_per_slab(c, nm);
    if (!(slabs < dev_sms() && slabs_n > slabs)) return mode;
    return mode | M_NARROW | (c.nk4 ? M_NK4 : 0);
}

// the generic backward keeps a private [vals][2S][S] fp32 partial per CTA; its grid is capped so
// that the partials stay within this budget (n = 8192 would otherwise need 1184 x 134 MB)
constexpr size_t kGenericPartialBudget = (size_t)4 << 30;

int64_t grid_for(const Cfg &c, int mode0, int64_t m) {
    const int mode = launch_mode(c, mode0, m);
    int64_t slabs = (m + cols_per_slab(c, mode) - 1) / cols_per_slab(c, mode);
    int64_t per_sm = c.fast ? 1 : 8;
    int64_t g = std::min<int64_t>(slabs, (int64_t)dev_sms() * per_sm);
    if (!c.fast && (mode & 3) == M_BWD) {
        const size_t per_cta = (size_t)2 * c.S * c.S * 4 * ((mode & M_UNI) ? 2 : 1);
        g = std::min<int64_t>(g, (int64_t)std::max<size_t>(1, kGenericPartialBudget / per_cta));
    }
    return std::max<int64_t>(g, 1);
}

// ---- coefficient-table tags. A backward with GIVENS_FLAG_REUSE_TABLES consumes the tables a
// forward call left in the workspace; the host remembers, per workspace address, what the last
// precompute into it was built from, and a reuse whose (device, n, configuration, theta, phi,
// mask, perm, reflect_col) differ is refused with GIVENS_EINVAL instead of silently reading stale
// tables. (Pointers, not contents: a caller that rewrites theta in place between the forward and
// a reusing backward must not pass the flag.)
struct TableTag {
    int dev, n, W, L, uni, refl;
    const void *theta, *phi, *mask, *perm;
    bool operator==(const TableTag &o) const {
        return dev == o.dev && n == o.n && W == o.W && L == o.L && uni == o.uni && refl == o.refl &&
               theta == o.theta && phi == o.phi && mask == o.mask && perm == o.perm;
    }
};
std::mutex g_tag_mu;
std::unordered_map<const void *, TableTag> g_tags;

TableTag make_tag(const Cfg &c, int n, const float *theta, const float *phi, const uint8_t *mask,
                  const int32_t *perm, int refl) {
    int d = -1;
    cudaGetDevice(&d);
    return TableTag{d, n, c.W, c.L, phi ? 1 : 0, refl, theta, phi, mask, perm};
}
void tag_tables(const void *ws, const TableTag &t) {
    std::lock_guard<std::mutex> g(g_tag_mu);
    g_tags[ws] = t;
}
void untag_tables(const void *ws) {
    std::lock_guard<std::mutex> g(g_tag_mu);
    g_tags.erase(ws);
}
int check_tables(const void *ws, const TableTag &want) {
    if (!ws) return fail(GIVENS_EINVAL, "GIVENS_FLAG_REUSE_TABLES needs the forward's workspace (ws is NULL)");
    std::lock_guard<std::mutex> g(g_tag_mu);
    auto it = g_tags.find(ws);
    if (it == g_tags.end())
        return fail(GIVENS_EINVAL, "GIVENS_FLAG_REUSE_TABLES: no forward call filled this workspace");
    if (!(it->second == want))
        return fail(GIVENS_EINVAL, "GIVENS_FLAG_REUSE_TABLES: the workspace tables were built for a different "
                                   "(n, theta, phi, mask, perm, reflect_col) or device");
    return 0;
}

// ---- ws == NULL: a stream-ordered workspace for this call (cudaMallocAsync / cudaFreeAsync on the
// call's stream, from the device's default memory pool)
struct AutoWs {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    int get(void *&ws, size_t &bytes, size_t need, cudaStream_t s);
    ~AutoWs() {
        if (p) {
            untag_tables(p);
            cudaFreeAsync(p, st);
        }
    }
};

struct WsLayout {
    size_t coef, coef_ph, coef_pf, coef_pt, coef_ab, amap, sig, sfin, lay, fgm, sfg, partial, scratch, total;
};

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

// ops 0..2: GIVENS_OP_*; 3..5: the unitary variants (m counts complex columns)
WsLayout ws_layout(const Cfg &c, int op, int64_t m) {
    const bool uni = op >= 3;
    const int base = op % 3;
    const int64_t mr = uni ? 2 * m : m;  // real columns
    WsLayout L;
    size_t off = 0;
    const size_t rows = (size_t)(2 * c.S + 1);
    L.coef = off; off = al256(off + rows * c.rowbytes);
    L.coef_ph = off; if (uni) off = al256(off + rows * c.S * 16);
    L.coef_pf = off; if (uni) off = al256(off + rows * c.S * 32);  // forward pairs (p, q, -q, p)
    L.coef_pt = off; if (uni) off = al256(off + rows * c.S * 32);  // adjoint pairs (p, -q, q, p)
    L.coef_ab = off; if (uni) off = al256(off + rows * c.S * 8);
    L.amap = off; off = al256(off + rows * c.S * 4);
    L.sig = off; off = al256(off + (size_t)c.ne * ((c.R + 31) / 32) * 4);  // sigma bits [label][block / 32]
    L.sfin = off; off = al256(off + (size_t)c.ne);
    L.lay = off; off = al256(off + (size_t)(c.ne + 2) * 4);
    L.fgm = off; off = al256(off + rows * 4);            // fast Givens: factoring bits per table row
    L.sfg = off; off = al256(off + (size_t)c.ne * 4);    // fast Givens: final scale per label
    L.partial = off;
    if (base == GIVENS_OP_BACKWARD) {
        int64_t g = grid_for(c, M_BWD | (uni ? M_UNI : 0), mr);
        size_t per_step = (size_t)c.S * 4 * (uni ? 2 : 1);  // generic kernel: natural order, [vals][2S][S]
        if (c.fast) {
            const RedGeom rg = red_geom(c.W, c.L, uni ? 2 : 1, ring_warps(launch_mode(c, M_BWD | (uni ? M_UNI : 0), mr)));
            per_step = (size_t)rg.NW * rg.OUTCH * 16;  // >= S floats (padded when chunks don't split evenly)
        }
        off = al256(off + (size_t)g * 2 * c.S * per_step);
    }
    L.scratch = off;
    if (!c.fast) {
        int mode = base == GIVENS_OP_BACKWARD ? M_BWD : M_FWD;
        int64_t g = grid_for(c, mode, mr);
        off = al256(off + (size_t)g * 32 * c.ne * (base == GIVENS_OP_BACKWARD ? 2 : 1) * (uni ? 2 : 1) * 4);
    }
    L.total = off;
    return L;
}

}  // namespace

namespace gk {

// ------------------------------------------------------------------ precompute kernels
// (0) layout block (one CTA): row of each label under the start permutation perm (NULL =
// identity), the odd-n bye label, and the label of the reflected column.
__global__ void k_layout(int n, int ne, const int32_t *__restrict__ perm, int refl, int32_t *__restrict__ lay) {
    if (threadIdx.x == 0) {
        lay[ne] = ne - 1;  // identity: the bye is label n
        lay[ne + 1] = refl;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < ne; l += blockDim.x) {
        int row = perm ? perm[l] : l;
        lay[l] = row;
        if (perm && row == n && n != ne) lay[ne] = l;
        if (perm && refl >= 0 && row == refl) lay[ne + 1] = l;
    }
}

// The precompute kernels read the layout block only under a start permutation; without one (lay ==
// NULL) label l is row l, the odd-n bye is label n_eff - 1 and the reflected column's label is the
// column itself -- and k_layout is not launched at all.
__device__ __forceinline__ int lay_row(const int32_t *__restrict__ lay, int l) { return lay ? lay[l] : l; }
__device__ __forceinline__ int lay_bye(const int32_t *__restrict__ lay, int ne) { return lay ? lay[ne] : ne - 1; }
__device__ __forceinline__ int lay_refl(const int32_t *__restrict__ lay, int ne, int refl) {
    return lay ? lay[ne + 1] : refl;
}

// theta -> the angle phi in [-pi/2, pi/2] with R(theta) = (-1)^flip R(phi). theta is
// any real (theta in R^N): it is first reduced to [-pi, pi] by the exact fp64
// remainder modulo 2 pi (R is 2 pi-periodic), then flipped by pi when |.| > pi/2, so the shear
// coefficient tan(phi/2) stays in [-1, 1] for every theta. k_sigma_bits, k_coef and k_coef_u all use it,
// so the flip bits and the table agree.
__device__ __forceinline__ double reduce_angle(double th, int *flip) {
    double r = remainder(th, 6.283185307179586);
    const int fl = fabs(r) > 1.5707963267948966 ? 1 : 0;
    if (fl) r -= copysign(3.141592653589793, r);
    if (flip) *flip = fl;
    return r;
}

// (1)+(2) sign bookkeeping, one kernel. The flip bit of a rotation: |theta| > pi/2 => R(theta) =
// -R(theta -/+ pi); sigma of label i before block r (in forward order the blocks r' > r
// come first) is the parity of the flips of the rotations on i in those blocks. One
// CTA per label i: lane j of a warp computes the flip of block 32c + j (one angle load and one fp64
// reduction per thread) and a ballot makes it the bit word c; then thread c turns word c into
// sigw[i][c] (bit j = sigma of label i before block 32c + j): the in-word exclusive suffix parity by a
// shift-XOR scan, XOR the parity of all higher words (ballot + shared memory across warps). A
// reflection D (applied before every block) flips the parity of its label in every block and in sfin;
// the kernels then load and store without knowing about it. blockDim = 32 min(RW, 32),
// RW = ceil((n_eff - 1) / 32) words per label (<= 1024).
__global__ void __launch_bounds__(1024) k_sigma_bits(int n, int ne, const float *__restrict__ theta,
                                                     const uint8_t *__restrict__ mask, const int32_t *__restrict__ lay,
                                                     int refl, uint32_t *__restrict__ sigw, uint8_t *__restrict__ sfin) {
    __shared__ uint32_t words[1024];
    __shared__ uint32_t wpar[32];
    const int R = ne - 1, RW = (R + 31) / 32, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarp = blockDim.x >> 5;
    pdl_trigger();  // k_coef may start its trigonometry (it waits for these bits)
    const int i = blockIdx.x;
    const int bl = lay_bye(lay, ne);
    for (int c = warp; c < RW; c += nwarp) {
        const int r = 32 * c + lane;
        int fl = 0;
        if (r < R) {
            const int p = pos_of(i, r, ne);
            const int k = p < ne - 1 - p ? p : ne - 1 - p;
            const int64_t f = flat_of_bl(r, k, n, ne, bl);
            if (f >= 0 && (!mask || mask[f])) reduce_angle((double)theta[f], &fl);
        }
        const uint32_t fb = __ballot_sync(0xffffffffu, fl != 0);
        if (lane == 0) words[c] = fb;
    }
    __syncthreads();
    const uint32_t fb = tid < RW ? words[tid] : 0u;
    const uint32_t bal = __ballot_sync(0xffffffffu, (__popc(fb) & 1u) != 0);
    if (lane == 0) wpar[warp] = __popc(bal) & 1u;
    __syncthreads();
    uint32_t carry = __popc(bal & (lane == 31 ? 0u : (0xffffffffu << (lane + 1)))) & 1u;  // higher words, my warp
    uint32_t total = 0;
    for (int v = 0; v < nwarp; v++) {
        total ^= wpar[v];
        if (v > warp) carry ^= wpar[v];
    }
    if (tid >= RW) return;
    uint32_t x = fb;  // inclusive suffix parity within the word: bit j = XOR of bits j..31
    x ^= x >> 1;
    x ^= x >> 2;
    x ^= x >> 4;
    x ^= x >> 8;
    x ^= x >> 16;
    const uint32_t rf = (lay_refl(lay, ne, refl) == i) ? 1u : 0u;
    sigw[(int64_t)i * RW + tid] = (x >> 1) ^ ((carry ^ rf) ? 0xffffffffu : 0u);
    if (tid == 0) sfin[i] = (uint8_t)(total ^ rf);
}
__device__ __forceinline__ int sig_bit(const uint32_t *__restrict__ sigw, int RW, int lab, int r) {
    return (int)((sigw[(int64_t)lab * RW + (r >> 5)] >> (r & 31)) & 1u);
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
                       const uint8_t *__restrict__ mask, const uint32_t *__restrict__ sigw,
                       const int32_t *__restrict__ lay, uint8_t *__restrict__ coef, int32_t *__restrict__ amap) {
    int S = ne / 2, R = ne - 1;
    pdl_trigger();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = idx < (int64_t)(R + 2) * S;
    const int rho = (int)(idx / S), k = (int)(idx % S);
    const bool pad = rho == 0 || rho == R + 1;
    const int r = rho - 1;
    int a = 0, b = 0;
    int64_t f = -1;
    bool active = false;
    double tq = 0.0, sq = 0.0;
    if (live && !pad) {
        a = seq_at(r, k, ne);  // labels; rows lay[a], lay[b]
        b = seq_at(r, ne - 1 - k, ne);
        f = flat_of_bl(r, k, n, ne, lay_bye(lay, ne));
        active = f >= 0 && (!mask || mask[f]);
        const double phi = reduce_angle(active ? (double)theta[f] : 0.0, nullptr);
        tq = tan(0.5 * phi);
        sq = sin(phi);
    }
    // (launched dependent on k_sigma_bits: the trigonometry above overlaps it; the sign bits are its
    // output. Every thread waits, so this grid cannot complete before its predecessor.)
    pdl_wait();
    if (!live) return;
    float2 *row = reinterpret_cast<float2 *>(coef + (int64_t)rho * rowbytes);
    const int pos = coef_pos(k, W, L);
    if (pad) {
        row[pos] = make_float2(0.f, 0.f);
        amap[(int64_t)rho * S + k] = -1;
        return;
    }
    const int RW = (R + 31) / 32;
    int neg = (sig_bit(sigw, RW, a, r) ^ sig_bit(sigw, RW, b, r)) ^ (lay_row(lay, a) > lay_row(lay, b) ? 1 : 0);
    if (neg) { tq = -tq; sq = -sq; }
    row[pos] = make_float2((float)tq, (float)sq);
    int32_t code = -1;
    if (f >= 0) code = (int32_t)f | (neg ? (1 << 30) : 0) | (active ? 0 : (1 << 29));
    amap[(int64_t)rho * S + k] = code;
}

// (3u) unitary tables (Appendix A): G^e = R(theta) diag(e^{i phi}, 1) on (i, j) (Alg. 4,
// PAPER.md:1002-1005). In (top, bottom) ring coordinates the phase sits on whichever of the two
// holds row i: ph[rho][slot] = (p_t, q_t, p_b, q_b) with (p, q) = (cos phi, sin phi) there and
// (1, 0) on the other. ab[rho][slot] = (alpha, beta): the dphi weights, w = alpha z_t + beta z_b
// = cos(th_r) z_i + sigma_i sigma_j sin(th_r) z_j, th_r the pi-reduced angle.
__global__ void k_coef_u(int n, int ne, int W, int L, const float *__restrict__ theta, const float *__restrict__ phi,
                         const uint8_t *__restrict__ mask, const uint32_t *__restrict__ sigw,
                         const int32_t *__restrict__ lay, float4 *__restrict__ ph, float4 *__restrict__ pf,
                         float4 *__restrict__ pt, float2 *__restrict__ ab) {
    int S = ne / 2, R = ne - 1;
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)(R + 2) * S) return;
    int rho = (int)(idx / S), k = (int)(idx % S);
    int t = k / W, q = k % W;
    float4 *phr = ph + (int64_t)rho * S;
    float2 *abr = ab + (int64_t)rho * S;
    int pos_ph = q * L + t;          // one float4 per slot
    int pos_ab = coef_pos(k, W, L);  // one float2 per slot, pairs of slots per float4
    if (rho == 0 || rho == R + 1) {
        phr[pos_ph] = make_float4(1.f, 0.f, 1.f, 0.f);
        abr[pos_ab] = make_float2(0.f, 0.f);
        const int64_t pp0 = (int64_t)rho * 2 * S + (2 * q) * L + t, pp1 = pp0 + L;
        pf[pp0] = pf[pp1] = pt[pp0] = pt[pp1] = make_float4(1.f, 0.f, 0.f, 1.f);
        return;
    }
    int r = rho - 1;
    int a = seq_at(r, k, ne), b = seq_at(r, ne - 1 - k, ne);
    int64_t f = flat_of_bl(r, k, n, ne, lay_bye(lay, ne));
    bool active = f >= 0 && (!mask || mask[f]);
    double th = active ? (double)theta[f] : 0.0, pv = active ? (double)phi[f] : 0.0;
    const double thr = reduce_angle(th, nullptr);
    float pc = (float)cos(pv), ps = (float)sin(pv);
    bool top_is_i = lay_row(lay, a) < lay_row(lay, b);
    phr[pos_ph] = top_is_i ? make_float4(pc, ps, 1.f, 0.f) : make_float4(1.f, 0.f, pc, ps);
    {   // FFMA2-ready pairs per side, top then bottom: (p, q, -q, p) forward, (p, -q, q, p) adjoint
        const int64_t pp0 = (int64_t)rho * 2 * S + (2 * q) * L + t, pp1 = pp0 + L;
        const float4 one = make_float4(1.f, 0.f, 0.f, 1.f);
        const float4 f = make_float4(pc, ps, -ps, pc), c = make_float4(pc, -ps, ps, pc);
        pf[pp0] = top_is_i ? f : one;
        pf[pp1] = top_is_i ? one : f;
        pt[pp0] = top_is_i ? c : one;
        pt[pp1] = top_is_i ? one : c;
    }
    double cr = cos(thr), sr = sin(thr);
    if (sig_bit(sigw, (R + 31) / 32, a, r) ^ sig_bit(sigw, (R + 31) / 32, b, r)) sr = -sr;
    abr[pos_ab] = top_is_i ? make_float2((float)cr, (float)sr) : make_float2((float)sr, (float)cr);
}

// (3f) fast Givens tables (one-lane columns, S <= 32, identity layout). One CTA of S
// threads walks the blocks in the forward's order (b_R first), thread k owning slot
// k. The values are kept as x = d z with a per-label scale d (fp64 here, 1 at the start). In
// (top, bottom) coordinates the block rotates by psi = theta (top holds the smaller row i) or -theta;
// with c = cos psi, s = sin psi:
//   |c| >= |s|: top' = c (u - (s/c) v), bottom' = c (v + (s/c) u):  z_t' = z_t - a z_b, z_b' = z_b + b z_t,
//               a = (s/c) d_b / d_t, b = (s/c) d_t / d_b, d_t' = c d_t, d_b' = c d_b;
//   |s| >  |c|: top' = -s (v - (c/s) u), bottom' = s (u + (c/s) v):  z_t' = z_b - a z_t, z_b' = z_t + b z_b,
//               a = (c/s) d_t / d_b, b = (c/s) d_b / d_t, d_t' = -s d_b, d_b' = s d_t  (bit q of the row set).
// The table row holds (a, b) where the three-shear table holds (t, s); masked / bye slots are the
// identity (a = b = 0, scales unchanged). |a|, |b| <= 1 x the scale ratio; for n <= 64 the scales stay
// within 2^-32 .. 1, so no renormalisation is needed.
__global__ void k_fg_tables(int n, int ne, const float *__restrict__ theta, const uint8_t *__restrict__ mask,
                            uint8_t *__restrict__ coef, int rowbytes, uint32_t *__restrict__ fgm,
                            float *__restrict__ sfg) {
    __shared__ double d[64];
    __shared__ uint32_t bits;
    const int S = ne / 2, R = ne - 1, k = threadIdx.x;
    for (int l = k; l < ne; l += blockDim.x) d[l] = 1.0;
    if (k < S) {  // pad rows: identity
        reinterpret_cast<float2 *>(coef)[coef_pos(k, S, 1)] = make_float2(0.f, 0.f);
        reinterpret_cast<float2 *>(coef + (int64_t)(R + 1) * rowbytes)[coef_pos(k, S, 1)] = make_float2(0.f, 0.f);
    }
    if (k == 0) fgm[0] = fgm[R + 1] = 0u;
    __syncthreads();
    for (int r = R - 1; r >= 0; r--) {  // forward order: b_R first
        if (k == 0) bits = 0u;
        __syncthreads();
        if (k < S) {
            const int la = seq_at(r, k, ne), lb = seq_at(r, ne - 1 - k, ne);
            const int64_t f = flat_of(r, k, n, ne);
            float2 ab = make_float2(0.f, 0.f);
            if (f >= 0 && (!mask || mask[f])) {
                const double th = remainder((double)theta[f], 6.283185307179586);
                const double psi = la < lb ? th : -th;  // identity layout: label = row
                const double c = cos(psi), sn = sin(psi), dt = d[la], db = d[lb];
                if (fabs(c) >= fabs(sn)) {
                    const double q = sn / c;
                    ab = make_float2((float)(q * db / dt), (float)(q * dt / db));
                    d[la] = c * dt;
                    d[lb] = c * db;
                } else {
                    const double q = c / sn;
                    ab = make_float2((float)(q * dt / db), (float)(q * db / dt));
                    d[la] = -sn * db;
                    d[lb] = sn * dt;
                    atomicOr(&bits, 1u << k);
                }
            }
            reinterpret_cast<float2 *>(coef + (int64_t)(r + 1) * rowbytes)[coef_pos(k, S, 1)] = ab;
        }
        __syncthreads();
        if (k == 0) fgm[r + 1] = bits;
    }
    __syncthreads();
    for (int l = k; l < ne; l += blockDim.x) sfg[l] = (float)d[l];
}

// ------------------------------------------------------------------ stage-2 dtheta reduction
// dtheta[flat] = sgn * sum_{cta = 0..G-1} partial[cta][rho][k] in fixed CTA order (PAPER.md:768-781
// "d <- A 1", made deterministic: no atomics). Masked angles get exactly 0. One thread per table slot
// summing the G CTAs in order (measured against an eight-phase variant and a memory-order variant in
// round 2: this one was fastest at every size -- C3 100 vs 179 us, C4 1.33 vs 2.58 ms under ncu).
__global__ void k_dtheta_reduce(int S, int W, int L, int NW, int G, int ring, int vals, const float *__restrict__ partial,
                                const int32_t *__restrict__ amap, float *__restrict__ dtheta, float *__restrict__ dphi) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int rows = 2 * S;
    if (idx >= (int64_t)rows * S) return;
    int32_t code = amap[idx];
    if (code < 0) return;
    int64_t f = code & 0x1FFFFFFF;
    if (code & (1 << 29)) {
        dtheta[f] = 0.f;
        if (vals > 1) dphi[f] = 0.f;
        return;
    }
    int rho = (int)(idx / S), k = (int)(idx % S);
    for (int v = 0; v < vals; v++) {
        int64_t pos, stride;
        if (ring) {
            // ring kernel layout: per CTA, per group of RG steps, NW warp blocks of RG x OUTCH float4;
            // slot k (lane t = k / W of the group, slot q = k % W) is chunk ci = v*NCHW1 + (q/4)*LW + t%LW
            // of the warp slice t/LW (v = 0: dtheta, 1: dphi), reduced by the warp c*H + slice owning ci
            const RedGeom rg = red_geom(W, L, vals, NW);
            const int nchw1 = rg.NCHW / vals;
            int t = k / W, q = k % W, hs = t / rg.LW, tl = t % rg.LW;
            int ci = v * nchw1 + (q >> 2) * rg.LW + tl;
            int c = 0;
            while (c + 1 < rg.NSUM && ((c + 1) * rg.NCHW) / rg.NSUM <= ci) c++;
            int j = ci - (c * rg.NCHW) / rg.NSUM;
            int w = c * rg.H + hs;
            int64_t blk = ((int64_t)(rho / rg.RG) * rg.NW + w) * rg.RG * rg.OUTCH;
            pos = (blk + (rho % rg.RG) * rg.OUTCH + j) * 4 + (q & 3);
            stride = (int64_t)rows * rg.NW * rg.OUTCH * 4;
        } else {
            pos = ((int64_t)v * rows + rho) * S + k;  // generic kernel: natural order, [vals][rows][S]
            stride = (int64_t)vals * rows * S;
        }
        float s = 0.f;
        const float *p = partial + pos;
        for (int cc = 0; cc < G; cc++) s += p[(int64_t)cc * stride];
        if (v == 0) dtheta[f] = (code & (1 << 30)) ? -s : s;
        else dphi[f] = s;  // dphi carries no sign: sigma_i^2 = 1
    }
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
    const float4 *coef_ph;  // unitary: phases per slot, natural order
    const float2 *coef_ab;  // unitary backward: dphi weights per slot, natural order
    const uint8_t *sfin;
    const int32_t *lrow;  // row of each label (start permutation)
    float *partial;
    float *scratch;  // [ne][G*32] (Z) and, for BWD, another [ne][G*32] (D); float2 entries when unitary
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
        for (int i = 0; i < ne; i++) {  // i: label, row = lrow[i]
            float v = 0.f, d = 0.f;
            const int row = a.lrow ? a.lrow[i] : i;
            if (row < n && live) {
                if (MODE == M_BUILDU) v = (col == row) ? 1.f : 0.f;
                else v = a.X[(int64_t)row * a.ldx + col];
                if (GRAD) d = a.dY[(int64_t)row * a.lddy + col];
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
            for (int i = 0; i < ne; i++) {
                const int row = a.lrow ? a.lrow[i] : i;
                if (row >= n) continue;
                float v = GRAD ? D[(int64_t)i * stride] : Z[(int64_t)i * stride];
                if (!UP && a.sfin[i]) v = -v;
                a.Y[(int64_t)row * a.ldy + col] = v;
            }
        }
    }
    if (GRAD && slab_i == 0) {
        // CTA without slabs: zero its partial so stage 2 can sum every CTA
        for (int64_t i = lane; i < (int64_t)steps * S; i += 32) a.partial[(int64_t)blockIdx.x * steps * S + i] = 0.f;
    }
}

// Unitary variant of k_generic (Appendix A, Alg. 4): one complex column per thread, the same
// table conventions as the ring's unitary path (k_coef_u), dtheta and dphi partials per CTA as
// [2][2S][S] (dtheta, then dphi). a.m counts real columns (2 per complex column).
template <int BM>
__global__ void __launch_bounds__(32) k_generic_u(const GenArgs a) {
    constexpr bool UP = (BM == M_TRANS || BM == M_BWD);
    constexpr bool GRAD = (BM == M_BWD);
    const int lane = threadIdx.x;
    const int ne = a.ne, n = a.n, S = a.S;
    const int steps = 2 * S;
    const int64_t mc = a.m / 2;
    const int64_t stride = (int64_t)gridDim.x * 32;
    float2 *Z = reinterpret_cast<float2 *>(a.scratch) + (int64_t)blockIdx.x * 32 + lane;
    float2 *D = Z + (int64_t)ne * stride;
    int64_t slab_i = 0;
    for (int64_t slab = blockIdx.x; slab < a.nslabs; slab += gridDim.x, slab_i++) {
        const int64_t col = slab * 32 + lane;
        const bool live = col < mc;
        for (int i = 0; i < ne; i++) {  // i: label, row = lrow[i]
            float2 v = make_float2(0.f, 0.f), d = make_float2(0.f, 0.f);
            const int row = a.lrow ? a.lrow[i] : i;
            if (row < n && live) {
                if (BM == M_BUILDU) v.x = (col == row) ? 1.f : 0.f;
                else v = make_float2(a.X[(int64_t)row * a.ldx + 2 * col], a.X[(int64_t)row * a.ldx + 2 * col + 1]);
                if (GRAD)
                    d = make_float2(a.dY[(int64_t)row * a.lddy + 2 * col], a.dY[(int64_t)row * a.lddy + 2 * col + 1]);
                if (UP && a.sfin[i]) { v = neg_v(v); d = neg_v(d); }
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
                const float2 cf = row[k];
                const float4 ph = a.coef_ph[(int64_t)rho * S + k];  // (p_t, q_t, p_b, q_b)
                float2 x = Z[(int64_t)rt * stride], y = Z[(int64_t)rbm * stride];
                if (GRAD) {
                    float2 dx = D[(int64_t)rt * stride], dy = D[(int64_t)rbm * stride];
                    const float2 ab = a.coef_ab[(int64_t)rho * S + k];
                    // dtheta: Re(conj(dz_b) z_t - conj(dz_t) z_b); dphi: Re(i conj(v) w) with
                    // w = alpha z_t + beta z_b, v = alpha dz_t + beta dz_b
                    float vt = 0.f, vp = 0.f;
                    if (live) {
                        vt = dy.x * x.x + dy.y * x.y - dx.x * y.x - dx.y * y.y;
                        float2 w = make_float2(ab.x * x.x + ab.y * y.x, ab.x * x.y + ab.y * y.y);
                        float2 v = make_float2(ab.x * dx.x + ab.y * dy.x, ab.x * dx.y + ab.y * dy.y);
                        vp = v.y * w.x - v.x * w.y;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        vt += __shfl_xor_sync(0xffffffffu, vt, o);
                        vp += __shfl_xor_sync(0xffffffffu, vp, o);
                    }
                    if (lane == 0) {
                        float *pt = a.partial + (((int64_t)blockIdx.x * 2 + 0) * steps + rho) * S + k;
                        float *pp = a.partial + (((int64_t)blockIdx.x * 2 + 1) * steps + rho) * S + k;
                        *pt = (slab_i > 0) ? (*pt + vt) : vt;
                        *pp = (slab_i > 0) ? (*pp + vp) : vp;
                    }
                    rot_inv(dx, dy, cf.x, cf.y);
                    dx = cmulc(dx, ph.x, ph.y);
                    dy = cmulc(dy, ph.z, ph.w);
                    D[(int64_t)rt * stride] = dx;
                    D[(int64_t)rbm * stride] = dy;
                }
                if (UP) {  // G^dagger = diag(conj phases) R^T
                    rot_inv(x, y, cf.x, cf.y);
                    x = cmulc(x, ph.x, ph.y);
                    y = cmulc(y, ph.z, ph.w);
                } else {  // G = R diag(phases)
                    x = cmul(x, ph.x, ph.y);
                    y = cmul(y, ph.z, ph.w);
                    rot_fwd(x, y, cf.x, cf.y);
                }
                Z[(int64_t)rt * stride] = x;
                Z[(int64_t)rbm * stride] = y;
            }
        }
        if (live && !(GRAD && a.Y == nullptr)) {
            for (int i = 0; i < ne; i++) {
                const int row = a.lrow ? a.lrow[i] : i;
                if (row >= n) continue;
                float2 v = GRAD ? D[(int64_t)i * stride] : Z[(int64_t)i * stride];
                if (!UP && a.sfin[i]) v = neg_v(v);
                a.Y[(int64_t)row * a.ldy + 2 * col] = v.x;
                a.Y[(int64_t)row * a.ldy + 2 * col + 1] = v.y;
            }
        }
    }
    if (GRAD && slab_i == 0) {
        for (int64_t i = lane; i < (int64_t)2 * steps * S; i += 32) a.partial[(int64_t)blockIdx.x * 2 * steps * S + i] = 0.f;
    }
}

// ------------------------------------------------------------------ index trace
template <int W>
__global__ void k_trace(int ne, int L, int width, int up, int32_t *out) {
    const int lane = threadIdx.x;
    const int t = lane % width;      // every lane runs (shuffles need the full warp)
    const bool writer = lane < L;    // group 0's active lanes record
    const bool first = t == 0, last = t == L - 1;
    const int S = ne / 2, R = ne - 1;
    float T[W], B[W];
    for (int q = 0; q < W; q++) {
        int k = (t < L ? t : L - 1) * W + q;
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
            if (up) shift_up<W>(T, B, first, last, width);
            else shift_down<W>(T, B, first, last, width);
        }
    }
}

// the same for column groups spanning H = L/32 warps (one CTA of L threads): the values that
// cross a warp boundary go through shared memory, as in k_ring
template <int W>
__global__ void k_trace_multi(int ne, int La, int up, int32_t *out) {
    __shared__ float xs[2][32][2];  // [parity][warp][0: to warp h-1, 1: to warp h+1]
    const int t = threadIdx.x, lane = t & 31, h = t >> 5, H = blockDim.x / 32;
    const bool first = t == 0, last = t == La - 1;
    const int S = ne / 2, R = ne - 1;
    float T[W], B[W];
    for (int q = 0; q < W; q++) {
        int k = (t < La ? t : La - 1) * W + q;
        T[q] = (float)(up ? row_sRm1(k, ne) : row_s0(k));
        B[q] = (float)(up ? row_sRm1(ne - 1 - k, ne) : row_s0(ne - 1 - k));
    }
    for (int body = 0; body < 2 * S / W; body++) {
#pragma unroll
        for (int uu = 0; uu < W; uu++) {
            int u = body * W + uu, par = u & 1;
            if (u >= 1 && t < La) {
                int r = up ? (u - 1) : (R - u);
                for (int q = 0; q < W; q++) {
                    int k = t * W + q;
                    int a = (int)T[q], b = (int)B[q];
                    out[((int64_t)r * S + k) * 2] = a < b ? a : b;
                    out[((int64_t)r * S + k) * 2 + 1] = a < b ? b : a;
                }
            }
            if (up) {
                if (lane == 31) xs[par][h][1] = T[W - 1];
                if (lane == 0) xs[par][h][0] = B[0];
            } else {
                if (lane == 0) xs[par][h][0] = T[0];
                if (lane == 31) xs[par][h][1] = B[W - 1];
            }
            __syncthreads();
            if (up) {
                float fp = shfl_up_v(T[W - 1], 32), fn = shfl_dn_v(B[0], 32);
                if (lane == 0 && h > 0) fp = xs[par][h - 1][1];
                if (lane == 31 && h < H - 1) fn = xs[par][h + 1][0];
                shift_up_with<W>(T, B, first, last, fp, fn);
            } else {
                float fn = shfl_dn_v(T[0], 32), fp = shfl_up_v(B[W - 1], 32);
                if (lane == 31 && h < H - 1) fn = xs[par][h + 1][0];
                if (lane == 0 && h > 0) fp = xs[par][h - 1][1];
                shift_down_with<W>(T, B, first, last, fn, fp);
            }
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

// ring configurations compiled in ring_inst.cu (one object per (W, L))
#define GK_RING_CONFIGS(X) X(4, 1) X(8, 1) X(16, 1) X(32, 1) X(16, 4) X(16, 8) X(16, 16) X(16, 32) X(8, 64) \
    X(16, 64) X(32, 32) X(16, 128) X(8, 32) X(8, 128) X(8, 16)

int launch_ring(int mode, const Cfg &c, RingArgs &ra, int64_t grid, cudaStream_t st) {
    cudaError_t e = cudaErrorInvalidConfiguration;
    bool found = false;
#define GK_TRY(WW, LL)                                        \
    if (!found && c.W == WW && c.L == LL) {                   \
        found = true;                                         \
        e = gk::ring_launch_##WW##_##LL(mode, ra, grid, st);  \
    }
    GK_RING_CONFIGS(GK_TRY)
#undef GK_TRY
    if (!found) return fail(GIVENS_EUNSUPPORTED, "no ring kernel for W=%d L=%d", c.W, c.L);
    if (e != cudaSuccess) return fail(GIVENS_ECUDA, "ring kernel launch: %s", cudaGetErrorString(e));
    return 0;
}

// Layout options (start permutation, reflection); perm is a device int32[n_eff] or NULL.
struct Lay {
    const int32_t *perm;
    int refl;
};
constexpr Lay kNoLay{nullptr, -1};

// a launch with the programmatic-stream-serialization attribute (pdl_wait / pdl_trigger, common.cuh)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kfn)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = (GK_PDL && pdl) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kfn, static_cast<KArgs>(args)...);
}

// the same without the attribute: the stage-2 reduction (launched early, its small CTAs would sit
// beside the latency-bound ring CTAs on the same SMs while they wait; measured slower at n = 1024)
template <typename... KArgs, typename... Args>
cudaError_t launch_plain(void (*kfn)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, Args... args) {
    kfn<<<grid, block, 0, st>>>(static_cast<KArgs>(args)...);
    return cudaGetLastError();
}

int run_precompute(const Cfg &c, int n, const float *theta, const uint8_t *mask, uint8_t *ws, const WsLayout &L,
                   cudaStream_t st, const float *phi = nullptr, Lay lo = kNoLay) {
    untag_tables(ws);  // partially rebuilt tables must not pass for the old ones if a launch fails
    // the layout block only under a start permutation (the kernels take lay == NULL as the identity)
    int32_t *lay = nullptr;
    if (lo.perm) {
        lay = reinterpret_cast<int32_t *>(ws + L.lay);
        k_layout<<<1, 1024, 0, st>>>(n, c.ne, lo.perm, lo.refl, lay);
        CUDA_TRY(cudaGetLastError());
    }
    {
        const int RW = (c.R + 31) / 32;
        k_sigma_bits<<<(unsigned)c.ne, (unsigned)(32 * std::min(RW, 32)), 0, st>>>(
            n, c.ne, theta, mask, lay, lo.refl, reinterpret_cast<uint32_t *>(ws + L.sig), ws + L.sfin);
        CUDA_TRY(cudaGetLastError());
    }
    int64_t tot = (int64_t)(c.R + 2) * c.S;
    int W = c.fast ? c.W : c.S, Lq = c.fast ? c.La : 1;
    // (dependent launch where the table is small enough for k_coef's first wave to matter: n_eff <= 2048;
    // the n = 4096 U-build measured 6.98 -> 7.06 ms with it)
    CUDA_TRY(launch_pdl(k_coef, (unsigned)((tot + 255) / 256), 256, st, tot <= (int64_t)1 << 21, n, c.ne, W, Lq, c.rowbytes, theta, mask,
                        reinterpret_cast<const uint32_t *>(ws + L.sig), lay, ws + L.coef,
                        reinterpret_cast<int32_t *>(ws + L.amap)));
    if (phi) {
        k_coef_u<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, c.ne, W, Lq, theta, phi, mask,
                                                                reinterpret_cast<const uint32_t *>(ws + L.sig), lay,
                                                                reinterpret_cast<float4 *>(ws + L.coef_ph),
                                                                reinterpret_cast<float4 *>(ws + L.coef_pf),
                                                                reinterpret_cast<float4 *>(ws + L.coef_pt),
                                                                reinterpret_cast<float2 *>(ws + L.coef_ab));
        CUDA_TRY(cudaGetLastError());
    }
    tag_tables(ws, make_tag(c, n, theta, phi, mask, lo.perm, lo.refl));
    return 0;
}

int AutoWs::get(void *&ws, size_t &bytes, size_t need, cudaStream_t s) {
    if (ws) return 0;
    cudaError_t e = cudaMallocAsync(&p, need ? need : 256, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return fail(e == cudaErrorMemoryAllocation ? GIVENS_ENOMEM : GIVENS_ECUDA,
                    "cudaMallocAsync of a %zu-byte workspace: %s", need, cudaGetErrorString(e));
    }
    st = s;
    ws = p;
    bytes = need;
    return 0;
}

// ws may be NULL (a stream-ordered workspace is then allocated for the call, AutoWs)
int check_common(int32_t n, int64_t m, const void *ws, size_t ws_bytes, int op) {
    if (n < 2) return fail(GIVENS_EINVAL, "n must be >= 2 (got %d)", n);
    if (n > 32768) return fail(GIVENS_EINVAL, "n must be <= 32768 (got %d)", n);
    if (m < 0) return fail(GIVENS_EINVAL, "m must be >= 0");
    if (!ws) return 0;
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
                   float *Y, int64_t ldy, uint8_t *ws, const WsLayout &L, const Cfg &c, cudaStream_t st,
                   const int32_t *perm) {
    if (m == 0) return 0;
    int64_t grid = grid_for(c, mode, m);
    if (c.fast) mode = launch_mode(c, mode, m);
    if (c.fast) {
        RingArgs ra;
        ra.n = n; ra.ne = c.ne; ra.La = c.La;
        ra.m = m; ra.X = X; ra.ldx = ldx; ra.dY = dY; ra.lddy = lddy; ra.Y = Y; ra.ldy = ldy;
        ra.coef = ws + L.coef; ra.sfin = ws + L.sfin;
        ra.lrow = perm ? reinterpret_cast<const int32_t *>(ws + L.lay) : nullptr;
        // unitary phases: FFMA2-ready pairs for the forward / adjoint apply, the compact form for the
        // backward (which also needs the (alpha, beta) weights)
        ra.coef_ph = ws + ((mode & 3) == M_BWD ? L.coef_ph : ((mode & 3) == M_TRANS ? L.coef_pt : L.coef_pf));
        ra.coef_ab = ws + L.coef_ab;
        ra.partial = reinterpret_cast<float *>(ws + L.partial);
        ra.fgmask = reinterpret_cast<const uint32_t *>(ws + L.fgm);
        ra.sfg = reinterpret_cast<const float *>(ws + L.sfg);
        ra.nslabs = (m + cols_per_slab(c, mode) - 1) / cols_per_slab(c, mode);
        int K = kcols(c.W, mode);
        ra.vec_ok = vec_ok_for(K, {{X, ldx}, {dY, lddy}, {Y, ldy}});
        return launch_ring(mode, c, ra, grid, st);
    }
    GenArgs ga;
    ga.n = n; ga.ne = c.ne; ga.S = c.S; ga.rowbytes = c.rowbytes; ga.m = m;
    ga.X = X; ga.ldx = ldx; ga.dY = dY; ga.lddy = lddy; ga.Y = Y; ga.ldy = ldy;
    ga.coef = ws + L.coef; ga.sfin = ws + L.sfin;
    ga.lrow = perm ? reinterpret_cast<const int32_t *>(ws + L.lay) : nullptr;
    ga.coef_ph = reinterpret_cast<const float4 *>(ws + L.coef_ph);
    ga.coef_ab = reinterpret_cast<const float2 *>(ws + L.coef_ab);
    ga.partial = reinterpret_cast<float *>(ws + L.partial);
    ga.scratch = reinterpret_cast<float *>(ws + L.scratch);
    ga.nslabs = (mode & M_UNI) ? (m / 2 + 31) / 32 : (m + 31) / 32;
    switch (mode) {
        case M_FWD: k_generic<M_FWD><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_BUILDU: k_generic<M_BUILDU><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_TRANS: k_generic<M_TRANS><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_BWD: k_generic<M_BWD><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_FWD | M_UNI: k_generic_u<M_FWD><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_BUILDU | M_UNI: k_generic_u<M_BUILDU><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_TRANS | M_UNI: k_generic_u<M_TRANS><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        case M_BWD | M_UNI: k_generic_u<M_BWD><<<(unsigned)grid, 32, 0, st>>>(ga); break;
        default: return fail(GIVENS_EINVAL, "bad mode %d", mode);
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

void givens_workspace_reset(const void *ws) {
    if (ws) untag_tables(ws);
}

int givens_check_perm(int32_t n, const int32_t *perm_host) {
    if (n < 2 || n > 32768) return fail(GIVENS_EINVAL, "n must be in [2, 32768] (got %d)", n);
    if (!perm_host) return 0;
    const int ne = n + (n & 1);
    std::string seen((size_t)ne, '\0');
    for (int l = 0; l < ne; l++) {
        int v = perm_host[l];
        if (v < 0 || v >= ne) return fail(GIVENS_EINVAL, "perm[%d] = %d out of range [0, %d)", l, v, ne);
        if (seen[(size_t)v]) return fail(GIVENS_EINVAL, "perm has a duplicate entry %d", v);
        seen[(size_t)v] = 1;
    }
    return 0;
}

int givens_schedule_ex(int32_t n, const int32_t *perm_host, int32_t *pairs_host, int64_t *flat_host) {
    int rc = givens_check_perm(n, perm_host);
    if (rc) return rc;
    int ne = n + (n & 1), S = ne / 2, R = ne - 1;
    int64_t f = 0;
    for (int r = 0; r < R; r++)
        for (int k = 0; k < S; k++) {
            int a = seq_at(r, k, ne), b = seq_at(r, ne - 1 - k, ne);  // labels
            if (perm_host) { a = perm_host[a]; b = perm_host[b]; }
            int64_t q = (int64_t)r * S + k;
            if (pairs_host) {
                pairs_host[2 * q] = a < b ? a : b;
                pairs_host[2 * q + 1] = a < b ? b : a;
            }
            int64_t idx = (a == n || b == n) ? -1 : f++;  // block-major, byes skipped
            if (flat_host) flat_host[q] = idx;
        }
    return 0;
}

int givens_schedule(int32_t n, int32_t *pairs_host, int64_t *flat_host) {
    return givens_schedule_ex(n, nullptr, pairs_host, flat_host);
}

int givens_mask_from_dims_ex(int32_t n, const int32_t *perm_host, const uint8_t *excl, uint8_t *mask) {
    if (n < 2 || !excl || !mask) return fail(GIVENS_EINVAL, "bad arguments");
    int rc = givens_check_perm(n, perm_host);
    if (rc) return rc;
    int ne = n + (n & 1), S = ne / 2, R = ne - 1;
    int64_t f = 0;
    for (int r = 0; r < R; r++)
        for (int k = 0; k < S; k++) {
            int a = seq_at(r, k, ne), b = seq_at(r, ne - 1 - k, ne);
            if (perm_host) { a = perm_host[a]; b = perm_host[b]; }
            if (a == n || b == n) continue;
            mask[f++] = (excl[a] && excl[b]) ? 0 : 1;
        }
    return 0;
}

int givens_mask_from_dims(int32_t n, const uint8_t *excl, uint8_t *mask) {
    return givens_mask_from_dims_ex(n, nullptr, excl, mask);
}

size_t givens_workspace_bytes(int op, int32_t n, int64_t m) {
    if (n < 2 || n > 32768 || m < 0 || op < 0 || op > 5) return 0;
    Cfg c = cfg_for_op(n, op, (op % 3) == GIVENS_OP_BUILD_U ? n : m);
    return ws_layout(c, op, (op % 3) == GIVENS_OP_BUILD_U ? n : m).total;
}

int givens_u_supported(int32_t n) { return (n >= 2 && n <= 32768) ? 1 : 0; }

int givens_u_apply_ex(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask, const float *X,
                   int64_t ldx, float *Y, int64_t ldy, int adjoint, const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_common(n, m, ws, ws_bytes, GIVENS_OP_U_APPLY);
    if (rc) return rc;
    if (reflect_col < -1 || reflect_col >= n) return fail(GIVENS_EINVAL, "reflect_col must be -1 or in [0, n)");
    if (!theta || !phi || (m > 0 && (!X || !Y))) return fail(GIVENS_EINVAL, "theta, phi, X and Y must be non-NULL");
    if (ldx < m || ldy < m) return fail(GIVENS_EINVAL, "leading dimension smaller than m");
    if (X == Y && ldx != ldy) return fail(GIVENS_EINVAL, "in-place apply needs ldx == ldy");
    Cfg c = make_cfg_u(n);
    WsLayout L = ws_layout(c, GIVENS_OP_U_APPLY, m);
    cudaStream_t st = (cudaStream_t)stream;
    AutoWs aw;
    if ((rc = aw.get(ws, ws_bytes, L.total, st))) return rc;
    uint8_t *w = (uint8_t *)ws;
    if ((rc = run_precompute(c, n, theta, mask, w, L, st, phi, Lay{perm, reflect_col}))) return rc;
    // a complex column is two interleaved real columns
    return run_apply_mode((adjoint ? M_TRANS : M_FWD) | M_UNI, n, 2 * m, X, 2 * ldx, nullptr, 0, Y, 2 * ldy, w, L,
                          c, st, perm);
}

int givens_u_build_U_ex(int32_t n, const float *theta, const float *phi, const uint8_t *mask, float *U, int64_t ldu,
                     const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_common(n, n, ws, ws_bytes, GIVENS_OP_U_BUILD_U);
    if (rc) return rc;
    if (reflect_col < -1 || reflect_col >= n) return fail(GIVENS_EINVAL, "reflect_col must be -1 or in [0, n)");
    if (!theta || !phi || !U) return fail(GIVENS_EINVAL, "theta, phi and U must be non-NULL");
    if (ldu < n) return fail(GIVENS_EINVAL, "ldu < n");
    Cfg c = make_cfg_u(n);
    WsLayout L = ws_layout(c, GIVENS_OP_U_BUILD_U, n);
    cudaStream_t st = (cudaStream_t)stream;
    AutoWs aw;
    if ((rc = aw.get(ws, ws_bytes, L.total, st))) return rc;
    uint8_t *w = (uint8_t *)ws;
    if ((rc = run_precompute(c, n, theta, mask, w, L, st, phi, Lay{perm, reflect_col}))) return rc;
    return run_apply_mode(M_BUILDU | M_UNI, n, 2 * (int64_t)n, nullptr, 0, nullptr, 0, U, 2 * ldu, w, L, c, st, perm);
}

int givens_u_backward_ex(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask,
                      const float *Y, int64_t ldy, const float *dY, int64_t lddy, float *dX, int64_t lddx,
                      float *dtheta, float *dphi, int flags, const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_common(n, m, ws, ws_bytes, GIVENS_OP_U_BACKWARD);
    if (rc) return rc;
    if (reflect_col < -1 || reflect_col >= n) return fail(GIVENS_EINVAL, "reflect_col must be -1 or in [0, n)");
    if (!theta || !phi || !dtheta || !dphi || (m > 0 && (!Y || !dY)))
        return fail(GIVENS_EINVAL, "theta, phi, Y, dY, dtheta and dphi must be non-NULL");
    if (ldy < m || lddy < m || (dX && lddx < m)) return fail(GIVENS_EINVAL, "leading dimension smaller than m");
    if (dX && dX == dY && lddx != lddy) return fail(GIVENS_EINVAL, "in-place dX needs lddx == lddy");
    Cfg c = make_cfg_u(n);
    WsLayout L = ws_layout(c, GIVENS_OP_U_BACKWARD, m);
    cudaStream_t st = (cudaStream_t)stream;
    if (flags & GIVENS_FLAG_REUSE_TABLES) {
        if ((rc = check_tables(ws, make_tag(c, n, theta, phi, mask, perm, reflect_col)))) return rc;
    }
    AutoWs aw;
    if ((rc = aw.get(ws, ws_bytes, L.total, st))) return rc;
    uint8_t *w = (uint8_t *)ws;
    if (!(flags & GIVENS_FLAG_REUSE_TABLES)) {
        if ((rc = run_precompute(c, n, theta, mask, w, L, st, phi, Lay{perm, reflect_col}))) return rc;
    }
    int64_t N = givens_num_angles(n);
    if (m == 0) {
        CUDA_TRY(cudaMemsetAsync(dtheta, 0, (size_t)N * 4, st));
        CUDA_TRY(cudaMemsetAsync(dphi, 0, (size_t)N * 4, st));
        return 0;
    }
    if ((rc = run_apply_mode(M_BWD | M_UNI, n, 2 * m, Y, 2 * ldy, dY, 2 * lddy, dX, 2 * lddx, w, L, c, st, perm))) return rc;
    int64_t G = grid_for(c, M_BWD | M_UNI, 2 * m);
    const int64_t tot = (int64_t)2 * c.S * c.S;
    CUDA_TRY(launch_plain(k_dtheta_reduce, (unsigned)((tot + 255) / 256), 256, st,
        c.S, c.fast ? c.W : c.S, c.fast ? c.L : 1, ring_warps(launch_mode(c, M_BWD | M_UNI, 2 * m)), (int)G, c.fast, 2,
        reinterpret_cast<const float *>(w + L.partial),
        reinterpret_cast<const int32_t *>(w + L.amap), dtheta, dphi));
    return 0;
}

int givens_apply_ex(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx,
                 float *Y, int64_t ldy, int transpose, const int32_t *perm, int32_t reflect_col, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_common(n, m, ws, ws_bytes, GIVENS_OP_APPLY);
    if (rc) return rc;
    if (reflect_col < -1 || reflect_col >= n) return fail(GIVENS_EINVAL, "reflect_col must be -1 or in [0, n)");
    if (!theta || (m > 0 && (!X || !Y))) return fail(GIVENS_EINVAL, "theta, X and Y must be non-NULL");
    if (ldx < m || ldy < m) return fail(GIVENS_EINVAL, "leading dimension smaller than m");
    if (X == Y && ldx != ldy) return fail(GIVENS_EINVAL, "in-place apply needs ldx == ldy");
    Cfg c = make_cfg(n, m);
    WsLayout L = ws_layout(c, GIVENS_OP_APPLY, m);
    cudaStream_t st = (cudaStream_t)stream;
    AutoWs aw;
    if ((rc = aw.get(ws, ws_bytes, L.total, st))) return rc;
    uint8_t *w = (uint8_t *)ws;
    if ((rc = run_precompute(c, n, theta, mask, w, L, st, nullptr, Lay{perm, reflect_col}))) return rc;
    return run_apply_mode(transpose ? M_TRANS : M_FWD, n, m, X, ldx, nullptr, 0, Y, ldy, w, L, c, st, perm);
}

int givens_build_U_ex(int32_t n, const float *theta, const uint8_t *mask, float *U, int64_t ldu,
                      const int32_t *perm, int32_t reflect_col, void *ws,
                   size_t ws_bytes, void *stream) {
    int rc = check_common(n, n, ws, ws_bytes, GIVENS_OP_BUILD_U);
    if (rc) return rc;
    if (reflect_col < -1 || reflect_col >= n) return fail(GIVENS_EINVAL, "reflect_col must be -1 or in [0, n)");
    if (!theta || !U) return fail(GIVENS_EINVAL, "theta and U must be non-NULL");
    if (ldu < n) return fail(GIVENS_EINVAL, "ldu < n");
    Cfg c = make_cfg(n, n);
    WsLayout L = ws_layout(c, GIVENS_OP_BUILD_U, n);
    cudaStream_t st = (cudaStream_t)stream;
    AutoWs aw;
    if ((rc = aw.get(ws, ws_bytes, L.total, st))) return rc;
    uint8_t *w = (uint8_t *)ws;
    if ((rc = run_precompute(c, n, theta, mask, w, L, st, nullptr, Lay{perm, reflect_col}))) return rc;
    return run_apply_mode(M_BUILDU, n, n, nullptr, 0, nullptr, 0, U, ldu, w, L, c, st, perm);
}

int givens_backward_ex(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *Y, int64_t ldy,
                    const float *dY, int64_t lddy, float *dX, int64_t lddx, float *dtheta, int flags, const int32_t *perm, int32_t reflect_col, void *ws,
                    size_t ws_bytes, void *stream) {
    int rc = check_common(n, m, ws, ws_bytes, GIVENS_OP_BACKWARD);
    if (rc) return rc;
    if (reflect_col < -1 || reflect_col >= n) return fail(GIVENS_EINVAL, "reflect_col must be -1 or in [0, n)");
    if (!theta || !dtheta || (m > 0 && (!Y || !dY))) return fail(GIVENS_EINVAL, "theta, Y, dY and dtheta must be non-NULL");
    if (ldy < m || lddy < m || (dX && lddx < m)) return fail(GIVENS_EINVAL, "leading dimension smaller than m");
    if (dX && dX == dY && lddx != lddy) return fail(GIVENS_EINVAL, "in-place dX needs lddx == lddy");
    Cfg c = make_cfg(n, m);
    WsLayout L = ws_layout(c, GIVENS_OP_BACKWARD, m);
    cudaStream_t st = (cudaStream_t)stream;
    if (flags & GIVENS_FLAG_REUSE_TABLES) {
        if ((rc = check_tables(ws, make_tag(c, n, theta, nullptr, mask, perm, reflect_col)))) return rc;
    }
    AutoWs aw;
    if ((rc = aw.get(ws, ws_bytes, L.total, st))) return rc;
    uint8_t *w = (uint8_t *)ws;
    if (!(flags & GIVENS_FLAG_REUSE_TABLES)) {
        if ((rc = run_precompute(c, n, theta, mask, w, L, st, nullptr, Lay{perm, reflect_col}))) return rc;
    }
    int64_t N = givens_num_angles(n);
    if (m == 0) {
        CUDA_TRY(cudaMemsetAsync(dtheta, 0, (size_t)N * 4, st));
        return 0;
    }
    if ((rc = run_apply_mode(M_BWD, n, m, Y, ldy, dY, lddy, dX, lddx, w, L, c, st, perm))) return rc;
    int64_t G = grid_for(c, M_BWD, m);
    const int64_t tot = (int64_t)2 * c.S * c.S;
    CUDA_TRY(launch_plain(k_dtheta_reduce, (unsigned)((tot + 255) / 256), 256, st,
        c.S, c.fast ? c.W : c.S, c.fast ? c.L : 1, ring_warps(launch_mode(c, M_BWD, m)), (int)G, c.fast, 1,
        reinterpret_cast<const float *>(w + L.partial), reinterpret_cast<const int32_t *>(w + L.amap),
        dtheta, nullptr));
    return 0;
}

// ------------------------------------------------------------------ identity-layout entry points
int givens_apply(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx,
                 float *Y, int64_t ldy, int transpose, void *ws, size_t ws_bytes, void *stream) {
    return givens_apply_ex(n, m, theta, mask, X, ldx, Y, ldy, transpose, nullptr, -1, ws, ws_bytes, stream);
}
int givens_build_U(int32_t n, const float *theta, const uint8_t *mask, float *U, int64_t ldu, void *ws,
                   size_t ws_bytes, void *stream) {
    return givens_build_U_ex(n, theta, mask, U, ldu, nullptr, -1, ws, ws_bytes, stream);
}
int givens_backward(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *Y, int64_t ldy,
                    const float *dY, int64_t lddy, float *dX, int64_t lddx, float *dtheta, int flags, void *ws,
                    size_t ws_bytes, void *stream) {
    return givens_backward_ex(n, m, theta, mask, Y, ldy, dY, lddy, dX, lddx, dtheta, flags, nullptr, -1, ws,
                              ws_bytes, stream);
}
int givens_u_apply(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask, const float *X,
                   int64_t ldx, float *Y, int64_t ldy, int adjoint, void *ws, size_t ws_bytes, void *stream) {
    return givens_u_apply_ex(n, m, theta, phi, mask, X, ldx, Y, ldy, adjoint, nullptr, -1, ws, ws_bytes, stream);
}
int givens_u_build_U(int32_t n, const float *theta, const float *phi, const uint8_t *mask, float *U, int64_t ldu,
                     void *ws, size_t ws_bytes, void *stream) {
    return givens_u_build_U_ex(n, theta, phi, mask, U, ldu, nullptr, -1, ws, ws_bytes, stream);
}
int givens_u_backward(int32_t n, int64_t m, const float *theta, const float *phi, const uint8_t *mask,
                      const float *Y, int64_t ldy, const float *dY, int64_t lddy, float *dX, int64_t lddx,
                      float *dtheta, float *dphi, int flags, void *ws, size_t ws_bytes, void *stream) {
    return givens_u_backward_ex(n, m, theta, phi, mask, Y, ldy, dY, lddy, dX, lddx, dtheta, dphi, flags, nullptr, -1,
                                ws, ws_bytes, stream);
}

// ------------------------------------------------------------------ fast Givens
namespace {
int fast_common(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx, float *Y,
                int64_t ldy, int mode, void *ws, size_t ws_bytes, cudaStream_t st) {
    Cfg c = make_cfg(n, m);
    if (!(c.fast && c.L == 1 && c.La == 1))
        return fail(GIVENS_EUNSUPPORTED, "fast Givens runs on one-lane columns only (n_eff in {8, 16, 32, 64}; n = %d)", n);
    WsLayout L = ws_layout(c, GIVENS_OP_APPLY, m);
    AutoWs aw;
    int rc;
    if ((rc = aw.get(ws, ws_bytes, L.total, st))) return rc;
    uint8_t *w = (uint8_t *)ws;
    untag_tables(w);  // the tables below are not the three-shear ones a backward could reuse
    k_fg_tables<<<1, 32, 0, st>>>(n, c.ne, theta, mask, w + L.coef, c.rowbytes, reinterpret_cast<uint32_t *>(w + L.fgm),
                                  reinterpret_cast<float *>(w + L.sfg));
    CUDA_TRY(cudaGetLastError());
    return run_apply_mode(mode | M_FG, n, m, X, ldx, nullptr, 0, Y, ldy, w, L, c, st, nullptr);
}
}  // namespace

int givens_fast_apply(int32_t n, int64_t m, const float *theta, const uint8_t *mask, const float *X, int64_t ldx,
                      float *Y, int64_t ldy, void *ws, size_t ws_bytes, void *stream) {
    int rc = check_common(n, m, ws, ws_bytes, GIVENS_OP_APPLY);
    if (rc) return rc;
    if (!theta || (m > 0 && (!X || !Y))) return fail(GIVENS_EINVAL, "theta, X and Y must be non-NULL");
    if (ldx < m || ldy < m) return fail(GIVENS_EINVAL, "leading dimension smaller than m");
    if (X == Y && ldx != ldy) return fail(GIVENS_EINVAL, "in-place apply needs ldx == ldy");
    if (m == 0) return make_cfg(n).L == 1 && make_cfg(n).fast ? 0 : fail(GIVENS_EUNSUPPORTED, "fast Givens: n = %d", n);
    return fast_common(n, m, theta, mask, X, ldx, Y, ldy, M_FWD, ws, ws_bytes, (cudaStream_t)stream);
}

int givens_fast_build_U(int32_t n, const float *theta, const uint8_t *mask, float *U, int64_t ldu, void *ws,
                        size_t ws_bytes, void *stream) {
    int rc = check_common(n, n, ws, ws_bytes, GIVENS_OP_BUILD_U);
    if (rc) return rc;
    if (!theta || !U) return fail(GIVENS_EINVAL, "theta and U must be non-NULL");
    if (ldu < n) return fail(GIVENS_EINVAL, "ldu < n");
    return fast_common(n, n, theta, mask, nullptr, 0, U, ldu, M_BUILDU, ws, ws_bytes, (cudaStream_t)stream);
}

int givens_index_trace(int32_t n, int direction, int32_t *out_dev, void *stream) {
    if (n < 2 || n > 32768 || !out_dev) return fail(GIVENS_EINVAL, "bad arguments");
    Cfg c = make_cfg(n);
    cudaStream_t st = (cudaStream_t)stream;
    int up = direction ? 1 : 0;
    if (c.fast && c.L > 32) {
        switch (c.W) {
            case 8: k_trace_multi<8><<<1, c.L, 0, st>>>(c.ne, c.La, up, out_dev); break;
            case 16: k_trace_multi<16><<<1, c.L, 0, st>>>(c.ne, c.La, up, out_dev); break;
            case 32: k_trace_multi<32><<<1, c.L, 0, st>>>(c.ne, c.La, up, out_dev); break;
        }
    } else if (c.fast) {
        const int width = c.L < 32 ? c.L : 32;
        switch (c.W) {
            case 4: k_trace<4><<<1, 32, 0, st>>>(c.ne, c.La, width, up, out_dev); break;
            case 8: k_trace<8><<<1, 32, 0, st>>>(c.ne, c.La, width, up, out_dev); break;
            case 16: k_trace<16><<<1, 32, 0, st>>>(c.ne, c.La, width, up, out_dev); break;
            case 32: k_trace<32><<<1, 32, 0, st>>>(c.ne, c.La, width, up, out_dev); break;
        }
    } else {
        int64_t RS = (int64_t)c.R * c.S;
        k_trace_generic<<<(unsigned)((RS + 255) / 256), 256, 0, st>>>(c.ne, out_dev);
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // extern "C"

#include "gemm_path.inc"
