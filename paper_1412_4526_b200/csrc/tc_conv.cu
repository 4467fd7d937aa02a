// d-regularly sparse convolution on the 5th-gen tensor cores (tcgen05, sm_100a),
// fp32 in/out with 3xTF32 products -- the "fast tier" of the conv data path.
//
// Computes, like conv_direct.cu (same argument meaning),
//   forward        y[o,u,v]  = b[o] + sum_{c,i,j} w[o,c,i,j] * x[c, u+i*d, v+j*d]
//   data gradient  dx[c,y,x] = sum_{o,i,j} w[o,c,l-1-i,l-1-j] * dy_pad[o, y+i*d, x+j*d]
// (reference _kernels.pyx:23-53 and :56-91) as an implicit GEMM with
//   M = 128 output pixels (4 rows x 32 columns), N = output channels (padded to 16),
//   K = (channel chunk of 8, tap i, tap j): one tcgen05.mma kind::tf32 K-step each.
// A CTA tile stacks MT such M tiles vertically (4*MT rows x 32 columns).
//
// 3xTF32: every product is (A_hi + A_lo)(B_hi + B_lo) ~ A_hi B_hi + A_hi B_lo + A_lo B_hi
// with hi = raw fp32 bits (the tensor core truncates to tf32) and lo = x - trunc(x);
// results agree with fp32 up to summation order (~1e-6 normwise on 400-term sums; the
// reference tolerance for this path is 1e-4).
//
// Data flow per CTA (persistent, one per SM, 25 warps):
//   warps 16-23 loaders: for every (tile, channel chunk) copy the input window the l^2
//               taps need into a shared-memory "halo" buffer [8 ch][rows][cols] with
//               coalesced loads (any alignment; zero-fill outside the map = the data
//               gradient's padding).  Rows/columns are the halo (4*MT + (l-1)d rows,
//               32 + (l-1)d columns) or, for large dilations, only the l tap rows /
//               l*32 tap columns -- whichever is smaller.  Two or three buffers.
//   warps 8-15  converters, 2 groups x 4 warps (warp % 4 = TMEM lane quarter = pixel row
//               of every M tile): per K-step read the 8 channel values of their pixel
//               from the halo buffer (lane = column -> bank-conflict-free LDS), split
//               hi/lo in registers, write both into a TMEM stage with tcgen05.st.  The
//               tap only moves the read window; every input element is fetched from
//               global memory once per tile instead of l^2 times.
//   warp 24     streams the packed weights (B, K-major, hi and lo) through a 3-buffer
//               ring with bulk async copies, one unit per (channel chunk, tap row),
//               allocates TMEM, and issues the MMAs (one elected lane), one stage = one
//               K-step = MT M tiles:
//               A_hi x [B_hi|B_lo] (N = 2*Npad) + A_lo x B_hi   (Npad <= 16), or
//               A_hi x B_hi + A_hi x B_lo + A_lo x B_hi          (Npad >= 32),
//               and releases the stage with one tcgen05.commit.
//   warps 0-7   epilogue, 2 per TMEM lane quarter (M tiles split by parity): tcgen05.ld
//               the accumulators (double-buffered in TMEM so the next tile's MMAs
//               overlap), add bias + nonlinearity (forward) or apply the upstream
//               nonlinearity's derivative (data gradient), store NCHW.
// Measured before this layout (tools/tc_trace.cu): producers that gathered A straight
// from global memory spent ~2000 cycles per K-step on load latency, and a 4-warp
// epilogue with out-of-line tanh stalled the MMA ~12k cycles per tile.
#include <stdlib.h>

#include "dp_common.cuh"
#include "tc_ptx.cuh"

namespace dp {

constexpr int TC_MAX_STAGES = 16;
constexpr int TC_MAX_MT = 4;  // M tiles per CTA tile
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_NGROUPS = 2;      // converter groups of 4 warps, K-steps round-robin
constexpr int TC_CONV_WARP0 = 8;   // 2 groups x 4
constexpr int TC_LOAD_WARP0 = 16;  // 8 loader warps
constexpr int TC_LOAD_WARPS = 8;
constexpr int TC_MMA_WARP = 24;
constexpr int TC_MAX_HROWS = 128;  // halo buffer rows per channel
constexpr int TC_THREADS = (TC_MMA_WARP + 1) * 32;
constexpr int TC_MIN_STAGES = 4;
constexpr int TC_MAX_HB = 3;  // halo buffers (2 or 3, as shared memory allows)
constexpr int TC_LB = 8;  // loader: buffer rows in flight per warp
constexpr int TC_LC = 3;  // loader: 32-column groups per row (halo columns <= 96)
constexpr int TC_SMEM_BUDGET = 220 * 1024;
constexpr int TC_WB = 3;       // streamed weight-unit ring (per channel chunk and tap row)
constexpr int TC_MAX_WB = 64;  // resident mode: one buffer per unit

struct TcConvArgs {
    const float *in;     // (n, R, Hin, Win)
    const float *wpack;  // [n_ks][hi|lo][Npad x 8] K-major core-matrix layout
    const float *bias;   // (Q) for forward, nullptr for the data gradient
    float *out;          // (n, Q, Ho, Wo)
    const float *gate;   // (n, Q, Ho, Wo) nonlinearity output, or nullptr
    int R, Hin, Win, Q, Ho, Wo, l, d, pad, act, gate_kind;
    int n_rc, n_ks, Npad, MT, acc_cols, stages, tiles_x, tiles_y, total_tiles;
    uint32_t wbytes;
    uint32_t unit_bytes;  // packed weights of one (channel chunk, tap row): l K-steps
    int nwb, resident;    // weight-unit buffers; resident: all units loaded once
    // halo buffer geometry: rows (RB-row blocks per tap row i, step RS in the converter),
    // columns (CB-column blocks per tap column j, step CS)
    int hrows, hcols, RB, RS, CB, CS, HB;
    uint32_t hbytes;
    unsigned long long *trace;  // DP_TC_TRACE: per-K-step clock64 stamps of CTA 0 (8 slots)
};

#define TC_TRACE(A, KS, SLOT, COND)                                                  \
    do {                                                                             \
        if ((A).trace && (COND) && blockIdx.x == 0 && (KS) < 1024)                   \
            (A).trace[(KS) * 8 + (SLOT)] = clock64();                                \
    } while (0)

// --------------------------------------------------------------------------------
// weight packing: W(q, r, i, j) -> per K-step ks = (rc*l + i)*l + j two Npad x 8 tiles
// (hi = raw, lo = residual) in the K-major no-swizzle core-matrix layout:
// element (n, k) at byte (n>>3)*256 + (k>>2)*128 + (n&7)*16 + (k&3)*4.
// --------------------------------------------------------------------------------
// rp > 0: the last channel chunk holds rp <= 4 channels, tap-packed -- its K steps hold
// tp = 8 / rp column taps, slot k = t*rp + c <-> (c, j = g*tp + t), G = ceil(l / tp) K steps
// per tap row, after all (n_rc - 1) * l * l full K steps.
__global__ void tc_pack_weights(const float *__restrict__ w, float *__restrict__ wp, int Q, int R,
                                int l, int Npad, int n_rc, int n_ks, int bwd, int rp) {
    const int tp = rp ? 8 / rp : 1;
    const int G = (l + tp - 1) / tp;
    const int full = rp ? (n_rc - 1) * l * l : n_ks;
    int total = n_ks * 2 * Npad * 8;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += gridDim.x * blockDim.x) {
        int k = idx & 7;
        int n = (idx >> 3) % Npad;
        int hl = (idx / (8 * Npad)) & 1;
        int ks = idx / (16 * Npad);
        int c, i, j;
        bool slot_ok = true;
        if (ks < full) {
            j = ks % l;
            i = (ks / l) % l;
            c = (ks / (l * l)) * 8 + k;
        } else {
            const int kp = ks - full;
            i = kp / G;
            c = (n_rc - 1) * 8 + k % rp;
            j = (kp % G) * tp + k / rp;
            slot_ok = k < rp * tp && j < l;
        }
        float v = 0.f;
        if (n < Q && c < R && slot_ok) {
            if (!bwd)
                v = w[(((long long)n * R + c) * l + i) * l + j];
            else  // w is (R = cout, Q = cin, l, l), rotated by 180 degrees
                v = w[(((long long)c * Q + n) * l + (l - 1 - i)) * l + (l - 1 - j)];
        }
        if (hl) v = ptx::tf32_lo(v);
        int byte = hl * Npad * 32 + (n >> 3) * 256 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4;
        wp[(long long)ks * (Npad * 16) + byte / 4] = v;
    }
}

// fp16 split of the same weights for the flat kernel's HALF mode: K steps of 16
// channels, per K step [W_hi | W_lo] (Npad rows x 16 halves each), element (n, k) at byte
// (n>>3)*256 + (k>>3)*128 + (n&7)*16 + (k&7)*2 -- the same 64 * Npad bytes per K step.
// bwd: the data gradient's rotated weights (w is (R = cout, Q = cin, l, l)), lo' scaled by
// 2^11 (the offset split of the fp16 data gradient: cross products in their own columns)
// rp > 0: the LAST chunk holds rp <= 8 channels, tap-packed (tp = 16 / rp column taps per K
// step, slot k = t*rp + c <-> (c, j = g*tp + t), G = ceil(l / tp) K steps per tap row), after
// the (n_rc - 1) * l * l K steps of the full chunks
__global__ void tc_pack_weights_f16(const float *__restrict__ w, __half *__restrict__ wp, int Q,
                                    int R, int l, int Npad, int n_ks, int bwd, int *flag,
                                    int rp, int n_rc) {
    const int total = n_ks * 2 * Npad * 16;
    const int tp = rp ? 16 / rp : 1, G = (l + tp - 1) / tp;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += gridDim.x * blockDim.x) {
        const int k = idx & 15;
        const int n = (idx >> 4) % Npad;
        const int hl = (idx / (16 * Npad)) & 1;
        const int ks = idx / (32 * Npad);
        int j, i, c;
        bool slot_ok = true;
        const int full = rp ? (n_rc - 1) * l * l : n_ks;  // K steps of the full chunks
        if (ks >= full) {  // the tap-packed last chunk
            const int kp = ks - full;
            i = kp / G;
            c = (n_rc - 1) * 16 + k % rp;
            j = (kp % G) * tp + k / rp;
            slot_ok = k < rp * tp && j < l;
        } else {
            j = ks % l, i = (ks / l) % l, c = (ks / (l * l)) * 16 + k;
        }
        float v = 0.f;
        if (n < Q && c < R && slot_ok)  // bwd 1: rotated + offset split, 2: offset split only
            v = bwd == 1 ? w[(((long long)c * Q + n) * l + (l - 1 - i)) * l + (l - 1 - j)]
                         : w[(((long long)n * R + c) * l + i) * l + j];
        if (!(fabsf(v) < ptx::F16_SPLIT_MAX)) atomicOr(flag, 1);
        __half hi, lo;
        if (bwd) {
            hi = __float2half_rn(v);
            lo = __float2half_rn((v - __half2float(hi)) * ptx::F16_LO_SCALE);
        } else {
            ptx::f16_split(v, hi, lo);
        }
        const int byte = hl * Npad * 32 + (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
        wp[((long long)ks * Npad * 64 + byte) / 2] = hl ? lo : hi;
    }
}

int tc_pack_f16(const float *w, void *wp, int Q, int R, int l, int bwd, int *flag,
                cudaStream_t st, int rp) {
    const int Npad = (Q + 15) / 16 * 16, n_rc = (R + 15) / 16;
    const int tp = rp ? 16 / rp : 1;
    // rp: the last chunk tap-packed (G = ceil(l / tp) K steps per tap row)
    const int n_ks = rp ? (n_rc - 1) * l * l + l * ((l + tp - 1) / tp) : n_rc * l * l;
    const int total = n_ks * 2 * Npad * 16;
    tc_pack_weights_f16<<<ceil_div(total, 256), 256, 0, st>>>(w, (__half *)wp, Q, R, l, Npad,
                                                              n_ks, bwd, flag, rp, n_rc);
    return check_launch("tc_pack_weights_f16");
}

int tc_pack(const float *w, float *wp, int Q, int R, int l, int bwd, int rp, cudaStream_t st) {
    const int Npad = (Q + 15) / 16 * 16, n_rc = (R + 7) / 8;
    const int tp = rp ? 8 / rp : 1;
    const int n_ks = rp ? (n_rc - 1) * l * l + l * ((l + tp - 1) / tp) : n_rc * l * l;
    const int total = n_ks * 2 * Npad * 8;
    tc_pack_weights<<<ceil_div(total, 256), 256, 0, st>>>(w, wp, Q, R, l, Npad, n_rc, n_ks, bwd,
                                                          rp);
    return check_launch("tc_pack_weights");
}

// tap-stacked variant (tc_conv_tap.cu): preferred when it applies AND the caller's workspace
// holds its relayout planes (dp_conv_*_fast_workspace); else the flat variant
size_t tt_conv_workspace(int n, int R, int Hin, int Win, int Q, int l, int d, int pad, int Ho,
                         int Wo);
int tt_launch(const float *in, const float *w, const float *bias, float *out, const float *gate,
              int n, int R, int Hin, int Win, int Q, int Ho, int Wo, int l, int d, int pad,
              int act, int gate_kind, bool bwd, void *ws, size_t ws_bytes, cudaStream_t st,
              bool f16_ok = false);
// flattened shared-memory-operand variant (tc_conv_flat.cu), preferred when it applies
bool tf_conv_supported(int R, int Q, int l, int d);
size_t tf_relayout_workspace(int n, int R, int Hin, int Win, int Q, int l, int d, int pad,
                             int Ho, int Wo, bool bwd);
int tf_conv_forward(const float *, const float *, const float *, float *, int, int, int, int, int,
                    int, int, int, void *, size_t, cudaStream_t, int f16_ok);
int tf_conv_backward_data(const float *, const float *, float *, int, int, int, int, int, int,
                          int, const float *, int, void *, size_t, cudaStream_t);

// Epilogue tanh: single-precision tanhf (<= 2 ulp) kept out of line so the unrolled
// epilogue stays small (instruction cache); relu / identity are inlined.
__device__ __noinline__ float tc_tanh(float v) { return tanhf(v); }
__device__ __forceinline__ float tc_act(float v, int kind) {
    if (kind == DP_TANH || kind == DP_TANH_FAST) return tc_tanh(v);
    if (kind == DP_RELU) return dp_relu(v);
    return v;
}

__device__ __forceinline__ void tc_tile_origin(const TcConvArgs &a, int tile, int &img, int &u0,
                                               int &v0) {
    const int per_img = a.tiles_x * a.tiles_y;
    img = tile / per_img;
    const int rem = tile - img * per_img;
    const int ty = rem / a.tiles_x;
    u0 = ty * 4 * a.MT;
    v0 = (rem - ty * a.tiles_x) * 32;
}

template <bool STACKED, bool BWD, bool STREAM>
__global__ void __launch_bounds__(TC_THREADS, 1) tc_conv_kernel(const TcConvArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *wsm = smem_raw;  // nwb weight-unit buffers
    unsigned char *hsm = smem_raw + (size_t)a.nwb * a.unit_bytes;  // HB halo buffers
    __shared__ uint64_t full_bar[TC_MAX_STAGES], empty_bar[TC_MAX_STAGES];
    __shared__ uint64_t tfull_bar[2], tempty_bar[2], hfull[TC_MAX_HB], hempty[TC_MAX_HB];
    __shared__ uint64_t wfull[TC_MAX_WB], wempty[TC_MAX_WB];
    __shared__ uint32_t s_tmem;
    __shared__ int s_rowrel[TC_MAX_HROWS];  // halo row -> input row offset from u0 - pad

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int MT = a.MT;
    const int ll = a.l * a.l;
    for (int r = threadIdx.x; r < a.hrows; r += blockDim.x) {
        const int ib = r / a.RB;
        s_rowrel[r] = (r - ib * a.RB) + ib * a.d;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            ptx::mbar_init(&full_bar[s], 4);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull_bar[b], 1);
            ptx::mbar_init(&tempty_bar[b], TC_EPI_WARPS);
        }
        for (int b = 0; b < a.HB; ++b) {
            ptx::mbar_init(&hfull[b], TC_LOAD_WARPS);
            ptx::mbar_init(&hempty[b], 8);
        }
        for (int b = 0; b < a.nwb; ++b) {
            ptx::mbar_init(&wfull[b], 1);
            ptx::mbar_init(&wempty[b], 1);
        }
        ptx::mbar_fence_init();
    }
    if (warp == TC_MMA_WARP) ptx::tmem_alloc<512>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;
    // TMEM columns: [0, 2*MT*acc_cols) accumulators (2 tile buffers), then the A stages
    const uint32_t a_base = tmem + (uint32_t)(2 * MT * a.acc_cols);
    const long long plane_in = (long long)a.Hin * a.Win;

    if (warp >= TC_LOAD_WARP0 && warp < TC_MMA_WARP) {
        // ============================ halo loaders ============================
        // buffer rows (c, srow) are spread over the loader warps, lanes walk the columns:
        // row srow holds input row u0 - pad + s_rowrel[srow], column scol holds input
        // column v0 - pad + colrel (both fixed per kernel).  Coalesced LDG (lanes =
        // consecutive columns) -> STS with TC_LB rows of loads in flight per warp.
        // (4-byte cp.async measured ~43k cycles per chunk: LDGSTS throughput is per
        // thread-op, not per byte.)
        const int lw = warp - TC_LOAD_WARP0;
        const int nrows = 8 * a.hrows;
        int colrel[TC_LC];
#pragma unroll
        for (int cc = 0; cc < TC_LC; ++cc) {
            const int scol = lane + 32 * cc;
            const int jb = scol / a.CB;
            colrel[cc] = scol < a.hcols ? (scol - jb * a.CB) + jb * a.d : -(1 << 29);
        }
        int g = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            int img, u0, v0;
            tc_tile_origin(a, tile, img, u0, v0);
            const int ub = u0 - a.pad, vb = v0 - a.pad;
            for (int rc = 0; rc < a.n_rc; ++rc, ++g) {
                const int hb = g % a.HB;
                // loaders idle most of a chunk: back off instead of spinning on issue slots
                ptx::mbar_wait_sleep(&hempty[hb], ((g / a.HB) & 1) ^ 1);
                TC_TRACE(a, g * ll, 0, lw == 0 && lane == 0);
                float *buf = reinterpret_cast<float *>(hsm + (size_t)hb * a.hbytes);
                const float *src_c = a.in + ((long long)img * a.R + rc * 8) * plane_in;
                const int cvalid = min(8, a.R - rc * 8);
                int c = 0, srow = lw;  // row = c * hrows + srow, advanced without divides
                while (srow >= a.hrows) {
                    srow -= a.hrows;
                    ++c;
                }
                for (int row0 = lw; row0 < nrows; row0 += TC_LOAD_WARPS * TC_LB) {
                    float v[TC_LB][TC_LC];
                    int cb = c, sb = srow;
#pragma unroll
                    for (int b = 0; b < TC_LB; ++b) {
                        const int grow = ub + s_rowrel[sb < a.hrows ? sb : 0];
                        const bool rok = cb < cvalid && grow >= 0 && grow < a.Hin;
                        const float *src_r =
                            src_c + (long long)cb * plane_in + (long long)grow * a.Win + vb;
#pragma unroll
                        for (int cc = 0; cc < TC_LC; ++cc) {
                            const int gcol = vb + colrel[cc];
                            const bool ok = rok && gcol >= 0 && gcol < a.Win;
                            v[b][cc] = ok ? __ldg(src_r + colrel[cc]) : 0.f;
                        }
                        sb += TC_LOAD_WARPS;
                        while (sb >= a.hrows) {
                            sb -= a.hrows;
                            ++cb;
                        }
                    }
#pragma unroll
                    for (int b = 0; b < TC_LB; ++b) {
                        const int row = row0 + b * TC_LOAD_WARPS;
                        if (row >= nrows) break;
                        float *dst_r = buf + (size_t)row * a.hcols;
#pragma unroll
                        for (int cc = 0; cc < TC_LC; ++cc) {
                            const int scol = lane + 32 * cc;
                            if (scol < a.hcols) dst_r[scol] = v[b][cc];
                        }
                    }
                    c = cb;
                    srow = sb;
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&hfull[hb]);
                TC_TRACE(a, g * ll, 1, lw == 0 && lane == 0);
            }
        }
    } else if (warp >= TC_CONV_WARP0 && warp < TC_LOAD_WARP0) {
        // ============================ converters ============================
        const int q = warp & 3, grp = (warp - TC_CONV_WARP0) >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int cstride = a.hrows * a.hcols;  // floats between channels in a buffer
        int KS = 0, g = 0;
        int stage = 0, sphase = 0, hb = 0, hphase = 0, kmod = 0;  // incremental counters
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            for (int rc = 0; rc < a.n_rc; ++rc, ++g) {
                ptx::mbar_wait(&hfull[hb], hphase);
                const float *buf = reinterpret_cast<const float *>(hsm + (size_t)hb * a.hbytes);
                int i = 0, j = 0;
                for (int tap = 0; tap < ll; ++tap, ++KS) {
                    const bool mine = kmod == grp;
                    const int cur_stage = stage, cur_phase = sphase;
                    const int ci = i, cj = j;
                    if (++kmod == TC_NGROUPS) kmod = 0;
                    if (++stage == a.stages) {
                        stage = 0;
                        sphase ^= 1;
                    }
                    if (++j == a.l) {
                        j = 0;
                        ++i;
                    }
                    if (!mine) continue;
                    TC_TRACE(a, KS, 2, q == 0 && lane == 0);
                    ptx::mbar_wait(&empty_bar[cur_stage], cur_phase ^ 1);
                    ptx::tc_fence_after();
                    TC_TRACE(a, KS, 3, q == 0 && lane == 0);
                    const uint32_t sbase = a_base + lane_off + (uint32_t)(cur_stage * MT * 16);
                    const float *p0 = buf + (ci * a.RS + q) * a.hcols + lane + cj * a.CS;
#pragma unroll
                    for (int mt = 0; mt < TC_MAX_MT; ++mt) {
                        if (mt >= MT) break;
                        const float *p = p0 + 4 * mt * a.hcols;
                        float hi[8], lo[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) hi[k] = p[k * cstride];
#pragma unroll
                        for (int k = 0; k < 8; ++k) lo[k] = ptx::tf32_lo(hi[k]);
                        ptx::tmem_st8(sbase + mt * 16, hi);
                        ptx::tmem_st8(sbase + mt * 16 + 8, lo);
                    }
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&full_bar[cur_stage]);
                    TC_TRACE(a, KS, 4, q == 0 && lane == 0);
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&hempty[hb]);
                if (++hb == a.HB) {
                    hb = 0;
                    hphase ^= 1;
                }
            }
        }
    } else if (warp == TC_MMA_WARP) {
        // ============================ weights + MMA issuer ============================
        // The packed weights stream through a TC_WB-buffer ring in units of one (channel
        // chunk, tap row) = l K-steps (bulk async copies, L2-resident across tiles), so
        // wide layers fit (the whole weight set of e.g. a 96->128 3x3 layer is 884 KB).
        // Unit v+1 is requested when unit v starts; its buffer was last used by unit
        // v+2-TC_WB, whose MMAs have retired by then.
        const int units_per_tile = a.n_rc * a.l;
        const int my_tiles = (a.total_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
        const int total_units = my_tiles * units_per_tile;
        const unsigned char *wsrc = reinterpret_cast<const unsigned char *>(a.wpack);
        // request the next unit (incremental ring position; no divides on the MMA path)
        int rq = 0, rq_b = 0, rq_w = 0;  // next unit to request, its buffer, its weight unit
        uint32_t rq_ph = 0;              // completions of wempty[rq_b] to wait for (parity)
        auto request_next = [&]() {
            if (rq >= total_units) return;
            if (STREAM && rq >= TC_WB) ptx::mbar_wait(&wempty[rq_b], rq_ph ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_expect_tx(&wfull[rq_b], a.unit_bytes);
                const unsigned char *src = wsrc + (size_t)rq_w * a.unit_bytes;
                unsigned char *dst = wsm + (size_t)rq_b * a.unit_bytes;
                for (uint32_t off = 0; off < a.unit_bytes; off += 32768u) {
                    const uint32_t n = a.unit_bytes - off < 32768u ? a.unit_bytes - off : 32768u;
                    ptx::bulk_g2s(dst + off, src + off, n, &wfull[rq_b]);
                }
            }
            __syncwarp();
            ++rq;
            if (++rq_w == units_per_tile) rq_w = 0;
            if (++rq_b == a.nwb) {
                rq_b = 0;
                rq_ph ^= 1;
            }
        };
        if (!STREAM) {
            for (int v = 0; v < units_per_tile && v < total_units; ++v) request_next();
        } else {
            request_next();
        }
        int unit = 0, wb = 0;
        uint32_t wph = 0;
        const uint32_t wsm_addr = ptx::smem_u32(wsm);
        const uint32_t ks_bytes = (uint32_t)a.Npad * 64;  // hi + lo tiles
        const uint32_t idesc_n = ptx::idesc_tf32(128, a.Npad);
        const uint32_t idesc_2n = ptx::idesc_tf32(128, 2 * a.Npad);
        int stage = 0, buf = 0, mks = 0;
        uint32_t phase = 0, tphase = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tempty_bar[buf], tphase ^ 1);
            ptx::tc_fence_after();
            const uint32_t dbase = tmem + (uint32_t)(buf * MT * a.acc_cols);
            for (int ks = 0, kin = 0; ks < a.n_ks; ++ks) {
                uint32_t bhi;
                if (STREAM) {
                    if (kin == 0) {  // first K-step of a weight unit
                        request_next();
                        ptx::mbar_wait(&wfull[wb], wph);
                    }
                    bhi = wsm_addr + (uint32_t)wb * a.unit_bytes + (uint32_t)kin * ks_bytes;
                } else {
                    // resident: all units were requested up front into consecutive buffers
                    if (unit < units_per_tile && kin == 0) ptx::mbar_wait(&wfull[unit], 0);
                    bhi = wsm_addr + (uint32_t)ks * ks_bytes;
                }
                const uint64_t dhi = ptx::smem_desc(bhi, 128, 256);
                const uint64_t dlo = ptx::smem_desc(bhi + (uint32_t)a.Npad * 32, 128, 256);
                const uint32_t sbase = a_base + (uint32_t)(stage * MT * 16);
                const uint32_t acc = ks > 0;
                TC_TRACE(a, mks, 5, lane == 0);
                ptx::mbar_wait(&full_bar[stage], phase);
                ptx::tc_fence_after();
                TC_TRACE(a, mks, 6, lane == 0);
                if (ptx::elect_one()) {
                    for (int mt = 0; mt < MT; ++mt) {
                        const uint32_t ahi = sbase + mt * 16, alo = ahi + 8;
                        const uint32_t d = dbase + (uint32_t)(mt * a.acc_cols);
                        if (STACKED) {
                            ptx::mma_tf32_ts(d, ahi, dhi, idesc_2n, acc);
                            ptx::mma_tf32_ts(d, alo, dhi, idesc_n, 1);
                        } else {
                            ptx::mma_tf32_ts(d, ahi, dhi, idesc_n, acc);
                            ptx::mma_tf32_ts(d, ahi, dlo, idesc_n, 1);
                            ptx::mma_tf32_ts(d, alo, dhi, idesc_n, 1);
                        }
                    }
                    ptx::mma_commit(&empty_bar[stage]);
                    if (STREAM && kin == a.l - 1) ptx::mma_commit(&wempty[wb]);
                }
                __syncwarp();
                if (STREAM || unit < units_per_tile) {
                    if (++kin == a.l) {
                        kin = 0;
                        ++unit;
                        if (++wb == a.nwb) {
                            wb = 0;
                            wph ^= 1;
                        }
                    }
                }
                TC_TRACE(a, mks, 7, lane == 0);
                ++mks;
                if (++stage == a.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(&tfull_bar[buf]);
            __syncwarp();
            if (++buf == 2) {
                buf = 0;
                tphase ^= 1;
            }
        }
    } else {
        // ============================ epilogue ============================
        const int q = warp & 3, half = warp >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const long long ostride = (long long)a.Ho * a.Wo;
        int buf = 0;
        uint32_t tphase = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            int img, u0, v0;
            tc_tile_origin(a, tile, img, u0, v0);
            const int col = v0 + lane;
            ptx::mbar_wait_sleep(&tfull_bar[buf], tphase);
            ptx::tc_fence_after();
            const long long img_off = (long long)img * a.Q * ostride;
            for (int mt = half; mt < MT; mt += 2) {
                const int row = u0 + 4 * mt + q;
                const bool inside = row < a.Ho && col < a.Wo;
                const uint32_t dcol = tmem + lane_off + (uint32_t)((buf * MT + mt) * a.acc_cols);
                for (int o0 = 0; o0 < a.Npad; o0 += 16) {
                    uint32_t r[16], r2[16];
                    ptx::tmem_ld16(dcol + o0, r);
                    if (STACKED) ptx::tmem_ld16(dcol + a.Npad + o0, r2);
                    const long long off0 = img_off + (long long)o0 * ostride +
                                           (long long)row * a.Wo + col;
                    const int nq = min(16, a.Q - o0);
                    // gate / bias operands fetched while the TMEM loads are in flight
                    float aux[16];
                    if (BWD) {
#pragma unroll
                        for (int t = 0; t < 16; ++t)
                            aux[t] = (a.gate && inside && t < nq)
                                         ? __ldg(a.gate + off0 + t * ostride) : 0.f;
                    } else {
#pragma unroll
                        for (int t = 0; t < 16; ++t) aux[t] = t < nq ? __ldg(a.bias + o0 + t) : 0.f;
                    }
                    ptx::tmem_wait_ld();
                    if (!inside) continue;
#pragma unroll
                    for (int t = 0; t < 16; ++t) {
                        if (t >= nq) break;
                        float val = __uint_as_float(r[t]);
                        if (STACKED) val += __uint_as_float(r2[t]);
                        if (!BWD)
                            val = tc_act(val + aux[t], a.act);
                        else if (a.gate)
                            val = gate_from_output(val, aux[t], a.gate_kind);
                        a.out[off0 + t * ostride] = val;
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty_bar[buf]);
            if (++buf == 2) {
                buf = 0;
                tphase ^= 1;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == TC_MMA_WARP) ptx::tmem_dealloc<512>(tmem);
}

// --------------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------------
struct TcPlan {
    int Npad, n_rc, n_ks, MT, acc_cols, stages, nwb;
    bool stacked, resident;
    size_t wbytes, unit_bytes;
    // halo geometry for the chosen MT
    int hrows, hcols, RB, RS, CB, CS, HB;
    size_t hbytes;
};

// halo buffer geometry for M tiles MT: per axis the full halo or only the l tap blocks,
// whichever is smaller
static void tc_halo(TcPlan &p, int l, int d) {
    const int rh = 4 * p.MT + (l - 1) * d, rt = l * 4 * p.MT;
    if (rh <= rt) {
        p.hrows = rh;
        p.RB = rh;
        p.RS = d;
    } else {
        p.hrows = rt;
        p.RB = 4 * p.MT;
        p.RS = 4 * p.MT;
    }
    const int ch = 32 + (l - 1) * d, ct = l * 32;
    if (ch <= ct) {
        p.hcols = ch;
        p.CB = ch;
        p.CS = d;
    } else {
        p.hcols = ct;
        p.CB = 32;
        p.CS = 32;
    }
    p.hbytes = ((size_t)8 * p.hrows * p.hcols * 4 + 127) / 128 * 128;
}

// TMEM budget (512 columns): 2 * MT * acc_cols accumulator columns + stages * MT * 16
// A columns, with stages >= TC_MIN_STAGES; shared memory: packed weights + 2-3 halo
// buffers.  DP_TC_MT caps the M tiles per CTA tile.
static TcPlan tc_plan(int R, int Q, int l, int d) {
    TcPlan p;
    p.Npad = (Q + 15) / 16 * 16;
    p.n_rc = (R + 7) / 8;
    p.n_ks = p.n_rc * l * l;
    p.stacked = p.Npad <= 16;
    p.acc_cols = p.stacked ? 2 * p.Npad : p.Npad;
    p.wbytes = ((size_t)p.n_ks * p.Npad * 64 + 127) / 128 * 128;
    p.unit_bytes = (size_t)l * p.Npad * 64;  // one (channel chunk, tap row); multiple of 128
    int want = TC_MAX_MT;
    if (const char *e = getenv("DP_TC_MT")) {
        int v = atoi(e);
        if (v >= 1 && v <= TC_MAX_MT) want = v;
    }
    p.MT = 0;
    p.stages = 0;
    for (int mt = want; mt >= 1; --mt) {
        int acc_total = 2 * mt * p.acc_cols;
        int st = (512 - acc_total) / (mt * 16);
        if (st > TC_MAX_STAGES) st = TC_MAX_STAGES;
        TcPlan t = p;
        t.MT = mt;
        tc_halo(t, l, d);
        const int units = p.n_rc * l;
        const bool res = units <= TC_MAX_WB &&
                         (size_t)units * p.unit_bytes + 2 * t.hbytes <= (size_t)TC_SMEM_BUDGET;
        const size_t wring = (size_t)(res ? units : TC_WB) * p.unit_bytes;
        if (acc_total < 512 && st >= TC_MIN_STAGES && t.hcols <= 32 * TC_LC &&
            t.hrows <= TC_MAX_HROWS && wring + 2 * t.hbytes <= (size_t)TC_SMEM_BUDGET) {
            p = t;
            p.stages = st;
            p.resident = res;
            p.nwb = res ? units : TC_WB;
            p.HB = wring + 3 * t.hbytes <= (size_t)TC_SMEM_BUDGET ? 3 : 2;
            break;
        }
    }
    if (p.MT == 0) {
        p.MT = 1;
        tc_halo(p, l, d);
        p.MT = 0;
    }
    return p;
}

size_t tc_conv_workspace(int R, int Q, int l) {
    return ((size_t)(R + 7) / 8 * l * l * ((Q + 15) / 16 * 16) * 64 + 127) / 128 * 128;
}

bool tc_conv_supported(int R, int Q, int l, int d) {
    if (tf_conv_supported(R, Q, l, d)) return true;
    TcPlan p = tc_plan(R, Q, l, d);
    return p.Npad <= 128 && p.MT >= 1;
}

static int g_num_sms = 0;
static unsigned long long *g_tc_trace = nullptr;

// debugging aid (tools/tc_trace.py): the last traced launch's timestamps
int tc_trace_copy(void *host, size_t bytes) {
    if (!g_tc_trace) return DP_ERR_ARG;
    if (bytes > 1024 * 8 * 8) bytes = 1024 * 8 * 8;
    return cudaMemcpy(host, g_tc_trace, bytes, cudaMemcpyDeviceToHost) == cudaSuccess
               ? DP_OK
               : DP_ERR_CUDA;
}

// zeroed 1024 x 8 stamp buffer shared by both conv kernels' DP_TC_TRACE modes
unsigned long long *tc_trace_buffer(cudaStream_t st) {
    static unsigned long long *buf = nullptr;
    if (!buf && cudaMalloc(&buf, 1024 * 8 * 8) != cudaSuccess) buf = nullptr;
    if (buf) cudaMemsetAsync(buf, 0, 1024 * 8 * 8, st);
    g_tc_trace = buf;
    return buf;
}

static int launch_tc(const float *in, const float *w, const float *bias, float *out,
                     const float *gate, int n, int R, int Hin, int Win, int Q, int Ho, int Wo,
                     int l, int d, int pad, int act, int gate_kind, bool bwd, void *ws,
                     size_t ws_bytes, cudaStream_t st) {
    TcPlan p = tc_plan(R, Q, l, d);
    if (!(p.Npad <= 128 && p.MT >= 1))
        return set_error(DP_ERR_UNSUPPORTED,
                         "tensor-core conv: weights (%zu B) + halo buffers exceed shared "
                         "memory (R=%d Q=%d k=%d d=%d)",
                         p.wbytes, R, Q, l, d);
    if (ws == nullptr || ws_bytes < p.wbytes)
        return set_error(DP_ERR_ARG, "tensor-core conv: workspace %zu < %zu bytes", ws_bytes,
                         p.wbytes);
    if (((uintptr_t)ws & 15) != 0)
        return set_error(DP_ERR_ARG, "tensor-core conv: workspace must be 16-byte aligned");
    float *wp = (float *)ws;
    int total = p.n_ks * 2 * p.Npad * 8;
    tc_pack_weights<<<ceil_div(total, 256), 256, 0, st>>>(w, wp, Q, R, l, p.Npad, p.n_rc, p.n_ks,
                                                          bwd ? 1 : 0, 0);
    int rc = check_launch("tc_pack_weights");
    if (rc) return rc;
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    // fewer M tiles per CTA tile when the image is short (less padding waste)
    const int rows_needed = (Ho + 3) / 4;
    if (p.MT > rows_needed) {
        p.MT = rows_needed;
        tc_halo(p, l, d);
        p.HB = (size_t)p.nwb * p.unit_bytes + 3 * p.hbytes <= (size_t)TC_SMEM_BUDGET ? 3 : 2;
    }
    TcConvArgs a;
    a.in = in;
    a.wpack = wp;
    a.bias = bias;
    a.out = out;
    a.gate = gate;
    a.R = R;
    a.Hin = Hin;
    a.Win = Win;
    a.Q = Q;
    a.Ho = Ho;
    a.Wo = Wo;
    a.l = l;
    a.d = d;
    a.pad = pad;
    a.act = act;
    a.gate_kind = gate_kind;
    a.n_rc = p.n_rc;
    a.n_ks = p.n_ks;
    a.Npad = p.Npad;
    a.MT = p.MT;
    a.stages = p.stages;
    a.acc_cols = p.acc_cols;
    a.tiles_x = ceil_div(Wo, 32);
    a.tiles_y = ceil_div(Ho, 4 * a.MT);
    long long tt = (long long)n * a.tiles_x * a.tiles_y;
    if (tt > 0x7fffffff) return set_error(DP_ERR_UNSUPPORTED, "tensor-core conv: too many tiles");
    a.total_tiles = (int)tt;
    a.wbytes = (uint32_t)p.wbytes;
    a.unit_bytes = (uint32_t)p.unit_bytes;
    a.nwb = p.nwb;
    a.resident = p.resident ? 1 : 0;
    a.hrows = p.hrows;
    a.hcols = p.hcols;
    a.RB = p.RB;
    a.RS = p.RS;
    a.CB = p.CB;
    a.CS = p.CS;
    a.hbytes = (uint32_t)p.hbytes;
    a.HB = p.HB;
    a.trace = nullptr;
    if (getenv("DP_TC_TRACE")) a.trace = tc_trace_buffer(st);
    int grid = a.total_tiles < g_num_sms ? a.total_tiles : g_num_sms;
    size_t smem = (size_t)p.nwb * p.unit_bytes + (size_t)p.HB * p.hbytes;
    void (*kern)(const TcConvArgs);
    if (p.resident) {
        if (p.stacked)
            kern = bwd ? tc_conv_kernel<true, true, false> : tc_conv_kernel<true, false, false>;
        else
            kern = bwd ? tc_conv_kernel<false, true, false> : tc_conv_kernel<false, false, false>;
    } else {
        if (p.stacked)
            kern = bwd ? tc_conv_kernel<true, true, true> : tc_conv_kernel<true, false, true>;
        else
            kern = bwd ? tc_conv_kernel<false, true, true> : tc_conv_kernel<false, false, true>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tc_conv: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    kern<<<grid, TC_THREADS, smem, st>>>(a);
    return check_launch("tc_conv_kernel");
}

size_t tc_conv_fwd_workspace(int n, int cin, int h, int wd, int cout, int k, int d) {
    const int e = (k - 1) * d + 1;
    const size_t t = tt_conv_workspace(n, cin, h, wd, cout, k, d, 0, h - e + 1, wd - e + 1);
    const size_t w = tc_conv_workspace(cin, cout, k);
    // the flat kernel's TMA-fed forward (relayout planes) where the tap-stacked one is not used
    // (also when the tap kernel applies: it declines shapes at launch, see tt_launch)
    const size_t f =
        tf_relayout_workspace(n, cin, h, wd, cout, k, d, 0, h - e + 1, wd - e + 1, false);
    size_t m = t > w ? t : w;
    return f > m ? f : m;
}

size_t tc_conv_bwd_workspace(int n, int cout, int ho, int wo, int cin, int k, int d) {
    const int e = (k - 1) * d + 1;
    const size_t t = tt_conv_workspace(n, cout, ho, wo, cin, k, d, e - 1, ho + e - 1, wo + e - 1);
    const size_t w = tc_conv_workspace(cout, cin, k);
    const size_t f = tf_relayout_workspace(n, cout, ho, wo, cin, k, d, e - 1, ho + e - 1,
                                           wo + e - 1, true);
    size_t m = t > w ? t : w;
    return f > m ? f : m;
}

int tc_conv_forward(const float *x, const float *w, const float *b, float *y, int n, int cin,
                    int h, int wd, int cout, int k, int d, int act, void *ws, size_t ws_bytes,
                    cudaStream_t st, int flags) {
    const bool f16 = (flags & DP_FAST_INPUT_FP16_RANGE) != 0;
    {
        const int e = (k - 1) * d + 1;
        const size_t t = tt_conv_workspace(n, cin, h, wd, cout, k, d, 0, h - e + 1, wd - e + 1);
        if (t && ws_bytes >= t)
            return tt_launch(x, w, b, y, nullptr, n, cin, h, wd, cout, h - e + 1, wd - e + 1, k,
                             d, 0, act, 0, false, ws, ws_bytes, st, f16);
    }
    if (tf_conv_supported(cin, cout, k, d))
        return tf_conv_forward(x, w, b, y, n, cin, h, wd, cout, k, d, act, ws, ws_bytes, st,
                               f16 ? (flags & 3) : 0);
    int e = (k - 1) * d + 1;
    return launch_tc(x, w, b, y, nullptr, n, cin, h, wd, cout, h - e + 1, wd - e + 1, k, d, 0, act,
                     0, false, ws, ws_bytes, st);
}

int tc_conv_backward_data(const float *dy, const float *w, float *dx, int n, int cout, int ho,
                          int wo, int cin, int k, int d, const float *gate, int gate_kind,
                          void *ws, size_t ws_bytes, cudaStream_t st) {
    {
        const int e = (k - 1) * d + 1;
        const size_t t =
            tt_conv_workspace(n, cout, ho, wo, cin, k, d, e - 1, ho + e - 1, wo + e - 1);
        if (t && ws_bytes >= t)
            return tt_launch(dy, w, nullptr, dx, gate, n, cout, ho, wo, cin, ho + e - 1,
                             wo + e - 1, k, d, e - 1, 0, gate_kind, true, ws, ws_bytes, st);
    }
    if (tf_conv_supported(cout, cin, k, d))
        return tf_conv_backward_data(dy, w, dx, n, cout, ho, wo, cin, k, d, gate, gate_kind, ws,
                                     ws_bytes, st);
    int e = (k - 1) * d + 1;
    return launch_tc(dy, w, nullptr, dx, gate, n, cout, ho, wo, cin, ho + e - 1, wo + e - 1, k, d,
                     e - 1, 0, gate_kind, true, ws, ws_bytes, st);
}

}  // namespace dp
