// d-regularly sparse convolution on the tcgen05 tensor cores with the column taps of a tap
// row stacked into N ("tap-stacked" flat implicit GEMM, fast tier, 3xTF32).
//
// Same maths and argument meaning as tc_conv_flat.cu (reference _kernels.pyx:23-53 forward,
// :56-91 data gradient).  On the virtual (zero-padded) input grid of width Wv output pixel
// (u, v) is p = u*Wv + v and tap (i, j) reads input record p + i*d*Wv + j*d.  The flat kernel
// reads one 128-record A window per TAP; here one window per TAP ROW serves all l taps:
//   D'[r, (j, o)] = sum_c A[s + r, c] * W[o, c, i, j]     (N = l * QS columns, rounded to 16)
// and the epilogue forms y[s + r] = sum_j D'[r + j*d, (j, o)].  The MT M tiles of a CTA tile
// are contiguous (record offsets 0, 128, ...): rows past 128 come from the next tile's TMEM
// accumulator through the epilogue's shared-memory exchange, so a CTA tile of MT*128 rows
// yields MT*128 - (l-1)*d outputs (round 1 overlapped every M tile by (l-1)d rows: c3's head,
// d = 8, l = 7, wasted 48 of 128 MMA rows).  Per tap row and M tile the
// tensor core reads A_hi twice and A_lo once (three N = LN MMAs: A_hi W_hi, A_hi W_lo,
// A_lo W_hi) instead of 2*l times -- the flat kernel's limiter was exactly these A reads.
// QS, the column stride of one tap in N, is Q rounded to 16 -- or to 8 when Q <= 8 (the
// 8-class heads): c3's head (l = 7, Q = 8) then has N = 64 instead of 112, half the B reads
// and TMEM columns per M tile, so 4 instead of 2 M tiles share a CTA tile's weight rows.
//
// Input records come from tc_relayout: per (image, channel chunk of 8) four planes
// [hi c0-3 | hi c4-7 | lo c0-3 | lo c4-7] of 16-byte records over the whole virtual grid
// (zero padding materialised, lo = x - trunc_tf32(x) precomputed), so a unit's A windows
// are plain contiguous ranges: one bulk async copy per (tap row, plane).
//
// Per CTA (persistent, one per SM, 6 warps):
//   warp 4   producer: per unit (tile, chunk, TR tap rows) 4*TR record copies + the unit's
//            packed weights ([tap row][B_hi (LN rows) | B_lo]), one expect_tx;
//   warp 5   MMA issuer: TR * MT * 3 MMAs per unit, one commit frees the unit buffer, one
//            commit per tile hands the accumulators (double-buffered) to the epilogue;
//   warps 0-3 epilogue, one per TMEM lane quarter: per 16-channel chunk and tap j,
//            tcgen05.ld, exchange through shared memory to fetch row r + j*d, accumulate;
//            bias + nonlinearity (forward) or the upstream derivative (data gradient).
#include <stdlib.h>

#include "dp_common.cuh"
#include "tc_ptx.cuh"

namespace dp {

constexpr int TT_EPI_WARPS = 4;
constexpr int TT_PROD_WARP = 4;
constexpr int TT_MMA_WARP = 5;
constexpr int TT_THREADS = 6 * 32;
constexpr int TT_MAX_HB = 6;
constexpr int TT_MAX_L = 8;                 // taps per row the epilogue exchange supports
constexpr int TT_SMEM_TOTAL = 222 * 1024;   // unit buffers + epilogue exchange (dynamic)

struct TtArgs {
    const float *xr;     // relayout: [n][n_rc][4 planes][plane_recs] 16-byte records
    const float *wpack;  // [n_rc][l][hi|lo][LN x 8] core-matrix layout
    const float *bias;
    float *out;          // (n, Q, Ho, Wo)
    const float *gate;
    int n_rc, l, d, Q, Npad, QS, LN, MT, S, NR, TR, n_tr;
    int STEP, XR;          // outputs per CTA tile (MT*128 - (l-1)d), exchange rows (128 + (l-1)d)
    const int *exit_if;    // fp16 launch: exit when the range flag is set (tf32 fallback runs)
    int Wv, Ho, Wo, act, gate_kind;
    long long plane_recs;
    int flat_len, tiles_per_img, total_tiles, HB;
    uint32_t seg_bytes;    // NR * 16
    uint32_t wrow_bytes;   // one tap row of packed weights: 2 * LN * 32
    uint32_t ubytes;       // unit buffer
    uint32_t xoff;         // epilogue exchange area: [l][8 or 16][XR] floats after the units
};

__device__ __forceinline__ float tt_act(float v, int kind) {
    if (kind == DP_TANH || kind == DP_TANH_FAST) return tanhf(v);
    if (kind == DP_RELU) return dp_relu(v);
    return v;
}

// HALF (forward only): fp16-split records / weights and kind::f16 MMAs (K = 16 channels per
// K step, same byte geometry as the tf32 records) -- half the record and weight feed
template <bool BWD, bool HALF = false>
__global__ void __launch_bounds__(TT_THREADS, 1) tc_conv_tap_kernel(const TtArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint64_t ufull[TT_MAX_HB], uempty[TT_MAX_HB], tfull[2], tempty[2];
    __shared__ uint32_t s_tmem;
    __shared__ float s_bias[256];
    // epilogue exchange (dynamic): [tap j][XC columns][XR = 128 + (l-1)d rows: the tile's own
    // D' rows, then the next M tile's first (l-1)d rows]
    float *s_x = reinterpret_cast<float *>(smem_raw + a.xoff);

    if (a.exit_if && *(volatile const int *)a.exit_if) return;  // uniform, before any barrier
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int MT = a.MT;
    const int units = a.n_rc * a.n_tr;
    for (int o = threadIdx.x; o < a.Npad; o += blockDim.x)
        s_bias[o] = (!BWD && o < a.Q) ? a.bias[o] : 0.f;
    const int XC = a.QS == 8 ? 8 : 16;  // exchange columns per tap
    const int XR = a.XR, halo = a.XR - 128;
    for (int e = threadIdx.x; e < a.l * XC * halo; e += blockDim.x)
        s_x[(e / halo) * XR + 128 + e % halo] = 0.f;
    if (threadIdx.x == 0) {
        for (int b = 0; b < a.HB; ++b) {
            ptx::mbar_init(&ufull[b], 1);
            ptx::mbar_init(&uempty[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], TT_EPI_WARPS);
        }
        ptx::mbar_fence_init();
    }
    if (warp == TT_MMA_WARP) ptx::tmem_alloc<512>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == TT_PROD_WARP) {
        // ================================ producer ================================
        if (lane == 0) {
            const unsigned char *xr = reinterpret_cast<const unsigned char *>(a.xr);
            const unsigned char *wsrc = reinterpret_cast<const unsigned char *>(a.wpack);
            int b = 0;
            uint32_t uph = 0;
            for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
                const int img = tile / a.tiles_per_img;
                const int f0 = (tile - img * a.tiles_per_img) * a.STEP;
                for (int rc = 0; rc < a.n_rc; ++rc) {
                    const unsigned char *pl =
                        xr + ((size_t)img * a.n_rc + rc) * 4 * a.plane_recs * 16;
                    for (int i0 = 0; i0 < a.l; i0 += a.TR) {
                        const int ntr = min(a.TR, a.l - i0);
                        ptx::mbar_wait(&uempty[b], uph ^ 1);
                        unsigned char *ub = smem_raw + (size_t)b * a.ubytes;
                        ptx::mbar_expect_tx(&ufull[b], (uint32_t)ntr * (4 * a.seg_bytes + a.wrow_bytes));
                        for (int t = 0; t < ntr; ++t) {
                            const long long rec0 = f0 + (long long)(i0 + t) * a.d * a.Wv;
                            for (int p = 0; p < 4; ++p)
                                ptx::bulk_g2s(ub + (size_t)(t * 4 + p) * a.seg_bytes,
                                              pl + ((size_t)p * a.plane_recs + rec0) * 16,
                                              a.seg_bytes, &ufull[b]);
                        }
                        const unsigned char *ws =
                            wsrc + ((size_t)rc * a.l + i0) * a.wrow_bytes;
                        const uint32_t wb = (uint32_t)ntr * a.wrow_bytes;
                        unsigned char *wd = ub + (size_t)a.TR * 4 * a.seg_bytes;
                        for (uint32_t off = 0; off < wb; off += 32768u)
                            ptx::bulk_g2s(wd + off, ws + off, wb - off < 32768u ? wb - off : 32768u,
                                          &ufull[b]);
                        if (++b == a.HB) {
                            b = 0;
                            uph ^= 1;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == TT_MMA_WARP) {
        // ================================ MMA issuer ================================
        const uint32_t sb = ptx::smem_u32(smem_raw);
        const uint32_t idesc = HALF ? ptx::idesc_f16(128, a.LN) : ptx::idesc_tf32(128, a.LN);
        const uint32_t lo_units = (2 * a.seg_bytes) >> 4;
        const uint32_t blo_units = (uint32_t)(a.LN * 32) >> 4;
        int b = 0, buf = 0;
        uint32_t uph = 0, tph = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tempty[buf], tph ^ 1);
            ptx::tc_fence_after();
            const uint32_t dbase = tmem + (uint32_t)(buf * MT * a.LN);
            for (int u = 0, i0 = 0; u < units; ++u) {
                const int ntr = min(a.TR, a.l - i0);
                ptx::mbar_wait(&ufull[b], uph);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t ub = sb + (uint32_t)b * a.ubytes;
                    const uint32_t wb = ub + (uint32_t)a.TR * 4 * a.seg_bytes;
                    for (int t = 0; t < ntr; ++t) {
                        const uint64_t a0 = ptx::smem_desc(ub + (uint32_t)t * 4 * a.seg_bytes,
                                                           a.seg_bytes, 128);
                        const uint64_t bh = ptx::smem_desc(wb + (uint32_t)t * a.wrow_bytes, 128, 256);
                        const uint32_t acc0 = (u | t) != 0;
                        for (int mt = 0; mt < MT; ++mt) {
                            const uint64_t ad = a0 + (uint64_t)(mt * 128);
                            const uint32_t dd = dbase + (uint32_t)(mt * a.LN);
                            if (HALF) {
                                ptx::mma_f16_ss(dd, ad, bh, idesc, acc0);
                                ptx::mma_f16_ss(dd, ad, bh + blo_units, idesc, 1);
                                ptx::mma_f16_ss(dd, ad + lo_units, bh, idesc, 1);
                            } else {
                                ptx::mma_tf32_ss(dd, ad, bh, idesc, acc0);
                                ptx::mma_tf32_ss(dd, ad, bh + blo_units, idesc, 1);
                                ptx::mma_tf32_ss(dd, ad + lo_units, bh, idesc, 1);
                            }
                        }
                    }
                    ptx::mma_commit(&uempty[b]);
                }
                __syncwarp();
                if (++b == a.HB) {
                    b = 0;
                    uph ^= 1;
                }
                i0 += a.TR;
                if (i0 >= a.l) i0 = 0;
            }
            if (ptx::elect_one()) ptx::mma_commit(&tfull[buf]);
            __syncwarp();
            if (++buf == 2) {
                buf = 0;
                tph ^= 1;
            }
        }
    } else {
        // ================================ epilogue ================================
        const int q = warp;  // 0..3 = TMEM lane quarter
        const int r = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const long long ostride = (long long)a.Ho * a.Wo;
        int buf = 0;
        uint32_t tph = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            const int img = tile / a.tiles_per_img;
            const int f0 = (tile - img * a.tiles_per_img) * a.STEP;
            ptx::mbar_wait_sleep(&tfull[buf], tph);
            ptx::tc_fence_after();
            const long long img_off = (long long)img * a.Q * ostride;
            for (int mt = 0; mt < MT; ++mt) {
                // M tiles are contiguous: row r of tile mt needs D rows r + j*d, the ones
                // past 128 from the next tile (its first (l-1)d rows go to the exchange's
                // spill rows); the CTA tile's last (l-1)d rows wait for the next CTA tile
                const int p = f0 + mt * 128 + r;
                const int u = p / a.Wv, v = p - u * a.Wv;
                const bool inside = mt * 128 + r < a.STEP && p < a.flat_len && v < a.Wo;
                // tcgen05.ld is warp-collective: the whole warp loads the next tile's rows
                // when any of its lanes needs them; only lanes r < halo publish them
                const bool spill_w = mt + 1 < MT && q * 32 < halo;
                const bool spill = spill_w && r < halo;
                const long long pix = img_off + (long long)u * a.Wo + v;
                const uint32_t dcol = tmem + lane_off + (uint32_t)((buf * MT + mt) * a.LN);
                const uint32_t ncol = dcol + (uint32_t)a.LN;  // tile mt + 1
                for (int o0 = 0; o0 < a.QS; o0 += 16) {
                    // all l taps' columns of this chunk: l TMEM loads, one wait; publish
                    // rows; one barrier; gather rows r + j*d; one barrier (reuse)
                    float acc[16];
#pragma unroll
                    for (int t = 0; t < 16; ++t) acc[t] = 0.f;
                    // gate operands (data gradient) requested now, consumed after the exchange
                    const long long off0 = pix + (long long)o0 * ostride;
                    const int nq = min(16, a.Q - o0);
                    float aux[16];
#pragma unroll
                    for (int t = 0; t < 16; ++t)
                        aux[t] = (BWD && a.gate && inside && t < nq)
                                     ? __ldg(a.gate + off0 + t * ostride) : 0.f;
#pragma unroll
                    for (int j = 0; j < TT_MAX_L; ++j) {
                        if (j >= a.l) break;
                        uint32_t rv[16], rn[16];
                        float *xs = s_x + j * XC * XR;
                        if (a.QS == 8) {  // one 8-column tap group (never past the allocation)
                            ptx::tmem_ld8(dcol + (uint32_t)(j * 8), rv);
                            if (spill_w) ptx::tmem_ld8(ncol + (uint32_t)(j * 8), rn);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int t = 0; t < 8; ++t) xs[t * XR + r] = __uint_as_float(rv[t]);
                            if (spill) {
#pragma unroll
                                for (int t = 0; t < 8; ++t)
                                    xs[t * XR + 128 + r] = __uint_as_float(rn[t]);
                            }
                        } else {
                            ptx::tmem_ld16(dcol + (uint32_t)(j * a.QS + o0), rv);
                            if (spill_w) ptx::tmem_ld16(ncol + (uint32_t)(j * a.QS + o0), rn);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int t = 0; t < 16; ++t) xs[t * XR + r] = __uint_as_float(rv[t]);
                            if (spill) {
#pragma unroll
                                for (int t = 0; t < 16; ++t)
                                    xs[t * XR + 128 + r] = __uint_as_float(rn[t]);
                            }
                        }
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < TT_MAX_L; ++j) {
                        if (j >= a.l) break;
                        const int rr = r + j * a.d;  // < XR
                        const float *xs = s_x + j * XC * XR + rr;
                        if (a.QS == 8) {
#pragma unroll
                            for (int t = 0; t < 8; ++t) acc[t] += xs[t * XR];
                        } else {
#pragma unroll
                            for (int t = 0; t < 16; ++t) acc[t] += xs[t * XR];
                        }
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (!inside) continue;
#pragma unroll
                    for (int t = 0; t < 16; ++t) {
                        if (t >= nq) break;
                        float val = acc[t];
                        if (!BWD)
                            val = tt_act(val + s_bias[o0 + t], a.act);
                        else if (a.gate)
                            val = gate_from_output(val, aux[t], a.gate_kind);
                        a.out[off0 + t * ostride] = val;
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
            if (++buf == 2) {
                buf = 0;
                tph ^= 1;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == TT_MMA_WARP) ptx::tmem_dealloc<512>(tmem);
}

// NCHW (n, R, Hin, Win) -> per (n, chunk) four planes of 16-byte records over the virtual
// grid (Hv = Hin + 2 pad, Wv = Win + 2 pad; zeros outside the input and past Hv*Wv up to
// plane_recs): [hi c0-3 | hi c4-7 | lo c0-3 | lo c4-7].
__global__ void __launch_bounds__(256) tc_relayout(const float *__restrict__ in,
                                                   float4 *__restrict__ xr, int R, int Hin,
                                                   int Win, int Wv, int pad, int n_rc,
                                                   long long plane_recs, long long vrecs,
                                                   long long total) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long nrc = idx / plane_recs;
        const long long f = idx - nrc * plane_recs;
        const int rc = (int)(nrc % n_rc);
        const long long n = nrc / n_rc;
        float v[8];
        const long long yv = f / Wv;
        const int y = (int)yv - pad, x = (int)(f - yv * Wv) - pad;
        const bool ok = f < vrecs && y >= 0 && y < Hin && x >= 0 && x < Win;
        const float *src = in + ((n * R + rc * 8) * Hin + (ok ? y : 0)) * (long long)Win + (ok ? x : 0);
        const long long cs = (long long)Hin * Win;
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (ok && rc * 8 + k < R) ? __ldg(src + k * cs) : 0.f;
        float4 *dst = xr + nrc * 4 * plane_recs + f;
        dst[0] = make_float4(v[0], v[1], v[2], v[3]);
        dst[plane_recs] = make_float4(v[4], v[5], v[6], v[7]);
        dst[2 * plane_recs] = make_float4(ptx::tf32_lo(v[0]), ptx::tf32_lo(v[1]),
                                          ptx::tf32_lo(v[2]), ptx::tf32_lo(v[3]));
        dst[3 * plane_recs] = make_float4(ptx::tf32_lo(v[4]), ptx::tf32_lo(v[5]),
                                          ptx::tf32_lo(v[6]), ptx::tf32_lo(v[7]));
    }
}

// weights W(q, r, i, j) -> per (chunk rc, tap row i): [hi | lo] tiles of LN rows
// (row n = j*QS + q, zero rows past l*QS) x K = 8 channels, K-major core-matrix layout
// (n>>3)*256 + (k>>2)*128 + (n&7)*16 + (k&3)*4; bwd: W is (R = cout, Q = cin, l, l) rotated.
__global__ void tc_pack_tap(const float *__restrict__ w, float *__restrict__ wp, int Q, int R,
                            int l, int QS, int LN, int n_rc, int bwd) {
    const long long total = (long long)n_rc * l * 2 * LN * 8;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(idx & 7);
        const long long rest = idx >> 3;
        const int n = (int)(rest % LN);
        const long long r2 = rest / LN;
        const int hl = (int)(r2 & 1);
        const long long ri = r2 >> 1;  // rc * l + i
        const int i = (int)(ri % l), rc = (int)(ri / l);
        const int j = n / QS, qo = n - j * QS;
        const int c = rc * 8 + k;
        float v = 0.f;
        if (j < l && qo < Q && c < R) {
            if (!bwd)
                v = w[(((long long)qo * R + c) * l + i) * l + j];
            else
                v = w[(((long long)c * Q + qo) * l + (l - 1 - i)) * l + (l - 1 - j)];
        }
        if (hl) v = ptx::tf32_lo(v);
        const long long byte = (ri * 2 + hl) * (long long)LN * 32 + (n >> 3) * 256 + (k >> 2) * 128 +
                               (n & 7) * 16 + (k & 3) * 4;
        wp[byte / 4] = v;
    }
}

// fp16 forms (HALF): records [hi c0-7 | hi c8-15 | lo c0-7 | lo c8-15] per 16-channel chunk
// SCALED: the offset split (ptx::f16_split2_scaled) for deltas of unknown magnitude
// (compile time: a runtime switch in the conversion loop cost the pass 25 %)
// flag: set (atomicOr) when any element is outside the fp16-split's safe range (|x| >= 2^15)
// or not finite -- the fp16 kernel then exits and the tf32 fallback launched after it runs
// n_rc_do <= n_rc: only the first n_rc_do chunks of every image (the last one may be
// tap-packed by tc_relayout_f16_pk); total = n * n_rc_do * plane_recs
template <bool SCALED>
__global__ void __launch_bounds__(256) tc_relayout_f16(const float *__restrict__ in,
                                                       uint4 *__restrict__ xr, int R, int Hin,
                                                       int Win, int Wv, int pad, int n_rc,
                                                       int n_rc_do, long long plane_recs,
                                                       long long vrecs, long long total,
                                                       int *flag) {
    bool bad = false;
    // 32-bit index math whenever the pass fits it (every config): the 64-bit divides by
    // plane_recs and Wv were a large share of this HBM-bound pass's issue slots
    const bool small = total < 0x7fffffffLL;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        long long nrd, f;
        int yvi;
        if (small) {
            const unsigned ui = (unsigned)idx, pr = (unsigned)plane_recs;
            const unsigned q = ui / pr;
            nrd = q;
            f = ui - q * pr;
            yvi = (int)((unsigned)f / (unsigned)Wv);
        } else {
            nrd = idx / plane_recs;
            f = idx - nrd * plane_recs;
            yvi = (int)(f / Wv);
        }
        const int rc = (int)(nrd % n_rc_do);
        const long long n = nrd / n_rc_do;
        const long long nrc = n * n_rc + rc;
        const int y = yvi - pad, x = (int)(f - (long long)yvi * Wv) - pad;
        const bool ok = f < vrecs && y >= 0 && y < Hin && x >= 0 && x < Win;
        const float *src = in + ((n * R + rc * 16) * Hin + (ok ? y : 0)) * (long long)Win + (ok ? x : 0);
        const long long cs = (long long)Hin * Win;
        uint32_t hw[8], lw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int c0 = rc * 16 + 2 * q;
            const float v0 = (ok && c0 < R) ? __ldg(src + (2 * q) * cs) : 0.f;
            const float v1 = (ok && c0 + 1 < R) ? __ldg(src + (2 * q + 1) * cs) : 0.f;
            bad |= !(fabsf(v0) < ptx::F16_SPLIT_MAX) || !(fabsf(v1) < ptx::F16_SPLIT_MAX);
            if constexpr (SCALED)
                ptx::f16_split2_scaled(v0, v1, hw[q], lw[q]);
            else
                ptx::f16_split2(v0, v1, hw[q], lw[q]);
        }
        uint4 *dst = xr + nrc * 4 * plane_recs + f;
        dst[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        dst[plane_recs] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
        dst[2 * plane_recs] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        dst[3 * plane_recs] = make_uint4(lw[4], lw[5], lw[6], lw[7]);
    }
    if (bad) atomicOr(flag, 1);
}

template __global__ void tc_relayout_f16<false>(const float *, uint4 *, int, int, int, int, int,
                                                int, int, long long, long long, long long, int *);
template __global__ void tc_relayout_f16<true>(const float *, uint4 *, int, int, int, int, int,
                                               int, int, long long, long long, long long, int *);

// weights W(q, r, i, j) -> per (16-channel chunk rc, tap row i): [hi | lo] tiles of LN rows
// (row n = j*QS + q) x K = 16 halves: element (n, k) at (n>>3)*256 + (k>>3)*128 + (n&7)*16 +
// (k&7)*2 (forward only)
__global__ void tc_pack_tap_f16(const float *__restrict__ w, __half *__restrict__ wp, int Q,
                                int R, int l, int QS, int LN, int n_rc, int *flag) {
    const long long total = (long long)n_rc * l * 2 * LN * 16;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(idx & 15);
        const long long rest = idx >> 4;
        const int n = (int)(rest % LN);
        const long long r2 = rest / LN;
        const int hl = (int)(r2 & 1);
        const long long ri = r2 >> 1;  // rc * l + i
        const int i = (int)(ri % l), rc = (int)(ri / l);
        const int j = n / QS, qo = n - j * QS;
        const int c = rc * 16 + k;
        const float v = (j < l && qo < Q && c < R) ? w[(((long long)qo * R + c) * l + i) * l + j] : 0.f;
        if (!(fabsf(v) < ptx::F16_SPLIT_MAX)) atomicOr(flag, 1);
        __half hi, lo;
        ptx::f16_split(v, hi, lo);
        const long long byte = (ri * 2 + hl) * (long long)LN * 32 + (n >> 3) * 256 + (k >> 3) * 128 +
                               (n & 7) * 16 + (k & 7) * 2;
        wp[byte / 2] = hl ? lo : hi;
    }
}

// --------------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------------
struct TtPlan {
    int Npad, QS, LN, n_rc, MT, S, NR, TR, n_tr, HB, STEP, XR;
    bool ok;
    uint32_t seg_bytes, wrow_bytes, ubytes, xbytes;
    size_t wbytes;
};

static TtPlan tt_plan(int R, int Q, int l, int d, int max_mt, bool half = false) {
    TtPlan p;
    p.ok = false;
    p.Npad = (Q + 15) / 16 * 16;
    p.QS = (Q <= 8 && !getenv("DP_TT_QS16")) ? 8 : p.Npad;
    p.LN = (l * p.QS + 15) / 16 * 16;
    p.n_rc = half ? (R + 15) / 16 : (R + 7) / 8;
    p.S = 128 - (l - 1) * d;
    if (p.LN > 256 || p.S < 32 || p.Npad > 256) return p;
    int mt = 256 / p.LN;
    if (mt > 4) mt = 4;
    if (const char *e = getenv("DP_TT_MT")) {
        int v = atoi(e);
        if (v >= 1 && v < mt) mt = v;
    }
    if (max_mt >= 1 && mt > max_mt) mt = max_mt;
    if (mt < 1) return p;
    p.MT = mt;
    // contiguous M tiles: the MT*128 records of a tap row window give D' rows for MT*128 -
    // (l-1)d outputs (the last (l-1)d rows' sums need the next CTA tile: one overlap per
    // CTA tile instead of one per M tile)
    p.NR = mt * 128;
    p.STEP = mt * 128 - (l - 1) * d;
    p.XR = 128 + (l - 1) * d;
    p.seg_bytes = (uint32_t)p.NR * 16;
    p.wrow_bytes = (uint32_t)(2 * p.LN * 32);
    p.wbytes = (size_t)p.n_rc * l * p.wrow_bytes;
    if (l > TT_MAX_L) return p;
    // tap rows per unit: as many as leave room for 2 unit buffers next to the exchange area
    p.xbytes = (uint32_t)l * (p.QS == 8 ? 8 : 16) * p.XR * 4;
    const size_t budget = (size_t)TT_SMEM_TOTAL - p.xbytes - 2048;
    p.TR = 0;
    int tr_max = l;
    if (const char *e = getenv("DP_TT_TR")) {  // experiments: cap the tap rows per unit
        int v = atoi(e);
        if (v >= 1 && v < tr_max) tr_max = v;
    }
    for (int tr = tr_max; tr >= 1; --tr) {
        const size_t ub = ((size_t)tr * (4 * p.seg_bytes + p.wrow_bytes) + 127) / 128 * 128;
        if (2 * ub <= budget) {
            p.TR = tr;
            p.ubytes = (uint32_t)ub;
            break;
        }
    }
    if (p.TR == 0) return p;
    p.n_tr = (l + p.TR - 1) / p.TR;
    long long hb = (long long)budget / p.ubytes;
    p.HB = (int)(hb > TT_MAX_HB ? TT_MAX_HB : hb);
    p.ok = p.HB >= 2 && (p.seg_bytes >> 4) < (1u << 14);
    return p;
}


// workspace: packed weights, then the relayout planes
static size_t tt_relayout_recs(int Hin, int Win, int pad, int l, int d, const TtPlan &p,
                               long long &plane_recs, int &tiles_per_img, long long &flat_len,
                               int Ho, int Wo) {
    const int Wv = Win + 2 * pad, Hv = Hin + 2 * pad;
    flat_len = (long long)(Ho - 1) * Wv + Wo;
    tiles_per_img = (int)((flat_len + p.STEP - 1) / p.STEP);
    // the last tile's windows reach f0 + (l-1)*d*Wv + NR
    long long need = (long long)(tiles_per_img - 1) * p.STEP + (long long)(l - 1) * d * Wv + p.NR;
    long long vrecs = (long long)Hv * Wv;
    plane_recs = (need > vrecs ? need : vrecs);
    plane_recs = (plane_recs + 7) / 8 * 8;
    return (size_t)plane_recs;
}

size_t tt_conv_workspace(int n, int R, int Hin, int Win, int Q, int l, int d, int pad, int Ho,
                         int Wo) {
    if (getenv("DP_TC_FLAT")) return 0;  // force the flat kernel (experiments)
    TtPlan p = tt_plan(R, Q, l, d, 0);
    if (!p.ok || Ho < 1 || Wo < 1) return 0;
    // Only where it wins (measured, c2 at batch 16, kernel + relayout vs the flat kernel):
    // with >= 3 M tiles per CTA tile the per-tile weight rows and the (l-1)d overlap are
    // amortised (conv3 fwd 213 vs 327 us, conv2 data grad 303 vs 449 us); at MT <= 2 the
    // l*Npad-wide weight rows re-streamed per tile and the 64 B/pixel/tap-row record
    // copies cost more than the saved A reads (conv1/conv2 fwd, conv3 data grad lose).
    // Wide inputs (R >= 32, four or more channel chunks) win even at MT 1-2 (c3 conv2 fwd /
    // data grad 0.74 -> 0.65 / 0.76 -> 0.67 ms, c3 head fwd 1.15 -> 1.03, c4 conv2 fwd and
    // the c4 data grads 5-15 %): there the flat kernel's per-tap-row record loads and hi/lo
    // splits, not the tap kernel's re-streamed weight rows, dominate.
    // DP_TT_ALL uses it wherever it applies (experiments).
    // Round 2 (tools/conv_ab.py, identity epilogue, relayout included): with MT = 1 the wide
    // layers are now slightly faster on the flat kernel (c3 conv2 fwd 2.47 vs 2.50 ms, data
    // grad 2.50 vs 2.60; c4 L2 fwd 1.08 vs 1.23), so wide inputs need MT >= 2 as well.
    if ((p.MT < 3 && R < 32) || p.MT < 2) {
        if (!getenv("DP_TT_ALL")) return 0;
    }
    long long plane_recs, flat_len;
    int tpi;
    tt_relayout_recs(Hin, Win, pad, l, d, p, plane_recs, tpi, flat_len, Ho, Wo);
    const size_t wb = (p.wbytes + 255) / 256 * 256;
    return wb + (size_t)n * p.n_rc * 4 * plane_recs * 16;
}

// the flat kernel's tf32 fallback of an fp16-split launch (tc_conv_flat.cu)
size_t tf_fallback_bytes(int R, int Q, int l, int d, bool bwd);
int tf_fallback(const float *in, const float *w, const float *bias, float *out, const float *gate,
                int n, int R, int Hin, int Win, int Q, int Ho, int Wo, int l, int d, int pad,
                int act, int gate_kind, bool bwd, void *wp, const int *flag, cudaStream_t st);

static int g_tt_sms = 0;

int tt_launch(const float *in, const float *w, const float *bias, float *out, const float *gate,
              int n, int R, int Hin, int Win, int Q, int Ho, int Wo, int l, int d, int pad,
              int act, int gate_kind, bool bwd, void *ws, size_t ws_bytes, cudaStream_t st,
              bool f16_ok) {
    // fp16-split operands for the forward of inputs with >= 16 channels the caller vouches
    // are in fp16 range (DP_FAST_INPUT_FP16_RANGE; DP_TF_HALF=0: tf32); the workspace query
    // stays tf32-sized (a superset)
    const char *he = getenv("DP_TF_HALF");
    bool half = f16_ok && !bwd && R >= 16 && !(he && he[0] == '0');
    const size_t fb_bytes = half ? tf_fallback_bytes(R, Q, l, d, false) : 0;
    if (half && fb_bytes == 0) half = false;
    TtPlan p = tt_plan(R, Q, l, d, 0, half);
    if (!p.ok)
        return set_error(DP_ERR_UNSUPPORTED, "tap-stacked conv: unsupported (R=%d Q=%d k=%d d=%d)",
                         R, Q, l, d);
    long long plane_recs, flat_len;
    int tiles_per_img;
    tt_relayout_recs(Hin, Win, pad, l, d, p, plane_recs, tiles_per_img, flat_len, Ho, Wo);
    if (half && (size_t)((p.wbytes + 255) / 256 * 256) + (size_t)n * p.n_rc * 4 * plane_recs * 16 +
                        256 + fb_bytes > ws_bytes) {  // no room for the fp16 layout: tf32
        half = false;
        p = tt_plan(R, Q, l, d, 0, false);
        tt_relayout_recs(Hin, Win, pad, l, d, p, plane_recs, tiles_per_img, flat_len, Ho, Wo);
    }
    const size_t wb = (p.wbytes + 255) / 256 * 256;
    const size_t planes = (size_t)n * p.n_rc * 4 * plane_recs * 16;
    // fp16: [weights | planes | range flag (256 B) | the flat tf32 fallback's weights]
    const size_t need = wb + planes + (half ? 256 + fb_bytes : 0);
    if (ws == nullptr || ws_bytes < need)
        return set_error(DP_ERR_ARG, "tap-stacked conv: workspace %zu < %zu bytes", ws_bytes, need);
    if (((uintptr_t)ws & 255) != 0)
        return set_error(DP_ERR_ARG, "tap-stacked conv: workspace must be 256-byte aligned");
    if (flat_len > 0x7fffffffLL || plane_recs > 0x7fffffffLL)
        return set_error(DP_ERR_UNSUPPORTED, "tap-stacked conv: image too large");
    float *wp = (float *)ws;
    float4 *xr = (float4 *)((unsigned char *)ws + wb);
    int *flag = half ? (int *)((unsigned char *)ws + wb + planes) : nullptr;
    if (half && cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tap-stacked conv: flag reset failed");
    {
        const long long total = (long long)p.n_rc * l * 2 * p.LN * 8;
        long long g = (total + 255) / 256;
        if (half)
            tc_pack_tap_f16<<<(int)(g < 4096 ? g : 4096), 256, 0, st>>>(w, (__half *)wp, Q, R, l,
                                                                        p.QS, p.LN, p.n_rc, flag);
        else
            tc_pack_tap<<<(int)(g < 4096 ? g : 4096), 256, 0, st>>>(w, wp, Q, R, l, p.QS, p.LN,
                                                                    p.n_rc, bwd ? 1 : 0);
        int rc = check_launch("tc_pack_tap");
        if (rc) return rc;
    }
    {
        const int Wv = Win + 2 * pad;
        const long long vrecs = (long long)(Hin + 2 * pad) * Wv;
        const long long total = (long long)n * p.n_rc * plane_recs;
        long long g = (total + 255) / 256;
        if (half)
            tc_relayout_f16<false><<<(int)(g < 148 * 64 ? g : 148 * 64), 256, 0, st>>>(
                in, (uint4 *)xr, R, Hin, Win, Wv, pad, p.n_rc, p.n_rc, plane_recs, vrecs, total,
                flag);
        else
            tc_relayout<<<(int)(g < 148 * 64 ? g : 148 * 64), 256, 0, st>>>(
                in, xr, R, Hin, Win, Wv, pad, p.n_rc, plane_recs, vrecs, total);
        int rc = check_launch("tc_relayout");
        if (rc) return rc;
    }
    if (g_tt_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_tt_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_tt_sms <= 0) g_tt_sms = 148;
    }
    TtArgs a;
    a.xr = (const float *)xr;
    a.wpack = wp;
    a.bias = bias;
    a.out = out;
    a.gate = gate;
    a.n_rc = p.n_rc;
    a.l = l;
    a.d = d;
    a.Q = Q;
    a.Npad = p.Npad;
    a.QS = p.QS;
    a.LN = p.LN;
    a.MT = p.MT;
    a.S = p.S;
    a.STEP = p.STEP;
    a.XR = p.XR;
    a.exit_if = flag;
    a.NR = p.NR;
    a.TR = p.TR;
    a.n_tr = p.n_tr;
    a.Wv = Win + 2 * pad;
    a.Ho = Ho;
    a.Wo = Wo;
    a.act = act;
    a.gate_kind = gate_kind;
    a.plane_recs = plane_recs;
    a.flat_len = (int)flat_len;
    a.tiles_per_img = tiles_per_img;
    const long long tt = (long long)n * tiles_per_img;
    if (tt > 0x7fffffff) return set_error(DP_ERR_UNSUPPORTED, "tap-stacked conv: too many tiles");
    a.total_tiles = (int)tt;
    a.HB = p.HB;
    a.seg_bytes = p.seg_bytes;
    a.wrow_bytes = p.wrow_bytes;
    a.ubytes = p.ubytes;
    if (a.total_tiles == 0) return DP_OK;
    const int grid = a.total_tiles < g_tt_sms ? a.total_tiles : g_tt_sms;
    a.xoff = (uint32_t)p.HB * p.ubytes;
    const size_t smem = (size_t)a.xoff + p.xbytes;
    void (*kern)(const TtArgs) = bwd    ? tc_conv_tap_kernel<true>
                                 : half ? tc_conv_tap_kernel<false, true>
                                        : tc_conv_tap_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tc_conv_tap: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    kern<<<grid, TT_THREADS, smem, st>>>(a);
    const int rc = check_launch("tc_conv_tap_kernel");
    if (rc || !half) return rc;
    // fp16 operands out of range (flag set): the flat tf32 kernel redoes the layer
    return tf_fallback(in, w, bias, out, gate, n, R, Hin, Win, Q, Ho, Wo, l, d, pad, act,
                       gate_kind, false, (unsigned char *)ws + wb + planes + 256, flag, st);
}

}  // namespace dp
