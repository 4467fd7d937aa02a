// d-regularly sparse convolution on the tcgen05 tensor cores as a FLATTENED implicit GEMM
// with both operands read by the tensor core from shared memory (fast tier, 3xTF32).
//
// Same maths and argument meaning as tc_conv.cu / conv_direct.cu:
//   forward        y[o,u,v]  = b[o] + sum_{c,i,j} w[o,c,i,j] * x[c, u+i*d, v+j*d]
//   data gradient  dx[c,y,x] = sum_{o,i,j} w[o,c,l-1-i,l-1-j] * dy_pad[o, y+i*d, x+j*d]
// (reference _kernels.pyx:23-53 and :56-91).
//
// Flattening: on the (virtual, zero-padded) input grid of width Wv an output pixel (u, v)
// is the flat index p = u*Wv + v, and tap (i, j) reads input flat index p + i*d*Wv + j*d.
// 128 consecutive output flat indices are therefore 128 consecutive input records for
// every tap, so one M=128 tile of the GEMM (M = pixels, N = output channels, K = 8
// channels of one tap) is a plain shared-memory window -- no per-tap re-layout.  The
// flat range covers the (l-1)*d wrap columns at the end of each row too; those outputs
// are computed and discarded (waste (l-1)d / Wv, ~3% at 256-pixel rows).
//
// Shared-memory operand layouts (K-major, SWIZZLE_NONE core matrices):
//   A (pixels): one halo unit = 4 planes [hi c0-3 | hi c4-7 | lo c0-3 | lo c4-7] of NR
//       16-byte records (4 channels of one input pixel).  Element (m, k) of the A tile
//       starting at record s is at s*16 + (m>>3)*128 + (m&7)*16 + (k>>2)*PLANE + (k&3)*4:
//       descriptor SBO = 128, LBO = PLANE.  hi = raw fp32 bits (kind::tf32 truncates),
//       lo = x - trunc(x), both produced once per element by the loaders.
//   B (weights): tc_pack_weights' per-K-step [W_hi (Npad rows) | W_lo (Npad rows)].
// 3xTF32 per K-step and M tile:  A_hi x [W_hi|W_lo] (N = 2 Npad) + A_lo x W_hi (N = Npad)
// (Npad <= 128), else three N = Npad MMAs.  D columns [0, Npad) + [Npad, 2 Npad) summed
// in the epilogue.
//
// Per CTA (persistent, one per SM, 14 warps):
//   warps 4-12 loaders, 3 groups of 3 taking units in turn (a single group was
//              latency-bound at ~2700 cycles per unit, above the MMA time):
//              per (tile, channel chunk rc, tap row i) unit fill one halo unit
//              buffer: records f0 + i*d*Wv + [0, NR) of the 8 channels (coalesced LDG,
//              lanes = consecutive pixels, zero outside the image / the padding), split
//              hi/lo, four 16-byte STS per pixel; loader warp 0 also requests the unit's
//              l K-steps of packed weights with one bulk async copy into the same buffer
//              (first warp of the group).
//   warp 13    MMA issuer: per unit l taps x MT M tiles x 2 MMAs, one tcgen05.commit
//              frees the unit buffer; one commit per tile hands the accumulators over.
//   warps 0-3  epilogue (one per TMEM lane quarter): tcgen05.ld, bias +
//              nonlinearity (forward) or the upstream nonlinearity's derivative (data
//              gradient), coalesced NCHW stores (lane = pixel).
#include <stdlib.h>

#include "dp_common.cuh"
#include "tc_ptx.cuh"

namespace dp {

int tc_pack(const float *w, float *wp, int Q, int R, int l, int bwd, int rp, cudaStream_t st);
int tc_pack_f16(const float *w, void *wp, int Q, int R, int l, int bwd, int *flag,
                cudaStream_t st, int rp = 0);
unsigned long long *tc_trace_buffer(cudaStream_t st);

// 14 warps: registers are granted per 4 warps, so 14 warps (as 16) leave 128 registers
// per thread for the loaders' 48 values in flight; 17 warps (as 20) would cap them at 96.
constexpr int TF_EPI_WARPS = 4;
constexpr int TF_LOAD_WARP0 = 4;
constexpr int TF_LOAD_WARPS = 9;
constexpr int TF_MMA_WARP = 13;
constexpr int TF_THREADS = (TF_MMA_WARP + 1) * 32;
constexpr int TF_MAX_MT = 8;
constexpr int TF_MAX_HB = 6;
constexpr int TF_LGROUPS = 3;  // loader groups of 3 warps, rotating units (three in flight)
constexpr int TF_LGW = TF_LOAD_WARPS / TF_LGROUPS;  // warps per loader group
constexpr int TF_LU = 6;  // loader: records per thread in flight (NR <= TF_LU * 128 per pass)
constexpr int TF_SMEM_BUDGET = 220 * 1024;

struct TfArgs {
    const float *in;     // (n, R, Hin, Win)
    const float *wpack;  // tc_pack_weights layout
    const float *bias;   // (Q) forward, nullptr for the data gradient
    float *out;          // (n, Q, Ho, Wo)
    const float *gate;   // (n, Q, Ho, Wo) nonlinearity output, or nullptr
    int R, Hin, Win;     // real input
    int Wv, pad;         // virtual (zero-padded) grid width; offset of the real input in it
    int Q, Ho, Wo, l, d, act, gate_kind;
    int n_rc, Npad, MT, acc_cols, NR, HB;
    int G, tpd;          // the tap-packed last chunk: K steps per unit, record step per K step
    uint32_t wunit_pk;   // its weight-unit bytes (other chunks: wunit_bytes)
    uint32_t plane_bytes, halo_bytes, wunit_bytes, ubytes;
    int tiles_per_img, total_tiles, flat_len;
    unsigned long long *trace;  // DP_TC_TRACE=<cta>: per-unit clock64 stamps of one CTA (8 slots)
    int trace_cta;
    const unsigned char *xr;    // relayout planes (TMA-fed mode) or nullptr (loader warps)
    long long plane_recs;       // records per relayout plane
    const int *exit_if;         // fp16 kernel: exit when its operands tripped the range flag
    const int *exit_unless;     // its tf32 fallback: run only when they did
};

// slots: 0/1 loader warp 0 unit start/end, 2/3/4 MMA wait/got/issued, 5/6 epilogue
// tile wait/got (at the tile's first unit), 7 epilogue tile done
#define TF_TRACE(A, U, SLOT, COND)                                                   \
    do {                                                                             \
        if ((A).trace && (COND) && (int)blockIdx.x == (A).trace_cta && (U) < 1024)    \
            (A).trace[(U) * 8 + (SLOT)] = clock64();                                 \
    } while (0)

// inlined so the 16 evaluations of an epilogue chunk interleave (an out-of-line call per
// value serialised them: measured ~30k cycles per tile with 4 epilogue warps)
__device__ __forceinline__ float tf_act(float v, int kind) {
    if (kind == DP_TANH || kind == DP_TANH_FAST) return tanhf(v);
    if (kind == DP_RELU) return dp_relu(v);
    return v;
}

// RP > 0: the LAST 8-channel chunk holds only RP <= 4 channels and uses tap-packed records
// -- slot k = t*RP + c of the record at flat index f holds x[c, f + t*d] (TP = 8 / RP column
// taps), so a K step covers TP taps of its channels instead of one tap with 8 - RP zero
// channels (c2 conv1: 3 channels, one chunk; c2 conv3 data gradient: 10 = 8 + 2)
template <bool B>
struct BoolTag {
    static constexpr bool value = B;
};
template <int V>
struct IntTag {
    static constexpr int value = V;
};

// HALF: fp16 split operands (kind::f16, K = 16 per MMA): records carry 16 channels as
// [hi c0-7 | hi c8-15 | lo c0-7 | lo c8-15] (8 halves per 16-byte core-matrix row, the same
// byte geometry as the tf32 records, so descriptors are unchanged) -- half the record and
// weight bytes and half the MMAs per channel.  Forward only (bounded activations).
// OFS: a forward with the data gradient's offset split (lo' scaled 2^11, cross products in
// the second accumulator half): single tap-packed chunks (first layers), whose small inputs
// would leave an unscaled fp16 lo subnormal
template <bool STACKED, bool BWD, int RP, bool HALF = false, bool OFS = false>
__global__ void __launch_bounds__(TF_THREADS, 1) tc_conv_flat_kernel(const TfArgs a) {
    constexpr int TP = RP ? 8 / RP : 1;
    constexpr int CH = HALF ? 16 : 8;  // channels per chunk (one K step per tap)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint64_t ufull[TF_MAX_HB], uempty[TF_MAX_HB], tfull[2], tempty[2];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) float s_bias[256];

    // fp16-split launches come in pairs (fp16 kernel, tf32 fallback) gated by the range flag
    // the fp16 relayout / weight packs set; exactly one of the two does the work (uniform,
    // before any barrier or TMEM allocation)
    if ((a.exit_if && *(volatile const int *)a.exit_if) ||
        (a.exit_unless && !*(volatile const int *)a.exit_unless))
        return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int MT = a.MT;
    const int units = a.n_rc * a.l;
    for (int o = threadIdx.x; o < a.Npad; o += blockDim.x)
        s_bias[o] = (!BWD && o < a.Q) ? a.bias[o] : 0.f;
    if (threadIdx.x == 0) {
        for (int b = 0; b < a.HB; ++b) {
            // loader warps + the weight copy's expect_tx; TMA-fed: one expect_tx
            ptx::mbar_init(&ufull[b], a.xr ? 1 : TF_LGW + 1);
            ptx::mbar_init(&uempty[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], a.xr ? 2 * TF_EPI_WARPS : TF_EPI_WARPS);
        }
        ptx::mbar_fence_init();
    }
    if (warp == TF_MMA_WARP) ptx::tmem_alloc<512>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;

    // TMA-fed: one producer thread; warps TF_LOAD_WARP0 + 1..4 join the epilogue (a second
    // group taking alternate 16-column chunks: a single group of 4 warps, latency bound at
    // ~950 cycles per chunk, set the pace of the narrow-K first layer -- tools/tf_trace.py)
    const bool epi2 = a.xr && warp > TF_LOAD_WARP0 && warp <= TF_LOAD_WARP0 + TF_EPI_WARPS;
    if (a.xr && warp == TF_LOAD_WARP0) {
        // ====================== TMA-fed producer (relayout planes) ======================
        // the unit's four record planes are contiguous ranges of the pre-split relayout
        // (tc_relayout / tc_relayout_f16): four bulk copies + the weight unit, one expect_tx
        if (warp == TF_LOAD_WARP0 && lane == 0) {
            const unsigned char *wsrc = reinterpret_cast<const unsigned char *>(a.wpack);
            int b = 0, gu = 0;
            uint32_t uph = 0;
            for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
                const int img = tile / a.tiles_per_img;
                const int f0 = (tile - img * a.tiles_per_img) * MT * 128;
                for (int rc = 0; rc < a.n_rc; ++rc) {
                    const unsigned char *pl = a.xr + ((size_t)img * a.n_rc + rc) * 4 *
                                                         (size_t)a.plane_recs * 16;
                    for (int i = 0; i < a.l; ++i, ++gu) {
                        ptx::mbar_wait(&uempty[b], uph ^ 1);
                        TF_TRACE(a, gu, 0, true);
                        unsigned char *ub = smem_raw + (size_t)b * a.ubytes;
                        const bool pk = RP > 0 && rc == a.n_rc - 1;  // tap-packed last chunk
                        const uint32_t wub = pk ? a.wunit_pk : a.wunit_bytes;
                        ptx::mbar_expect_tx(&ufull[b], 4 * a.plane_bytes + wub);
                        const long long rec0 = f0 + (long long)i * a.d * a.Wv;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            ptx::bulk_g2s(ub + (size_t)q * a.plane_bytes,
                                          pl + ((size_t)q * a.plane_recs + rec0) * 16,
                                          a.plane_bytes, &ufull[b]);
                        const unsigned char *ws =
                            wsrc + (size_t)rc * a.l * a.wunit_bytes + (size_t)i * wub;
                        for (uint32_t off = 0; off < wub; off += 32768u) {
                            const uint32_t nb = wub - off < 32768u ? wub - off : 32768u;
                            ptx::bulk_g2s(ub + a.halo_bytes + off, ws + off, nb, &ufull[b]);
                        }
                        TF_TRACE(a, gu, 1, true);
                        if (++b == a.HB) {
                            b = 0;
                            uph ^= 1;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (!a.xr && warp >= TF_LOAD_WARP0 && warp < TF_MMA_WARP) {
        // ================================ loaders ================================
        const int lw = (warp - TF_LOAD_WARP0) % TF_LGW, grp = (warp - TF_LOAD_WARP0) / TF_LGW;
        const long long plane_in = (long long)a.Hin * a.Win;
        const unsigned char *wsrc = reinterpret_cast<const unsigned char *>(a.wpack);
        int b = 0, gu = 0;
        uint32_t uph = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            const int img = tile / a.tiles_per_img;
            const int f0 = (tile - img * a.tiles_per_img) * MT * 128;
            for (int rc = 0, wu = 0; rc < a.n_rc; ++rc) {
                const float *src = a.in + ((long long)img * a.R + rc * CH) * plane_in;
                const int cvalid = min(CH, a.R - rc * CH);
                const bool pk = RP > 0 && rc == a.n_rc - 1;
                const uint32_t wub = pk ? a.wunit_pk : a.wunit_bytes;
                for (int i = 0; i < a.l; ++i, ++wu, ++gu) {
                    if ((gu % TF_LGROUPS) != grp) {  // the other group's unit
                        if (++b == a.HB) {
                            b = 0;
                            uph ^= 1;
                        }
                        continue;
                    }
                    ptx::mbar_wait_sleep(&uempty[b], uph ^ 1);
                    TF_TRACE(a, gu, 0, lw == 0 && lane == 0);
                    unsigned char *ub = smem_raw + (size_t)b * a.ubytes;
                    if (lw == 0) {
                        if (ptx::elect_one()) {
                            ptx::mbar_expect_tx(&ufull[b], wub);
                            // the packed chunk is the last: its units follow all full ones
                            const unsigned char *ws =
                                wsrc + (size_t)rc * a.l * a.wunit_bytes + (size_t)i * wub;
                            for (uint32_t off = 0; off < wub; off += 32768u) {
                                const uint32_t nb = wub - off < 32768u ? wub - off : 32768u;
                                ptx::bulk_g2s(ub + a.halo_bytes + off, ws + off, nb, &ufull[b]);
                            }
                        }
                        __syncwarp();
                    }
                    const int gbase = f0 + i * a.d * a.Wv;
                    // one straight-line record loop per record kind (a runtime branch inside
                    // the unrolled loads cost the loaders their ILP: measured 20 % slower)
                    // (LU records per thread in flight: 2 when the whole halo is <= 256 records
                    // -- one M tile per CTA tile, wide layers -- where 5 mostly idled)
                    auto fill = [&](auto packed, auto lu) {
                        constexpr bool PK = decltype(packed)::value;
                        constexpr int LU = decltype(lu)::value;
                        for (int r0 = lw * 32 + lane; r0 < a.NR; r0 += LU * TF_LGW * 32) {
                            float v[LU][CH];
#pragma unroll
                            for (int u = 0; u < LU; ++u) {
                                const int r = r0 + u * TF_LGW * 32;
                                const int gf = gbase + r;
                                const int yv = gf / a.Wv;
                                if (!PK) {
                                    const int y = yv - a.pad, x = gf - yv * a.Wv - a.pad;
                                    const bool ok =
                                        r < a.NR && y >= 0 && y < a.Hin && x >= 0 && x < a.Win;
                                    const float *p = src + (ok ? (long long)y * a.Win + x : 0);
#pragma unroll
                                    for (int k = 0; k < CH; ++k)
                                        v[u][k] = (ok && k < cvalid) ? __ldg(p + k * plane_in) : 0.f;
                                } else {
#pragma unroll
                                    for (int t = 0; t < TP; ++t) {
                                        // column tap t: flat index gf + t*d (wraps into the
                                        // next virtual row only for discarded outputs / zero
                                        // weights)
                                        int xt = gf - yv * a.Wv + t * a.d, yt = yv;
                                        while (xt >= a.Wv) {
                                            xt -= a.Wv;
                                            ++yt;
                                        }
                                        yt -= a.pad;
                                        xt -= a.pad;
                                        const bool okt = r < a.NR && yt >= 0 && yt < a.Hin &&
                                                         xt >= 0 && xt < a.Win;
                                        const float *p =
                                            src + (okt ? (long long)yt * a.Win + xt : 0);
#pragma unroll
                                        for (int c = 0; c < (RP ? RP : 1); ++c)
                                            v[u][t * RP + c] = okt ? __ldg(p + c * plane_in) : 0.f;
                                    }
#pragma unroll
                                    for (int k = TP * RP; k < 8; ++k) v[u][k] = 0.f;
                                }
                            }
#pragma unroll
                            for (int u = 0; u < LU; ++u) {
                                const int r = r0 + u * TF_LGW * 32;
                                if (r >= a.NR) break;
                                const uint32_t ps = a.plane_bytes / 16;  // plane stride (16 B)
                                if constexpr (HALF) {
                                    uint32_t hw[8], lw2[8];
#pragma unroll
                                    for (int q = 0; q < 8; ++q) {
                                        if (BWD || OFS)  // deltas: the offset split
                                            ptx::f16_split2_scaled(v[u][2 * q], v[u][2 * q + 1],
                                                                   hw[q], lw2[q]);
                                        else
                                            ptx::f16_split2(v[u][2 * q], v[u][2 * q + 1], hw[q],
                                                            lw2[q]);
                                    }
                                    uint4 *q0 = reinterpret_cast<uint4 *>(ub) + r;
                                    q0[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                                    q0[ps] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
                                    q0[2 * ps] = make_uint4(lw2[0], lw2[1], lw2[2], lw2[3]);
                                    q0[3 * ps] = make_uint4(lw2[4], lw2[5], lw2[6], lw2[7]);
                                    continue;
                                }
                                float4 *p0 = reinterpret_cast<float4 *>(ub) + r;
                                p0[0] = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
                                p0[ps] = make_float4(v[u][4], v[u][5], v[u][6], v[u][7]);
                                p0[2 * ps] =
                                    make_float4(ptx::tf32_lo(v[u][0]), ptx::tf32_lo(v[u][1]),
                                                ptx::tf32_lo(v[u][2]), ptx::tf32_lo(v[u][3]));
                                p0[3 * ps] =
                                    make_float4(ptx::tf32_lo(v[u][4]), ptx::tf32_lo(v[u][5]),
                                                ptx::tf32_lo(v[u][6]), ptx::tf32_lo(v[u][7]));
                            }
                        }
                    };
                    if (RP > 0 && pk)
                        fill(BoolTag<RP != 0>(), IntTag<TF_LU>());
                    else if (a.NR <= 2 * TF_LGW * 32)
                        fill(BoolTag<false>(), IntTag<2>());
                    else
                        fill(BoolTag<false>(), IntTag<HALF ? TF_LU / 2 : TF_LU>());
                    // generic-proxy stores -> visible to the tensor core (async proxy)
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&ufull[b]);
                    TF_TRACE(a, gu, 1, lw == 0 && lane == 0);
                    if (++b == a.HB) {
                        b = 0;
                        uph ^= 1;
                    }
                }
            }
        }
    } else if (warp == TF_MMA_WARP) {
        // ================================ MMA issuer ================================
        const uint32_t hs = ptx::smem_u32(smem_raw);
        const uint32_t idesc_n = HALF ? ptx::idesc_f16(128, a.Npad) : ptx::idesc_tf32(128, a.Npad);
        const uint32_t idesc_2n =
            HALF ? ptx::idesc_f16(128, 2 * a.Npad) : ptx::idesc_tf32(128, 2 * a.Npad);
        const uint32_t ks_units = (uint32_t)(a.Npad * 64) >> 4;  // descriptor units = 16 B
        const uint32_t wlo_units = (uint32_t)(a.Npad * 32) >> 4;
        const uint32_t lo_units = (2 * a.plane_bytes) >> 4;
        int b = 0, buf = 0, gu = 0;
        uint32_t uph = 0, tph = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tempty[buf], tph ^ 1);
            ptx::tc_fence_after();
            const uint32_t dbase = tmem + (uint32_t)(buf * MT * a.acc_cols);
            for (int u = 0; u < units; ++u, ++gu) {
                TF_TRACE(a, gu, 2, lane == 0);
                ptx::mbar_wait(&ufull[b], uph);
                ptx::tc_fence_after();
                TF_TRACE(a, gu, 3, lane == 0);
                if (ptx::elect_one()) {
                    const uint32_t ubase = hs + (uint32_t)b * a.ubytes;
                    const uint64_t a0 = ptx::smem_desc(ubase, a.plane_bytes, 128);
                    const uint64_t b0 = ptx::smem_desc(ubase + a.halo_bytes, 128, 256);
                    const bool pk = RP > 0 && u >= units - a.l;  // the packed last chunk
                    const int G = pk ? a.G : a.l, step = pk ? a.tpd : a.d;
                    for (int j = 0; j < G; ++j) {
                        const uint64_t bj = b0 + (uint64_t)(j * ks_units);
                        const uint32_t acc = (u | j) != 0;
                        for (int mt = 0; mt < MT; ++mt) {
                            const uint64_t ad = a0 + (uint64_t)(mt * 128 + j * step);
                            const uint32_t dd = dbase + (uint32_t)(mt * a.acc_cols);
                            if (HALF && STACKED && (BWD || OFS)) {
                                // offset split: [hi*hi | hi*lo'] + lo'*hi into the lo' half
                                ptx::mma_f16_ss(dd, ad, bj, idesc_2n, acc);
                                ptx::mma_f16_ss(dd + a.Npad, ad + lo_units, bj, idesc_n, 1);
                            } else if (HALF && STACKED) {
                                ptx::mma_f16_ss(dd, ad, bj, idesc_2n, acc);
                                ptx::mma_f16_ss(dd, ad + lo_units, bj, idesc_n, 1);
                            } else if (HALF) {
                                ptx::mma_f16_ss(dd, ad, bj, idesc_n, acc);
                                ptx::mma_f16_ss(dd, ad, bj + wlo_units, idesc_n, 1);
                                ptx::mma_f16_ss(dd, ad + lo_units, bj, idesc_n, 1);
                            } else if (STACKED) {
                                ptx::mma_tf32_ss(dd, ad, bj, idesc_2n, acc);
                                ptx::mma_tf32_ss(dd, ad + lo_units, bj, idesc_n, 1);
                            } else {
                                ptx::mma_tf32_ss(dd, ad, bj, idesc_n, acc);
                                ptx::mma_tf32_ss(dd, ad, bj + wlo_units, idesc_n, 1);
                                ptx::mma_tf32_ss(dd, ad + lo_units, bj, idesc_n, 1);
                            }
                        }
                    }
                    ptx::mma_commit(&uempty[b]);
                }
                __syncwarp();
                TF_TRACE(a, gu, 4, lane == 0);
                if (++b == a.HB) {
                    b = 0;
                    uph ^= 1;
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(&tfull[buf]);
            __syncwarp();
            if (++buf == 2) {
                buf = 0;
                tph ^= 1;
            }
        }
    } else if (warp < TF_EPI_WARPS || epi2) {
        // ================================ epilogue ================================
        const int q = warp & 3;
        const int eg = epi2 ? 1 : 0, neg = a.xr ? 2 : 1;  // epilogue group, groups
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const long long ostride = (long long)a.Ho * a.Wo;
        int buf = 0, gu = 0;
        uint32_t tph = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x, gu += units) {
            const int img = tile / a.tiles_per_img;
            const int f0 = (tile - img * a.tiles_per_img) * MT * 128;
            TF_TRACE(a, gu, 5, warp == 0 && lane == 0);
            ptx::mbar_wait_sleep(&tfull[buf], tph);
            ptx::tc_fence_after();
            TF_TRACE(a, gu, 6, warp == 0 && lane == 0);
            const long long img_off = (long long)img * a.Q * ostride;
            for (int mt = 0; mt < MT; ++mt) {
                const int p = f0 + mt * 128 + q * 32 + lane;
                const int u = p / a.Wv, v = p - u * a.Wv;
                const bool inside = p < a.flat_len && v < a.Wo;
                const long long pix = img_off + (long long)u * a.Wo + v;
                const uint32_t dcol =
                    tmem + lane_off + (uint32_t)((buf * MT + mt) * a.acc_cols);
                for (int o0 = 16 * eg; o0 < a.Npad; o0 += 16 * neg) {
                    uint32_t r[16], r2[16];
                    ptx::tmem_ld16(dcol + o0, r);
                    if (STACKED) ptx::tmem_ld16(dcol + a.Npad + o0, r2);
                    const long long off0 = pix + (long long)o0 * ostride;
                    const int nq = min(16, a.Q - o0);
                    float aux[16];
                    if (BWD) {
#pragma unroll
                        for (int t = 0; t < 16; ++t)
                            aux[t] = (a.gate && inside && t < nq)
                                         ? __ldg(a.gate + off0 + t * ostride) : 0.f;
                    } else {
#pragma unroll
                        for (int t = 0; t < 16; t += 4) {
                            const float4 b4 = *reinterpret_cast<const float4 *>(s_bias + o0 + t);
                            aux[t] = b4.x, aux[t + 1] = b4.y, aux[t + 2] = b4.z, aux[t + 3] = b4.w;
                        }
                    }
                    ptx::tmem_wait_ld();
                    if (!inside) continue;
#pragma unroll
                    for (int t = 0; t < 16; ++t) {
                        if (t >= nq) break;
                        float val = __uint_as_float(r[t]);
                        if (STACKED && HALF && (BWD || OFS))
                            val += __uint_as_float(r2[t]) * (1.f / ptx::F16_LO_SCALE);
                        else if (STACKED)
                            val += __uint_as_float(r2[t]);
                        if (!BWD)
                            val = tf_act(val + aux[t], a.act);
                        else if (a.gate)
                            val = gate_from_output(val, aux[t], a.gate_kind);
                        a.out[off0 + t * ostride] = val;
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            TF_TRACE(a, gu, 7, warp == 0 && lane == 0);
            if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
            if (++buf == 2) {
                buf = 0;
                tph ^= 1;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == TF_MMA_WARP) ptx::tmem_dealloc<512>(tmem);
}

// --------------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------------
struct TfPlan {
    int Npad, n_rc, MT, acc_cols, NR, HB, rp, G, tp;
    bool stacked, ok;
    uint32_t plane_bytes, halo_bytes, wunit_bytes, wunit_pk, ubytes;
};

// M tiles per CTA tile: accumulators double-buffered in the 512 TMEM columns; unit
// buffers (halo + one tap row of weights) as many as fit, at least two.
static TfPlan tf_plan(int R, int Q, int l, int d, int max_mt, bool bwd, bool half = false) {
    TfPlan p;
    p.Npad = (Q + 15) / 16 * 16;
    p.n_rc = half ? (R + 15) / 16 : (R + 7) / 8;
    // tap-packed records for inputs of <= 4 channels.  The kernel also packs the last
    // chunk of a wider input (DP_TF_PACK_LAST), but that measured slower (c2 conv3 data
    // gradient 0.76 -> 0.84 ms): the packed units' loads, not their MMAs, set the pace.
    const int rem = R - (p.n_rc - 1) * 8;
    (void)bwd;
    // fp16-split records hold 16 slots: inputs of <= 8 channels pack 16 / R column taps
    // (c3's 8-channel head data gradient: 4 K steps per tap row instead of 7 tf32 ones)
    // (and the last chunk of a wider input when it holds <= 8 channels: c3's 50 = 3 x 16 + 2
    // channels run one K step of 8 column taps there instead of l steps of 2 channels)
    const int rem16 = R - (p.n_rc - 1) * 16;
    if (half)
        p.rp = (rem16 <= 8 && l > 1 && !getenv("DP_TF_NOPACK") &&
                (p.n_rc == 1 || !getenv("DP_TF_F16_NOPACK_LAST")))
                   ? rem16
                   : 0;
    else
        p.rp = (rem <= 4 && l > 1 && (p.n_rc == 1 || getenv("DP_TF_PACK_LAST")) &&
                !getenv("DP_TF_NOPACK"))
                   ? rem
                   : 0;
    p.tp = p.rp ? (half ? 16 : 8) / p.rp : 1;
    p.G = p.rp ? (l + p.tp - 1) / p.tp : l;
    // Stacked ([W_hi | W_lo] in one N = 2 Npad MMA) saves an MMA per K step but doubles the
    // accumulator columns, halving the M tiles per CTA tile.  Wide inputs (>= 4 channel
    // chunks) are loader / feed bound, not MMA bound, and gain more from the extra M tiles
    // (round 2, tools/conv_ab.py: c3 conv2 fwd 2.47 -> 1.92 ms, data grad 2.51 -> 1.84 at
    // MT 2 -> 4); narrow ones, and outputs of <= 32 channels (three N = 32 MMAs cost 120
    // cycles vs 88 stacked), or with many taps per unit (l > 4: Plain CNN1's 7x7 head data
    // grad 1.19 stacked vs 1.26), are MMA bound and keep stacking (c2 conv2 fwd 0.83 vs 1.00).
    p.stacked = 2 * p.Npad <= 256 && !getenv("DP_TF_NOSTACK") &&
                (R < 32 || p.Npad < 64 || l > 4 || getenv("DP_TF_STACK"));
    // the fp16 data gradient needs the second accumulator half (offset-split cross terms)
    if (half && bwd) p.stacked = 2 * p.Npad <= 256;
    p.acc_cols = p.stacked ? 2 * p.Npad : p.Npad;
    p.ok = p.Npad <= 256 && (!(half && bwd) || p.stacked);
    int mt = p.acc_cols <= 256 ? 256 / p.acc_cols : 1;
    if (mt > TF_MAX_MT) mt = TF_MAX_MT;
    if (const char *e = getenv("DP_TF_MT")) {
        int v = atoi(e);
        if (v >= 1 && v < mt) mt = v;
    }
    if (max_mt >= 1 && mt > max_mt) mt = max_mt;
    // At least TF_LGROUPS unit buffers: a loader group starts waiting for a buffer up to
    // TF_LGROUPS units ahead, and with fewer buffers that wait would be two phases ahead
    // of the barrier -- a parity wait then passes on the stale phase.  Fewer M tiles
    // (a smaller halo) until they fit.
    for (;; mt = (mt + 1) / 2) {
        p.MT = mt;
        p.NR = (mt * 128 + (l - 1) * d + 7) / 8 * 8;
        p.plane_bytes = (uint32_t)p.NR * 16;
        p.halo_bytes = 4 * p.plane_bytes;
        p.wunit_pk = (uint32_t)(p.G * p.Npad * 64);
        // unit buffers hold the largest unit: a full one unless the packed chunk is the
        // only one
        p.wunit_bytes = (uint32_t)((p.rp && p.n_rc == 1 ? p.G : l) * p.Npad * 64);
        p.ubytes = (p.halo_bytes + p.wunit_bytes + 127) / 128 * 128;
        long long hb = (long long)TF_SMEM_BUDGET / p.ubytes;
        if (hb > TF_MAX_HB) hb = TF_MAX_HB;
        p.HB = (int)hb;
        if (p.HB >= TF_LGROUPS || mt == 1) break;
    }
    p.ok = p.ok && p.HB >= TF_LGROUPS && (p.plane_bytes >> 4) < (1u << 14);
    return p;
}

bool tf_conv_supported(int R, int Q, int l, int d) {
    if (getenv("DP_TC_HALO")) return false;  // force the halo-buffer kernel (tc_conv.cu)
    return tf_plan(R, Q, l, d, 0, true).ok;  // unpacked: the larger weight unit
}

// relayout kernels of the tap-stacked conv (tc_conv_tap.cu): the same record planes
__global__ void tc_relayout(const float *__restrict__ in, float4 *__restrict__ xr, int R, int Hin,
                            int Win, int Wv, int pad, int n_rc, long long plane_recs,
                            long long vrecs, long long total);
template <bool SCALED>
__global__ void tc_relayout_f16(const float *__restrict__ in, uint4 *__restrict__ xr, int R,
                                int Hin, int Win, int Wv, int pad, int n_rc, int n_rc_do,
                                long long plane_recs, long long vrecs, long long total,
                                int *flag);

// NCHW (n, R <= 4, Hin, Win) -> four planes of tap-packed 16-byte records over the virtual
// grid (the loaders' RP layout: slot t*R + c of record f = x[c] at virtual flat index
// f + t*d, TP = 8 / R column taps, zeros outside the input):
// [hi s0-3 | hi s4-7 | lo s0-3 | lo s4-7], hi = raw fp32 bits, lo = x - trunc_tf32(x).
// The packed chunk's loaders were the limit of the 3-channel first layers (ncu, c3 conv1:
// 28 % of the instructions at the record loads, 10 % at the flat-index divide).
// (R a template parameter: with a runtime R the slot index t*R + c put v[] on the stack)
template <int R>
__global__ void __launch_bounds__(256) tc_relayout_pk(const float *__restrict__ in,
                                                      float4 *__restrict__ xr, int Hin,
                                                      int Win, int Wv, int pad, int d,
                                                      long long plane_recs, long long vrecs,
                                                      long long total) {
    constexpr int TP = 8 / R;
    const long long cs = (long long)Hin * Win;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long n = idx / plane_recs;
        const long long f = idx - n * plane_recs;
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.f;
        // one 32-bit divide per record, the taps step along the row (a 64-bit divide per tap
        // made this pass issue bound); y < Hin implies the tap is inside the virtual grid
        const int fi = (int)f, yv0 = fi / Wv, xv0 = fi - yv0 * Wv;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (t >= TP) break;
            int xx = xv0 + t * d, yy = yv0;
            while (xx >= Wv) {
                xx -= Wv;
                ++yy;
            }
            const int y = yy - pad, x = xx - pad;
            if (!(y >= 0 && y < Hin && x >= 0 && x < Win)) continue;
            const float *src = in + n * R * cs + (long long)y * Win + x;
#pragma unroll
            for (int c = 0; c < R; ++c) v[t * R + c] = __ldg(src + c * cs);
        }
        float4 *dst = xr + n * 4 * plane_recs + f;
        dst[0] = make_float4(v[0], v[1], v[2], v[3]);
        dst[plane_recs] = make_float4(v[4], v[5], v[6], v[7]);
        dst[2 * plane_recs] = make_float4(ptx::tf32_lo(v[0]), ptx::tf32_lo(v[1]),
                                          ptx::tf32_lo(v[2]), ptx::tf32_lo(v[3]));
        dst[3 * plane_recs] = make_float4(ptx::tf32_lo(v[4]), ptx::tf32_lo(v[5]),
                                          ptx::tf32_lo(v[6]), ptx::tf32_lo(v[7]));
    }
}

// fp16-split records of a single tap-packed chunk (R <= 8 channels): slot t*R + c of record
// f = x[c] at virtual flat index f + t*d, TP = 16 / R column taps, planes
// [hi s0-7 | hi s8-15 | lo s0-7 | lo s8-15]; SCALED: the data gradient's offset split;
// flag as tc_relayout_f16
// (the LAST chunk of a wider input when n_rc > 1: channels c_base .. c_base + rp of the R,
// written to chunk n_rc - 1 of each image's planes)
template <bool SCALED, int R>
__global__ void __launch_bounds__(256) tc_relayout_f16_pk(const float *__restrict__ in,
                                                          uint4 *__restrict__ xr, int R_all,
                                                          int c_base, int n_rc,
                                                          int Hin, int Win, int Wv, int pad,
                                                          int d, long long plane_recs,
                                                          long long vrecs, long long total,
                                                          int *flag) {
    constexpr int TP = 16 / R;
    const long long cs = (long long)Hin * Win;
    bool bad = false;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long n = idx / plane_recs;
        const long long f = idx - n * plane_recs;
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.f;
        const int fi = (int)f, yv0 = fi / Wv, xv0 = fi - yv0 * Wv;  // (as tc_relayout_pk)
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t >= TP) break;
            int xx = xv0 + t * d, yy = yv0;
            while (xx >= Wv) {
                xx -= Wv;
                ++yy;
            }
            const int y = yy - pad, x = xx - pad;
            if (!(y >= 0 && y < Hin && x >= 0 && x < Win)) continue;
            const float *src = in + (n * R_all + c_base) * cs + (long long)y * Win + x;
#pragma unroll
            for (int c = 0; c < R; ++c)
                if (t * R + c < 16) v[t * R + c] = __ldg(src + c * cs);
        }
        uint32_t hw[8], lw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            bad |= !(fabsf(v[2 * q]) < ptx::F16_SPLIT_MAX) ||
                   !(fabsf(v[2 * q + 1]) < ptx::F16_SPLIT_MAX);
            if constexpr (SCALED)
                ptx::f16_split2_scaled(v[2 * q], v[2 * q + 1], hw[q], lw[q]);
            else
                ptx::f16_split2(v[2 * q], v[2 * q + 1], hw[q], lw[q]);
        }
        uint4 *dst = xr + (n * n_rc + n_rc - 1) * 4 * plane_recs + f;
        dst[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        dst[plane_recs] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
        dst[2 * plane_recs] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        dst[3 * plane_recs] = make_uint4(lw[4], lw[5], lw[6], lw[7]);
    }
    if (bad) atomicOr(flag, 1);
}

// the tf32 TMA-fed mode of single-chunk tap-packed inputs (R <= 4: first layers)
static bool tf_pk_relayout(const TfPlan &q) {
    const char *e = getenv("DP_TF_PK_RELAYOUT");
    return q.rp > 0 && q.n_rc == 1 && !(e && e[0] == '0');
}
// ... and of narrow unpacked tf32 inputs (<= DP_TF_R32_CHUNKS 8-channel chunks, default 2:
// c3's 8-channel head data gradient, whose loaders were the limit)
static bool tf_r32_relayout(const TfPlan &q) {
    const char *e = getenv("DP_TF_R32_CHUNKS");
    const int mx = e ? atoi(e) : 2;
    return q.rp == 0 && q.n_rc <= mx;
}

// TMA-fed mode (forward, fp16-split, inputs >= 16 channels): the fp16 loaders were the
// limit (tools/tf_trace.py, c3 conv2: ~2800 loader vs ~2000 MMA cycles per unit), so the
// split is done once by a bandwidth-bound relayout pass and units arrive as bulk copies.
// fp16-split operands: forward of inputs with >= 16 channels (DP_TF_HALF=0: tf32), and the
// data gradient of deltas with >= 16 channels through the offset split (DP_TF_HALF_BWD=0)
// fp16-split operands for inputs of >= 16 channels: forward when the caller allows it
// (DP_FAST_INPUT_FP16_RANGE; DP_TF_HALF=0: never), data gradient by default
// (DP_TF_HALF_BWD=0: never).  Always TMA-fed and always paired with a tf32 fallback launch
// that runs instead when an operand is outside the split's range (|x| >= 2^15, inf, NaN):
// c4's relu outputs errors exceeded fp16's 65504.
// f16_ok: DP_FAST_INPUT_FP16_RANGE (1) | DP_FAST_PACK_FWD (2) from the caller
static bool tf_half(int R, int l, bool bwd, int f16_ok) {
    // <= 8 channels: tap-packed, data gradient only by default.  A packed fp16 first-layer
    // forward (DP_TF_F16_PACK_FWD=1; the offset split since round 2 -- the unscaled one left lo
    // subnormal below |x| = 1/8) is faster (c3 conv1 0.65 -> 0.57 ms, step -1 %), but on the
    // relu net c4 it moves the unforced dw2 error to 2.3e-4 against the exact tier's 4.5e-5
    // (relu / max-pool flips amplify any operand rounding), past the 3x parity bar
    // (the engine sets DP_FAST_PACK_FWD on tanh nets: c3 unforced parity unchanged)
    const bool pack_fwd = (f16_ok & 2) || getenv("DP_TF_F16_PACK_FWD");
    if (R < 16 && (R > 8 || getenv("DP_TF_NOPACK") || (!bwd && !pack_fwd))) return false;
    // (and >= 5 taps a row: c4's 3x3 8-channel head data gradient measured 0.513 ms in tf32
    // against 0.553 packed, c3's 7x7 one 1.24 -> 0.94)
    if (R < 16 && bwd && l < 5) return false;
    const char *he = getenv(bwd ? "DP_TF_HALF_BWD" : "DP_TF_HALF");
    if (he && he[0] == '0') return false;
    return bwd || (f16_ok & 1);
}

static bool tf_relayout_mode(int R, int l, bool bwd, int f16_ok) {
    const char *re = getenv("DP_TF_RELAYOUT");
    return tf_half(R, l, bwd, f16_ok) && !(re && re[0] == '0');
}

static long long tf_plane_recs(const TfPlan &p, int Hin, int Win, int pad, int l, int d, int Ho,
                               int Wo) {
    const int Wv = Win + 2 * pad;
    const long long flat_len = (long long)(Ho - 1) * Wv + Wo;
    const long long tpi = (flat_len + (long long)p.MT * 128 - 1) / ((long long)p.MT * 128);
    const long long need = (tpi - 1) * p.MT * 128 + (long long)(l - 1) * d * Wv + p.NR;
    const long long vrecs = (long long)(Hin + 2 * pad) * Wv;
    return ((need > vrecs ? need : vrecs) + 7) / 8 * 8;
}

static size_t tf_weight_bytes(const TfPlan &p, int l) {
    return p.rp ? (size_t)(p.n_rc - 1) * l * l * p.Npad * 64 + (size_t)l * p.wunit_pk
                : (size_t)p.n_rc * l * p.wunit_bytes;
}

static size_t al256(size_t v) { return (v + 255) / 256 * 256; }

// workspace of the fp16-split flat conv: [fp16 weights | tf32 fallback weights | range flag
// (256 B) | fp16 relayout planes]; 0 when it does not apply.  The flat kernel uses it when
// the caller's workspace covers it (else tf32 alone).
size_t tf_relayout_workspace(int n, int R, int Hin, int Win, int Q, int l, int d, int pad,
                             int Ho, int Wo, bool bwd) {
    // (sized as if fp16 were allowed: the query cannot know the caller's flags)
    if (Ho < 1 || Wo < 1) return 0;
    const int Wv = Win + 2 * pad;
    const long long flat_len = (long long)(Ho - 1) * Wv + Wo;
    const int max_mt = (int)((flat_len + 127) / 128);
    if (!tf_relayout_mode(R, l, bwd, true)) {  // tap-packed tf32 planes: [weights | planes]
        TfPlan q = tf_plan(R, Q, l, d, max_mt, bwd, false);
        if (!q.ok || !(tf_pk_relayout(q) || tf_r32_relayout(q))) return 0;
        return al256(tf_weight_bytes(q, l)) +
               (size_t)n * q.n_rc * 4 * tf_plane_recs(q, Hin, Win, pad, l, d, Ho, Wo) * 16;
    }
    TfPlan p = tf_plan(R, Q, l, d, max_mt, bwd, true);
    TfPlan q = tf_plan(R, Q, l, d, max_mt, bwd, false);
    if (!p.ok || !q.ok) return 0;
    return al256(tf_weight_bytes(p, l)) + al256(tf_weight_bytes(q, l)) + 256 +
           (size_t)n * p.n_rc * 4 * tf_plane_recs(p, Hin, Win, pad, l, d, Ho, Wo) * 16;
}

static int g_tf_sms = 0;

// one launch of plan p (fp16 records when half; TMA-fed from xr when given), weights at wp
static int tf_run(const TfPlan &p, int half, const float *in, const void *wp, const float *bias,
                  float *out, const float *gate, int n, int R, int Hin, int Win, int Q, int Ho,
                  int Wo, int l, int d, int pad, int act, int gate_kind, bool bwd,
                  const unsigned char *xr, long long plane_recs, const int *exit_if,
                  const int *exit_unless, cudaStream_t st) {
    const int Wv = Win + 2 * pad;
    const long long flat_len = (long long)(Ho - 1) * Wv + Wo;
    if (g_tf_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_tf_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_tf_sms <= 0) g_tf_sms = 148;
    }
    if ((long long)(Hin + 2 * pad) * Wv + p.NR > 0x7fffffffLL)
        return set_error(DP_ERR_UNSUPPORTED, "flat tensor-core conv: image too large");
    TfArgs a;
    a.in = in;
    a.wpack = (const float *)wp;
    a.bias = bias;
    a.out = out;
    a.gate = gate;
    a.R = R;
    a.Hin = Hin;
    a.Win = Win;
    a.Wv = Wv;
    a.pad = pad;
    a.Q = Q;
    a.Ho = Ho;
    a.Wo = Wo;
    a.l = l;
    a.d = d;
    a.act = act;
    a.gate_kind = gate_kind;
    a.n_rc = p.n_rc;
    a.Npad = p.Npad;
    a.MT = p.MT;
    a.G = p.G;
    a.wunit_pk = p.wunit_pk;
    a.tpd = p.tp * d;
    a.acc_cols = p.acc_cols;
    a.NR = p.NR;
    a.HB = p.HB;
    a.plane_bytes = p.plane_bytes;
    a.halo_bytes = p.halo_bytes;
    a.wunit_bytes = p.wunit_bytes;
    a.ubytes = p.ubytes;
    a.flat_len = (int)flat_len;
    a.tiles_per_img = (int)((flat_len + p.MT * 128 - 1) / (p.MT * 128));
    const long long tt = (long long)n * a.tiles_per_img;
    if (tt > 0x7fffffff) return set_error(DP_ERR_UNSUPPORTED, "flat tensor-core conv: too many tiles");
    a.total_tiles = (int)tt;
    if (a.total_tiles == 0) return DP_OK;
    // (not for an fp16 launch's fallback: requesting the buffer clears it)
    a.trace = getenv("DP_TC_TRACE") && !exit_unless ? tc_trace_buffer(st) : nullptr;
    a.trace_cta = a.trace ? atoi(getenv("DP_TC_TRACE")) : 0;
    a.xr = xr;
    a.plane_recs = plane_recs;
    a.exit_if = exit_if;
    a.exit_unless = exit_unless;
    const int grid = a.total_tiles < g_tf_sms ? a.total_tiles : g_tf_sms;
    const size_t smem = (size_t)p.HB * p.ubytes;
    void (*kern)(const TfArgs);
    // (fp16 kernels are TMA-fed: RP only marks the tap-packed chunk, 1 = packed)
    if (half && bwd)
        kern = p.rp ? tc_conv_flat_kernel<true, true, 1, true>
                    : tc_conv_flat_kernel<true, true, 0, true>;
    else if (half == 2)  // (offset split: stacked only)
        kern = tc_conv_flat_kernel<true, false, 1, true, true>;
    else if (half && p.rp)
        kern = p.stacked ? tc_conv_flat_kernel<true, false, 1, true>
                         : tc_conv_flat_kernel<false, false, 1, true>;
    else if (half)
        kern = p.stacked ? tc_conv_flat_kernel<true, false, 0, true>
                         : tc_conv_flat_kernel<false, false, 0, true>;
    else if (bwd && p.stacked)
        kern = p.rp == 1   ? tc_conv_flat_kernel<true, true, 1>
               : p.rp == 2 ? tc_conv_flat_kernel<true, true, 2>
               : p.rp == 3 ? tc_conv_flat_kernel<true, true, 3>
               : p.rp == 4 ? tc_conv_flat_kernel<true, true, 4>
                           : tc_conv_flat_kernel<true, true, 0>;
    else if (bwd)
        kern = p.rp == 1   ? tc_conv_flat_kernel<false, true, 1>
               : p.rp == 2 ? tc_conv_flat_kernel<false, true, 2>
               : p.rp == 3 ? tc_conv_flat_kernel<false, true, 3>
               : p.rp == 4 ? tc_conv_flat_kernel<false, true, 4>
                           : tc_conv_flat_kernel<false, true, 0>;
    else if (p.stacked)
        kern = p.rp == 1   ? tc_conv_flat_kernel<true, false, 1>
               : p.rp == 2 ? tc_conv_flat_kernel<true, false, 2>
               : p.rp == 3 ? tc_conv_flat_kernel<true, false, 3>
               : p.rp == 4 ? tc_conv_flat_kernel<true, false, 4>
                           : tc_conv_flat_kernel<true, false, 0>;
    else
        kern = p.rp == 1   ? tc_conv_flat_kernel<false, false, 1>
               : p.rp == 2 ? tc_conv_flat_kernel<false, false, 2>
               : p.rp == 3 ? tc_conv_flat_kernel<false, false, 3>
               : p.rp == 4 ? tc_conv_flat_kernel<false, false, 4>
                           : tc_conv_flat_kernel<false, false, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tc_conv_flat: cudaFuncSetAttribute: %s",
                         cudaGetErrorString(e));
    kern<<<grid, TF_THREADS, smem, st>>>(a);
    return check_launch("tc_conv_flat_kernel");
}

// the tf32 flat conv as the fallback of an fp16-split launch: runs only when *flag is set
// (weights packed into wp, which must hold tf_fallback_bytes)
size_t tf_fallback_bytes(int R, int Q, int l, int d, bool bwd) {
    TfPlan q = tf_plan(R, Q, l, d, 0, bwd, false);
    return q.ok ? al256(tf_weight_bytes(q, l)) : 0;
}
int tf_fallback(const float *in, const float *w, const float *bias, float *out, const float *gate,
                int n, int R, int Hin, int Win, int Q, int Ho, int Wo, int l, int d, int pad,
                int act, int gate_kind, bool bwd, void *wp, const int *flag, cudaStream_t st) {
    const int Wv = Win + 2 * pad;
    const long long flat_len = (long long)(Ho - 1) * Wv + Wo;
    TfPlan q = tf_plan(R, Q, l, d, (int)((flat_len + 127) / 128), bwd, false);
    if (!q.ok) return set_error(DP_ERR_UNSUPPORTED, "flat conv fallback: unsupported shape");
    int rc = tc_pack(w, (float *)wp, Q, R, l, bwd ? 1 : 0, q.rp, st);
    if (rc) return rc;
    return tf_run(q, false, in, wp, bias, out, gate, n, R, Hin, Win, Q, Ho, Wo, l, d, pad, act,
                  gate_kind, bwd, nullptr, 0, nullptr, flag, st);
}

static int tf_launch(const float *in, const float *w, const float *bias, float *out,
                     const float *gate, int n, int R, int Hin, int Win, int Q, int Ho, int Wo,
                     int l, int d, int pad, int act, int gate_kind, bool bwd, void *ws,
                     size_t ws_bytes, cudaStream_t st, int f16_ok = 0) {
    const int Wv = Win + 2 * pad;
    const long long flat_len = (long long)(Ho - 1) * Wv + Wo;
    // short images: fewer M tiles per CTA tile
    const int max_mt = (int)((flat_len + 127) / 128);
    const TfPlan q = tf_plan(R, Q, l, d, max_mt, bwd, false);  // tf32
    if (!q.ok)
        return set_error(DP_ERR_UNSUPPORTED, "flat tensor-core conv: unsupported (R=%d Q=%d k=%d d=%d)",
                         R, Q, l, d);
    if (((uintptr_t)ws & 15) != 0)
        return set_error(DP_ERR_ARG, "tensor-core conv: workspace must be 16-byte aligned");
    // fp16-split (TMA-fed, with the tf32 fallback) when it applies and the workspace holds it
    if (tf_relayout_mode(R, l, bwd, f16_ok) && ((uintptr_t)ws & 255) == 0) {
        const TfPlan p = tf_plan(R, Q, l, d, max_mt, bwd, true);
        const long long plane_recs = p.ok ? tf_plane_recs(p, Hin, Win, pad, l, d, Ho, Wo) : 0;
        const size_t wb16 = p.ok ? al256(tf_weight_bytes(p, l)) : 0;
        const size_t wb32 = al256(tf_weight_bytes(q, l));
        const size_t need = wb16 + wb32 + 256 + (size_t)n * p.n_rc * 4 * plane_recs * 16;
        // (a single packed forward chunk needs the stacked accumulator for its offset split)
        const bool pk_fwd_ok = bwd || !p.rp || p.n_rc > 1 || p.stacked;
        if (p.ok && pk_fwd_ok && ws_bytes >= need && plane_recs < 0x7fffffffLL) {
            unsigned char *w8 = (unsigned char *)ws;
            int *flag = (int *)(w8 + wb16 + wb32);
            const unsigned char *xr = w8 + wb16 + wb32 + 256;
            if (cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess)
                return set_error(DP_ERR_CUDA, "flat conv: flag reset failed");
            // single tap-packed forward chunk: the offset split too (tf_half)
            const bool ofs = !bwd && p.rp && p.n_rc == 1 && p.stacked &&
                             !getenv("DP_TF_F16_PACK_FWD_UNSCALED");
            int rc = tc_pack_f16(w, w8, Q, R, l, bwd ? 1 : ofs ? 2 : 0, flag, st, p.rp);
            if (rc) return rc;
            const long long vrecs = (long long)(Hin + 2 * pad) * Wv;
            const long long total = (long long)n * p.n_rc * plane_recs;
            const long long g = (total + 255) / 256;
            const int gg = (int)(g < 148 * 64 ? g : 148 * 64);
            // full 16-channel chunks, then the tap-packed last one (if any)
            const int n_full = p.rp ? p.n_rc - 1 : p.n_rc;
            if (n_full > 0) {
                const long long tf = (long long)n * n_full * plane_recs;
                const long long gf = (tf + 255) / 256;
                const int ggf = (int)(gf < 148 * 64 ? gf : 148 * 64);
                if (bwd)
                    tc_relayout_f16<true><<<ggf, 256, 0, st>>>(in, (uint4 *)xr, R, Hin, Win, Wv,
                                                               pad, p.n_rc, n_full, plane_recs,
                                                               vrecs, tf, flag);
                else
                    tc_relayout_f16<false><<<ggf, 256, 0, st>>>(in, (uint4 *)xr, R, Hin, Win,
                                                                Wv, pad, p.n_rc, n_full,
                                                                plane_recs, vrecs, tf, flag);
            }
            if (p.rp) {
                const long long tp_ = (long long)n * plane_recs;
                const long long gp = (tp_ + 255) / 256;
                const int ggp = (int)(gp < 148 * 64 ? gp : 148 * 64);
                const int c_base = (p.n_rc - 1) * 16;
#define DP_PK16(S, RR)                                                                  \
    tc_relayout_f16_pk<S, RR><<<ggp, 256, 0, st>>>(in, (uint4 *)xr, R, c_base, p.n_rc, Hin,  \
                                                   Win, Wv, pad, d, plane_recs, vrecs, tp_,  \
                                                   flag)
#define DP_PK16_R(S)                                                                    \
    switch (p.rp) {                                                                     \
        case 1: DP_PK16(S, 1); break;                                                   \
        case 2: DP_PK16(S, 2); break;                                                   \
        case 3: DP_PK16(S, 3); break;                                                   \
        case 4: DP_PK16(S, 4); break;                                                   \
        case 5: DP_PK16(S, 5); break;                                                   \
        case 6: DP_PK16(S, 6); break;                                                   \
        case 7: DP_PK16(S, 7); break;                                                   \
        default: DP_PK16(S, 8); break;                                                  \
    }
                if (bwd || ofs) {
                    DP_PK16_R(true)
                } else {
                    DP_PK16_R(false)
                }
#undef DP_PK16_R
#undef DP_PK16
            }
            (void)gg;
            rc = check_launch("tc_relayout_f16");
            if (rc) return rc;
            rc = tc_pack(w, (float *)(w8 + wb16), Q, R, l, bwd ? 1 : 0, q.rp, st);
            if (rc) return rc;
            rc = tf_run(p, ofs ? 2 : 1, in, w8, bias, out, gate, n, R, Hin, Win, Q, Ho, Wo, l, d, pad,
                        act, gate_kind, bwd, xr, plane_recs, flag, nullptr, st);
            if (rc) return rc;
            return tf_run(q, false, in, w8 + wb16, bias, out, gate, n, R, Hin, Win, Q, Ho, Wo,
                          l, d, pad, act, gate_kind, bwd, nullptr, 0, nullptr, flag, st);
        }
    }
    const size_t wbytes = tf_weight_bytes(q, l);
    if ((tf_pk_relayout(q) || tf_r32_relayout(q)) && ((uintptr_t)ws & 255) == 0) {
        // narrow tf32 inputs: relayout once, TMA-fed units
        const long long plane_recs = tf_plane_recs(q, Hin, Win, pad, l, d, Ho, Wo);
        const size_t need = al256(wbytes) + (size_t)n * q.n_rc * 4 * plane_recs * 16;
        if (ws_bytes >= need && plane_recs < 0x7fffffffLL) {
            unsigned char *w8 = (unsigned char *)ws;
            int rc = tc_pack(w, (float *)w8, Q, R, l, bwd ? 1 : 0, q.rp, st);
            if (rc) return rc;
            float4 *xr = reinterpret_cast<float4 *>(w8 + al256(wbytes));
            const long long vrecs = (long long)(Hin + 2 * pad) * Wv;
            const long long total = (long long)n * q.n_rc * plane_recs;
            const long long g = (total + 255) / 256;
            const int gg = (int)(g < 148 * 64 ? g : 148 * 64);
            if (q.rp) {
#define DP_PK32(RR) \
    tc_relayout_pk<RR><<<gg, 256, 0, st>>>(in, xr, Hin, Win, Wv, pad, d, plane_recs, vrecs, total)
                switch (R) {
                    case 1: DP_PK32(1); break;
                    case 2: DP_PK32(2); break;
                    case 3: DP_PK32(3); break;
                    default: DP_PK32(4); break;
                }
#undef DP_PK32
            } else
                tc_relayout<<<gg, 256, 0, st>>>(in, xr, R, Hin, Win, Wv, pad, q.n_rc, plane_recs,
                                                vrecs, total);
            rc = check_launch("tc_relayout");
            if (rc) return rc;
            return tf_run(q, false, in, w8, bias, out, gate, n, R, Hin, Win, Q, Ho, Wo, l, d,
                          pad, act, gate_kind, bwd, (const unsigned char *)xr, plane_recs,
                          nullptr, nullptr, st);
        }
    }
    if (ws == nullptr || ws_bytes < wbytes)
        return set_error(DP_ERR_ARG, "tensor-core conv: workspace %zu < %zu bytes", ws_bytes,
                         wbytes);
    int rc = tc_pack(w, (float *)ws, Q, R, l, bwd ? 1 : 0, q.rp, st);
    if (rc) return rc;
    return tf_run(q, false, in, ws, bias, out, gate, n, R, Hin, Win, Q, Ho, Wo, l, d, pad, act,
                  gate_kind, bwd, nullptr, 0, nullptr, nullptr, st);
}

int tf_conv_forward(const float *x, const float *w, const float *b, float *y, int n, int cin,
                    int h, int wd, int cout, int k, int d, int act, void *ws, size_t ws_bytes,
                    cudaStream_t st, int f16_ok) {
    int e = (k - 1) * d + 1;
    return tf_launch(x, w, b, y, nullptr, n, cin, h, wd, cout, h - e + 1, wd - e + 1, k, d, 0, act,
                     0, false, ws, ws_bytes, st, f16_ok);
}

int tf_conv_backward_data(const float *dy, const float *w, float *dx, int n, int cout, int ho,
                          int wo, int cin, int k, int d, const float *gate, int gate_kind,
                          void *ws, size_t ws_bytes, cudaStream_t st) {
    int e = (k - 1) * d + 1;
    return tf_launch(dy, w, nullptr, dx, gate, n, cout, ho, wo, cin, ho + e - 1, wo + e - 1, k, d,
                     e - 1, 0, gate_kind, true, ws, ws_bytes, st);
}

}  // namespace dp
