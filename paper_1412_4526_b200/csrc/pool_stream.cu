// Streaming max-pool kernels (sm_100a), fp32 with uint8 argmax codes: one warp per strip of
// output columns (forward: 128, backward: 4 * (32 - NL)) x MS_RS rows, walking the rows with a
// cp.async ring of staged input rows (MS_NBF / MS_NBB rows in flight per warp).  Warps are independent
// (no __syncthreads); every lane owns 4 consecutive columns, so staging, smem reads and
// global stores are 16-byte vectors.  The shared-memory tile kernels in pool.cu were issue
// bound (ncu issue-active 73-84 %, DRAM 22-52 %, profiles/r02_ncu_c3.md) at ~100-130
// instructions per output; these spend ~30.  Results are bit-identical to pool.cu's kernels
// and to the reference (_kernels.pyx:133-191):
//  * forward: separable first-wins max.  Row pass: per input row, the first-wins max of the
//    P taps j*D of each column (best starts at -inf with strict '>', so NaN never wins and
//    the first of equal taps is kept); column pass: the first-wins max over the P row-pass
//    results i*D below; code = i*P + j is the reference's raster-first argmax (the first row
//    holding the window maximum, then its first column).  Fused nonlinearity.
//  * backward: ordered scatter.  Every window (u, v) adds dy to the input pixel its code
//    names.  Window rows are processed in ascending u and, inside a row, every lane applies
//    the windows of its left neighbours (received by shuffle) before its own, i.e. in
//    ascending v -- exactly the reference's row-major scatter order (_kernels.pyx:169-191),
//    so each pixel sums its contributions in the reference's order.  The accumulators are
//    lane-private smem rows (a ring of (P-1)*D+1 pixel rows, stored column-interleaved so
//    the scattered read-modify-writes are bank-conflict free); a pixel row is complete, and
//    written, once its last window row has been applied.  Out-of-map windows are zero-filled
//    (code 0, dy +0.0): adding +0.0 to an accumulator that started at +0.0 never changes
//    its bits (round-to-nearest never produces -0.0 from +0.0 + x).
#include <stdlib.h>

#include "dp_common.cuh"
#include "tc_ptx.cuh"

namespace dp {

// staged rows in flight per warp (powers of two): occupancy, not prefetch depth, set the pace
// (c3 pool1 fwd 679 / 650 / 648 us and pool2 bwd 638 / 603 / 587 us at 8 / 4 / 2 rows)
#ifndef DP_MS_NBF
#define DP_MS_NBF 4
#endif
constexpr int MS_NBF = DP_MS_NBF;  // forward (DP_NVCC_EXTRA=-DDP_MS_NBF=<n>: experiments)
constexpr int MS_NBB = 2;    // backward
constexpr int MS_RS = 64;    // output (forward) / pixel (backward) rows per work item
constexpr int MS_WARPS = 4;  // independent warps per CTA

__host__ __device__ constexpr int ms_pow2(int v) { return v <= 1 ? 1 : 2 * ms_pow2((v + 1) / 2); }

template <int P, int D>
struct MsFwd {
    static constexpr int HALO = (P - 1) * D;
    static constexpr int NC = 32 + (HALO + 3) / 4 + 1;  // 16-byte chunks per staged row
    static constexpr int RW = 4 * NC;                   // floats per staged row
    static constexpr int RING = ms_pow2(HALO + 1);      // row-pass results kept per lane
    // p = 4: row pairs (u, u + D) kept for the column pass (out(u) = pair(u) vs pair(u + 2D))
    static constexpr int PRING = P == 4 ? ms_pow2(2 * D + 1) : 0;
    static constexpr size_t WARP_BYTES =
        (size_t)MS_NBF * RW * 4 + (size_t)(RING + PRING) * (128 + 32) * 4;
};

// first-wins (strict '>') merge of a later candidate into (v, c), codes packed 4 per word:
// byte m of the result is the candidate's when its value m is greater
__device__ __forceinline__ void ms_merge4(float v[4], uint32_t &c, const float t[4],
                                          uint32_t cand) {
#pragma unroll
    for (int m = 0; m < 4; ++m)
        if (t[m] > v[m]) {
            v[m] = t[m];
            c = __byte_perm(c, cand, (0x3210 & ~(0xF << (4 * m))) | ((4 + m) << (4 * m)));
        }
}

template <int P, int D>
struct MsBwd {
    static constexpr int HALO = (P - 1) * D;
    static constexpr int NL = (HALO + 3) / 4;      // halo lanes: feed right neighbours only
    static constexpr int PX = 4 * (32 - NL);       // pixel columns per strip
    static constexpr int RING = ms_pow2(HALO + 1);  // pixel rows accumulated at once
    static constexpr size_t WARP_BYTES = (size_t)MS_NBB * 32 * (16 + 4) + (size_t)RING * 128 * 4;
};

// row pass of one staged row (S = the row's float shift inside its 16-byte staging):
// best[m] / code byte m = first-wins max over taps j*D of column 4*lane + m
template <int P, int D, int S>
__device__ __forceinline__ void ms_rowpass(const float *row, float best[4], uint32_t &codes) {
    constexpr int NV = 4 + (P - 1) * D;
    constexpr int NF = (S + NV + 3) / 4;
    float b[4 * NF];
#pragma unroll
    for (int k = 0; k < NF; ++k) {
        const float4 f = reinterpret_cast<const float4 *>(row)[k];
        b[4 * k] = f.x;
        b[4 * k + 1] = f.y;
        b[4 * k + 2] = f.z;
        b[4 * k + 3] = f.w;
    }
    uint32_t cw = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        float bb = fmaxf(b[S + m], neg_inf<float>());  // -inf when the first tap is NaN
        uint32_t c = 0;
#pragma unroll
        for (int j = 1; j < P; ++j) {
            const float t = b[S + m + j * D];
            if (t > bb) {
                bb = t;
                c = j;
            }
        }
        best[m] = bb;
        cw |= c << (8 * m);
    }
    codes = cw;
}

// the fused nonlinearity on 4 values, one (warp-uniform) branch per call
__device__ __forceinline__ void ms_act4(float o[4], int act) {
    if (act == DP_TANH_FAST) {
#pragma unroll
        for (int m = 0; m < 4; ++m) o[m] = dp_tanh_fast(o[m]);
    } else if (act != DP_IDENTITY) {
#pragma unroll
        for (int m = 0; m < 4; ++m) o[m] = apply_nonlin(o[m], act);
    }
}

template <int P, int D>
__global__ void __launch_bounds__(MS_WARPS * 32)
    maxpool_fwd_stream(const float *__restrict__ x, float *__restrict__ y,
                       uint8_t *__restrict__ arg, int H, int W, int Ho, int Wo, int act,
                       int sx_n, int sy_n, long long items, int vec, __half *__restrict__ yh,
                       __half *__restrict__ yl, int yp) {
    using G = MsFwd<P, D>;
    extern __shared__ __align__(16) unsigned char ms_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *xs = reinterpret_cast<float *>(ms_raw + wid * G::WARP_BYTES);
    float *rv = xs + MS_NBF * G::RW;                                    // [RING][128]
    uint32_t *rc = reinterpret_cast<uint32_t *>(rv + G::RING * 128);  // [RING][32]
    float *pv = reinterpret_cast<float *>(rc + G::RING * 32);          // [PRING][128]
    uint32_t *pc = reinterpret_cast<uint32_t *>(pv + G::PRING * 128);  // [PRING][32]
    const long long nw = (long long)gridDim.x * MS_WARPS;
    for (long long it = (long long)blockIdx.x * MS_WARPS + wid; it < items; it += nw) {
        const int sx = (int)(it % sx_n);
        const long long rest = it / sx_n;
        const int sy = (int)(rest % sy_n);
        const long long plane = rest / sy_n;
        const int x0 = sx * 128, u0 = sy * MS_RS;
        const int nout = min(MS_RS, Ho - u0);
        const int nin = nout + G::HALO;
        // input row k of the item starts at element e0 + k * W of x; it is staged from the
        // 16-byte boundary at or below it, so its float shift inside the staging is
        // (e0 + k * W) & 3 (x itself is 16-byte aligned, checked by the launcher).  Row
        // pointers and shifts advance incrementally (per-row 64-bit index math was ~40 % of
        // the first version's instructions, ncu)
        const long long e0 = (plane * H + u0) * (long long)W + x0;
        const int avail0 = W - x0;  // valid floats of a row from its column x0
        const int w3 = W & 3;
        const float *sp = x + e0;   // column x0 of the next row to stage
        int ssh = (int)(e0 & 3);    // its shift
        int k_st = 0;               // next row to stage
        auto stage = [&]() {
            if (k_st < nin) {
                const float *base = sp - ssh;
                const int avail = ssh + avail0;
                float *dst = xs + (k_st & (MS_NBF - 1)) * G::RW;
                if (avail >= 4 * G::NC) {
#pragma unroll
                    for (int c = lane; c < G::NC; c += 32) ptx::cp_async16(dst + 4 * c, base + 4 * c, 16);
                } else {
#pragma unroll
                    for (int c = lane; c < G::NC; c += 32) {
                        const int nb = min(max(avail - 4 * c, 0), 4) * 4;
                        ptx::cp_async16(dst + 4 * c, nb ? base + 4 * c : base, nb);
                    }
                }
                sp += W;
                ssh = (ssh + w3) & 3;
            }
            ++k_st;
            ptx::cp_async_commit();
        };
        int psh = (int)(e0 & 3);  // shift of the row being processed
        // row pass of row k into the lane-private ring slot k % RING; p = 4 also forms the
        // pair (k - D, k) into the pair ring, returned in (prv, prc)
        float prv[4];
        uint32_t prc = 0;
        auto rowstep = [&](int k) {
            __syncwarp();  // every lane is done with the slot the next stage overwrites
            stage();
            ptx::cp_async_wait_group(MS_NBF - 1);
            __syncwarp();
            const float *row = xs + (k & (MS_NBF - 1)) * G::RW + 4 * lane;
            float best[4];
            uint32_t cw;
            switch (psh) {
                case 0: ms_rowpass<P, D, 0>(row, best, cw); break;
                case 1: ms_rowpass<P, D, 1>(row, best, cw); break;
                case 2: ms_rowpass<P, D, 2>(row, best, cw); break;
                default: ms_rowpass<P, D, 3>(row, best, cw); break;
            }
            psh = (psh + w3) & 3;
            const int slot = k & (G::RING - 1);
            *reinterpret_cast<float4 *>(rv + slot * 128 + 4 * lane) =
                make_float4(best[0], best[1], best[2], best[3]);
            rc[slot * 32 + lane] = cw;
            if constexpr (P == 4) {
                if (k >= D) {
                    const int s0 = (k - D) & (G::RING - 1);
                    const float4 f = *reinterpret_cast<const float4 *>(rv + s0 * 128 + 4 * lane);
                    prv[0] = f.x, prv[1] = f.y, prv[2] = f.z, prv[3] = f.w;
                    prc = rc[s0 * 32 + lane];
                    ms_merge4(prv, prc, best, cw + (uint32_t)P * 0x01010101u);
                    const int ps = (k - D) & (G::PRING - 1);
                    *reinterpret_cast<float4 *>(pv + ps * 128 + 4 * lane) =
                        make_float4(prv[0], prv[1], prv[2], prv[3]);
                    pc[ps * 32 + lane] = prc;
                }
            }
        };
#pragma unroll 1
        for (int k = 0; k < MS_NBF - 1; ++k) stage();
#pragma unroll 1
        for (int k = 0; k < G::HALO; ++k) rowstep(k);
        float *yo = y + (plane * Ho + u0) * (long long)Wo + x0 + 4 * lane;
        uint8_t *ao = arg + (plane * Ho + u0) * (long long)Wo + x0 + 4 * lane;
        const int cols = Wo - x0 - 4 * lane;
        const bool vfull = vec && cols >= 4;
#pragma unroll 1
        for (int u = 0; u < nout; ++u, yo += Wo, ao += Wo) {
            rowstep(u + G::HALO);
            // column pass: output row u over the row-pass rows u + i*D; the codes stay packed
            // 4 per word (candidate word of row i = its row codes + i*P per byte)
            float ob[4];
            uint32_t oc;
            if constexpr (P == 4) {
                // pair(u) (rows u, u + D) vs pair(u + 2D), just formed: first-wins over the
                // four rows in order, as the sequential scan
                const int s0 = u & (G::PRING - 1);
                const float4 f = *reinterpret_cast<const float4 *>(pv + s0 * 128 + 4 * lane);
                oc = pc[s0 * 32 + lane];
                ob[0] = f.x, ob[1] = f.y, ob[2] = f.z, ob[3] = f.w;
                ms_merge4(ob, oc, prv, prc + (uint32_t)(2 * P) * 0x01010101u);
            } else {
                {
                    const int s0 = u & (G::RING - 1);
                    const float4 f = *reinterpret_cast<const float4 *>(rv + s0 * 128 + 4 * lane);
                    oc = rc[s0 * 32 + lane];
                    ob[0] = f.x, ob[1] = f.y, ob[2] = f.z, ob[3] = f.w;
                }
#pragma unroll
                for (int i = 1; i < P; ++i) {
                    const int si = (u + i * D) & (G::RING - 1);
                    const float4 f = *reinterpret_cast<const float4 *>(rv + si * 128 + 4 * lane);
                    const uint32_t cand = rc[si * 32 + lane] + (uint32_t)(i * P) * 0x01010101u;
                    const float t[4] = {f.x, f.y, f.z, f.w};
                    ms_merge4(ob, oc, t, cand);
                }
            }
            ms_act4(ob, act);
            if (yh) {
                // the fp16 weight gradient's split of this output (rows of yp halves)
                const long long ho_ = (plane * Ho + u0 + u) * (long long)yp + x0 + 4 * lane;
                uint32_t h2[2], l2[2];
                ptx::f16_split2_scaled(ob[0], ob[1], h2[0], l2[0]);
                ptx::f16_split2_scaled(ob[2], ob[3], h2[1], l2[1]);
                if (cols >= 4) {
                    *reinterpret_cast<uint2 *>(yh + ho_) = make_uint2(h2[0], h2[1]);
                    *reinterpret_cast<uint2 *>(yl + ho_) = make_uint2(l2[0], l2[1]);
                } else {
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        if (m < cols) {
                            yh[ho_ + m] = reinterpret_cast<const __half *>(h2)[m];
                            yl[ho_ + m] = reinterpret_cast<const __half *>(l2)[m];
                        }
                }
            }
            if (vfull) {
                *reinterpret_cast<float4 *>(yo) = make_float4(ob[0], ob[1], ob[2], ob[3]);
                *reinterpret_cast<uint32_t *>(ao) = oc;
            } else {
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    if (m < cols) {
                        yo[m] = ob[m];
                        ao[m] = (uint8_t)(oc >> (8 * m));
                    }
            }
        }
        ptx::cp_async_wait_group(0);
    }
}

template <int P, int D>
__global__ void __launch_bounds__(MS_WARPS * 32)
    maxpool_bwd_stream(const float *__restrict__ dy, const uint8_t *__restrict__ arg,
                       float *__restrict__ dx, const float *__restrict__ gate, int Ho, int Wo,
                       int Hi, int Wi, int Wd, int gate_kind, int sx_n, int sy_n,
                       long long items, int vec, int gvec) {
    // gvec: gate rows 16-byte aligned (staged as one chunk per lane, else 4 words)
    using G = MsBwd<P, D>;
    constexpr int NL = G::NL;
    extern __shared__ __align__(16) unsigned char ms_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t wbytes = G::WARP_BYTES + (gate ? MS_NBB * 128 * 4 : 0);
    float *dys = reinterpret_cast<float *>(ms_raw + wid * wbytes);    // [NB][128]
    uint32_t *cs = reinterpret_cast<uint32_t *>(dys + MS_NBB * 128);  // [NB][32]
    float *acc = reinterpret_cast<float *>(cs + MS_NBB * 32);          // [RING][4][32]
    float *gs = acc + G::RING * 128;                                   // [NB][128] (gate)
    const long long nw = (long long)gridDim.x * MS_WARPS;
    for (long long it = (long long)blockIdx.x * MS_WARPS + wid; it < items; it += nw) {
        const int sx = (int)(it % sx_n);
        const long long rest = it / sx_n;
        const int sy = (int)(rest % sy_n);
        const long long plane = rest / sy_n;
        const int x0 = sx * G::PX, r0 = sy * MS_RS;
        const int nout = min(MS_RS, Hi - r0);
        const int nwin = nout + G::HALO;  // window rows r0 - HALO .. r0 + nout - 1
        const int v0 = x0 + 4 * (lane - NL);  // this lane's 4 windows
        const bool colok = v0 >= 0 && v0 < Wo;
        const long long pbase = plane * Ho * (long long)Wo;
        const int gcols = min(max(Wi - v0, 0), 4);  // gate / pixel columns of this lane
        auto stage = [&](int k) {
            const int u = r0 - G::HALO + k;
            const bool ok = colok && k < nwin && u >= 0 && u < Ho;
            const long long off = pbase + (long long)(ok ? u : 0) * Wo + (ok ? v0 : 0);
            const int sl = k & (MS_NBB - 1);
            ptx::cp_async16(dys + sl * 128 + 4 * lane, dy + off, ok ? 16 : 0);
            ptx::cp_async4(cs + sl * 32 + lane, arg + off, ok ? 4 : 0);
            if (gate) {  // the gate row of pixel row u, when the item writes that row
                const bool gok = k < nwin && u >= r0 && lane >= NL && gcols > 0;
                const float *g = gate + (gok ? (plane * Hi + u) * (long long)Wi + v0 : 0);
                float *gd = gs + sl * 128 + 4 * lane;
                if (gvec) {
                    ptx::cp_async16(gd, g, gok ? 4 * gcols : 0);
                } else {
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        ptx::cp_async4(gd + m, gok && m < gcols ? g + m : g,
                                       gok && m < gcols ? 4 : 0);
                }
            }
            ptx::cp_async_commit();
        };
#pragma unroll
        for (int e = 0; e < G::RING * 4; ++e) acc[e * 32 + lane] = 0.f;
#pragma unroll 1
        for (int k = 0; k < MS_NBB - 1; ++k) stage(k);
#pragma unroll 1
        for (int k = 0; k < nwin; ++k) {
            stage(k + MS_NBB - 1);
            ptx::cp_async_wait_group(MS_NBB - 1);  // this lane's own copies of row k landed
            const int u = r0 - G::HALO + k;
            const int sl = k & (MS_NBB - 1);
            const float4 f = *reinterpret_cast<const float4 *>(dys + sl * 128 + 4 * lane);
            const uint32_t cw = cs[sl * 32 + lane];
            const float dv[4] = {f.x, f.y, f.z, f.w};
            // key = owner lane << 16 | accumulator index of the pixel the window names
            int key[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int c = (cw >> (8 * m)) & 0xff;
                const int i = c / P, j = c - (c / P) * P;
                const int rel = 4 * (lane - NL) + m + j * D;  // target column - x0
                const int owner = (rel >> 2) + NL;
                const int slot = (u + i * D) & (G::RING - 1);
                key[m] = (owner << 16) | (slot * 128 + (rel & 3) * 32 + (owner & 31));
            }
            // left neighbours' windows first (ascending v), then this lane's own
#pragma unroll
            for (int q = NL; q >= 1; --q) {
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int kk = __shfl_up_sync(0xffffffffu, key[m], q);
                    const float dd = __shfl_up_sync(0xffffffffu, dv[m], q);
                    if (lane >= q && (kk >> 16) == lane) {
                        float *p = acc + (kk & 0xffff);
                        *p = __fadd_rn(*p, dd);
                    }
                }
            }
#pragma unroll
            for (int m = 0; m < 4; ++m)
                if ((key[m] >> 16) == lane) {
                    float *p = acc + (key[m] & 0xffff);
                    *p = __fadd_rn(*p, dv[m]);
                }
            // pixel row u is complete: write it (inside the item) and recycle its slot
            float *ar = acc + (u & (G::RING - 1)) * 128 + lane;
            if (u >= r0 && lane >= NL) {
                const int px = x0 + 4 * (lane - NL);
                const int cols = Wi - px;
                if (cols > 0) {
                    float o[4] = {ar[0], ar[32], ar[64], ar[96]};
                    if (gate) {
                        const float4 g4 = *reinterpret_cast<const float4 *>(gs + sl * 128 + 4 * lane);
                        o[0] = gate_from_output(o[0], g4.x, gate_kind);
                        o[1] = gate_from_output(o[1], g4.y, gate_kind);
                        o[2] = gate_from_output(o[2], g4.z, gate_kind);
                        o[3] = gate_from_output(o[3], g4.w, gate_kind);
                    }
                    float *d = dx + (plane * Hi + u) * (long long)Wd + px;
                    if (vec && cols >= 4) {
                        *reinterpret_cast<float4 *>(d) = make_float4(o[0], o[1], o[2], o[3]);
                    } else {
#pragma unroll
                        for (int m = 0; m < 4; ++m)
                            if (m < cols) d[m] = o[m];
                    }
                }
            }
            ar[0] = 0.f;
            ar[32] = 0.f;
            ar[64] = 0.f;
            ar[96] = 0.f;
        }
        ptx::cp_async_wait_group(0);
    }
}

static int g_ms_sms = 0;

static int ms_grid(const void *kern, size_t smem, long long items) {
    if (g_ms_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_ms_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_ms_sms <= 0) g_ms_sms = 148;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, MS_WARPS * 32, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const long long want = (items + MS_WARPS - 1) / MS_WARPS;
    const long long cap = (long long)g_ms_sms * per_sm;
    return (int)(want < cap ? want : cap);
}

template <int P, int D>
static int ms_fwd_launch(const float *x, float *y, uint8_t *arg, long long planes, int h, int w,
                         int ho, int wo, int act, cudaStream_t st, __half *yh, __half *yl,
                         int yp) {
    using G = MsFwd<P, D>;
    const size_t smem = MS_WARPS * G::WARP_BYTES;
    auto kern = maxpool_fwd_stream<P, D>;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return set_error(DP_ERR_CUDA, "maxpool_fwd_stream: smem attribute");
    const int sx_n = ceil_div(wo, 128), sy_n = ceil_div(ho, MS_RS);
    const long long items = planes * sx_n * sy_n;
    const int vec = (wo % 4 == 0) && ((uintptr_t)y % 16 == 0) && ((uintptr_t)arg % 4 == 0);
    if ((uintptr_t)x % 16 != 0) return -1;  // rows are staged from 16-byte boundaries of x
    kern<<<ms_grid((const void *)kern, smem, items), MS_WARPS * 32, smem, st>>>(
        x, y, arg, h, w, ho, wo, act, sx_n, sy_n, items, vec, yh, yl, yp);
    return check_launch("maxpool_fwd_stream");
}

template <int P, int D>
static int ms_bwd_launch(const float *dy, const uint8_t *arg, float *dx, const float *gate,
                         long long planes, int ho, int wo, int hi, int wi, int wd, int gate_kind,
                         cudaStream_t st) {
    using G = MsBwd<P, D>;
    const size_t smem = MS_WARPS * (G::WARP_BYTES + (gate ? MS_NBB * 128 * 4 : 0));
    auto kern = maxpool_bwd_stream<P, D>;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return set_error(DP_ERR_CUDA, "maxpool_bwd_stream: smem attribute");
    const int sx_n = ceil_div(wi, G::PX), sy_n = ceil_div(hi, MS_RS);
    const long long items = planes * sx_n * sy_n;
    const int vec = (wd % 4 == 0) && ((uintptr_t)dx % 16 == 0);
    const int gvec = (wi % 4 == 0) && ((uintptr_t)gate % 16 == 0);
    kern<<<ms_grid((const void *)kern, smem, items), MS_WARPS * 32, smem, st>>>(
        dy, arg, dx, gate, ho, wo, hi, wi, wd, gate_kind, sx_n, sy_n, items, vec, gvec);
    return check_launch("maxpool_bwd_stream");
}

#define MS_PD_SWITCH(P_, D_, CALL)                     \
    switch ((P_) * 100 + (D_)) {                       \
        case 201: return CALL(2, 1);                   \
        case 202: return CALL(2, 2);                   \
        case 204: return CALL(2, 4);                   \
        case 208: return CALL(2, 8);                   \
        case 216: return CALL(2, 16);                  \
        case 301: return CALL(3, 1);                   \
        case 302: return CALL(3, 2);                   \
        case 304: return CALL(3, 4);                   \
        case 308: return CALL(3, 8);                   \
        case 401: return CALL(4, 1);                   \
        case 402: return CALL(4, 2);                   \
        case 404: return CALL(4, 4);                   \
        case 801: return CALL(8, 1);                   \
        default: return -1;                            \
    }

static bool ms_enabled() {
    const char *e = getenv("DP_POOL_STREAM");
    return !(e && e[0] == '0');
}

// -1: not applicable (the caller uses pool.cu's kernels); else DP_OK / an error code
// yh / yl (or null): also write the output's fp16 split (hi, lo' = (y - hi) * 2^11) in rows
// of yp halves (yp % 4 == 0, 8-byte aligned; columns past wo are left untouched)
int maxpool_forward_stream(const float *x, float *y, void *arg, int arg_bytes, long long planes,
                           int h, int w, int p, int d, int act, cudaStream_t st, void *yh,
                           void *yl, int yp) {
    // p = 2 stays on pool.cu's register-tile kernel except at d = 4..8 (c3 pool2: 0.50 ->
    // 0.47 ms here; d = 1 / 2 / 16 measured 3-65 % slower: two taps per output leave the
    // streaming overhead unamortised)
    const bool p2ok = (d >= 4 && d <= 8) || getenv("DP_POOL_STREAM_P2");
    if (arg_bytes != 1 || !ms_enabled() || (p < 3 && !p2ok)) return -1;
    const int ho = h - (p - 1) * d, wo = w - (p - 1) * d;
    if (yh && (yp < wo || (yp & 3) || ((uintptr_t)yh & 7) || ((uintptr_t)yl & 7))) return -1;
#define MS_F(PP, DD)                                                                    \
    ms_fwd_launch<PP, DD>(x, y, (uint8_t *)arg, planes, h, w, ho, wo, act, st, (__half *)yh, \
                          (__half *)yl, yp)
    MS_PD_SWITCH(p, d, MS_F)
#undef MS_F
}

int maxpool_backward_stream(const float *dy, const void *arg, int arg_bytes, float *dx,
                            long long planes, int ho, int wo, int p, int d, int hi, int wi,
                            const float *gate, int gate_kind, int wd, cudaStream_t st) {
    // windows are staged as whole 16-byte chunks: rows of 4k windows, aligned maps
    // (halos beyond 8 columns measured slower than pool.cu's kernels: c4's p2/d16 pool)
    if (arg_bytes != 1 || !ms_enabled() || wo % 4 != 0 || (uintptr_t)dy % 16 != 0 ||
        (uintptr_t)arg % 4 != 0 || (p - 1) * d > 8)
        return -1;
    // a gate whose rows are not 16-byte aligned is staged word by word: slower than pool.cu
    if (gate && (wi % 4 != 0 || (uintptr_t)gate % 16 != 0)) return -1;
#define MS_B(PP, DD)                                                                        \
    ms_bwd_launch<PP, DD>(dy, (const uint8_t *)arg, dx, gate, planes, ho, wo, hi, wi, wd, \
                          gate_kind, st)
    MS_PD_SWITCH(p, d, MS_B)
#undef MS_B
}

}  // namespace dp
