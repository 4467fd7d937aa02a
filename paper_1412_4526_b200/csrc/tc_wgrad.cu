// Weight / bias gradient of the d-regularly sparse convolution on the tcgen05 tensor
// cores (sm_100a), fp32 in/out with 3xTF32 products -- the fast tier of
// conv_backward_kernel (reference _kernels.pyx:94-130, _kernels_py.py:54-66):
//
//   dw[o,c,i,j] = sum_{n,u,v} dy[n,o,u,v] * x[n,c,u+i*d,v+j*d]      db[o] = sum dy[n,o,u,v]
//
// As a GEMM  D[r, o] = sum_k A[r, k] * B[o, k]  with
//   r = tap*Cpad + c   (tap = i*l + j; Cpad = cin rounded up to 8)  -> M, tiles of 128 rows
//   o                  (cout rounded up to 16 = Npad)                -> N
//   k = output pixel   (n, u, v), blocks of 32 consecutive v         -> K (the long axis)
// A[r, k] = x[n, c, u+i*d, v+j*d], B[o, k] = dy[n, o, u, v].
//
// Staging (shared memory, one stage per 32-pixel K block, filled by 2-5 large TMA boxes):
//   x is first copied (tc_stage_x) into a layout (n, h, c, wp) with 16-byte row pitch;
//   tensor maps over it use OVERLAPPING strides so that one box gathers every tap the
//   K block needs:
//   * tap mode (d % 4 == 0): dims (w, j: stride d, c, i: stride d rows, row), box
//     {32, l, C, l, 1} -> lines [i][c][j] of 128 B (SWIZZLE_128B), exactly the A rows;
//   * halo mode (otherwise: TMA box columns must start 16-byte aligned, and j*d is not):
//     dims (w, c, i: stride d rows, row), box {L, C, l, 1} with L = 32 + (l-1)*d
//     rounded to an odd multiple of 4 floats -> "halo segments" [i][c][L]; tap (i, j)
//     is the window at j*d inside segment (i, c).  Windows must start 16-byte aligned
//     too, so x is staged as copies shifted left by b = (j*d) & 3 (one box per residue
//     that occurs); window (i, j) reads copy b at offset j*d - b.
//   B = dy is one box {32, 1, Npad, 1} in the canonical SWIZZLE_128B K-major layout (TMA
//   zero-fills o >= cout and v >= wo; the latter also cancels A columns past the row
//   end); B_lo is written next to it by the converters.
//   Measured on B200 (tools/load_probe.cu, tools/wg_trace.py): 16-byte cp.async tops
//   out near 15 B/cycle/SM for these line patterns and small 2 KB TMA boxes near
//   15-25 B/cycle, while 16-64 KB boxes reach ~80 B/cycle from L2 -- hence a few big
//   boxes per K block rather than one copy per tap line.
//
// 3xTF32: D = A_hi B_hi + A_lo B_hi + A_hi B_lo (hi = raw bits, the tensor core truncates;
// lo = x - trunc(x), exact).  Per K=8 slice and 128-row tile the MMA warp issues
//   A_hi x [B_hi | B_lo]  (N = 2*Npad, one instruction)  +  A_lo x B_hi  (N = Npad)
// with both A operands in TMEM: converter warps read their row's 8 values of the slice
// (two 16-byte loads, bank-conflict free: swizzled lines in tap mode, an odd segment
// pitch L/4 in halo mode) and write (hi, lo) with tcgen05.st (lane = row).
//
// Split-K across CTAs: CTA (g, s) owns tile group g and K blocks s, s + splits, ...
// (interleaved, so concurrently running CTAs share image rows in L2); accumulators stay
// in TMEM and are written once to partials [s][row][o]; a second kernel sums splits in a
// fixed order -- run-to-run deterministic, no float atomics.  db is accumulated by the
// converter threads from the B tiles (fixed thread -> row mapping).
//
// Roles (one CTA per SM):
//   warps 0-7   converters, two groups of 4 (warp % 4 = TMEM lane quarter); group p
//               converts K blocks p, p+2, ... (B_lo, db, all slices of all tiles into one
//               TMEM stage); both groups run the epilogue
//   warp 8      TMA producer (one lane)
//   warp 9      TMEM allocator + MMA issuer (one elected lane)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>

#include "dp_common.cuh"
#include "tc_ptx.cuh"

namespace dp {

constexpr int WG_CONV_WARPS = 8;
constexpr int WG_TMA_WARP = 8;
constexpr int WG_MMA_WARP = 9;
constexpr int WG_THREADS = 320;
static_assert(WG_TMA_WARP == WG_CONV_WARPS && WG_THREADS == (WG_MMA_WARP + 1) * 32,
              "warp roles");
constexpr int WG_MAX_G = 2;
constexpr int WG_MAX_SS = 8;
constexpr int WG_MAX_TS = 16;
constexpr int WG_KSTEPS = 4;          // K=8 slices per 32-pixel K block
constexpr int WG_MAX_L4 = 64;         // halo segment length <= 256 floats (TMA box dim)
constexpr int WG_SMEM_BUDGET = 216 * 1024;

struct TcWgradArgs {
    int C, Cpad, l, d, Q, Npad;
    int rows_total, n_tiles, G, n_groups, splits;
    int Ho, Wo, nvb;          // output (= dy) height / width, 32-px blocks per row
    long long kb_total;       // n * Ho * nvb
    int SS, TS;               // shared-memory stages (K blocks), TMEM A stages (K slices)
    int tap_mode;             // 1: boxes of per-tap lines (d % 4 == 0), 0: halo segments
    int L4, n_b, shift_mask;  // segment length / 4 (odd), staged x copies and their residues
    uint32_t b_bytes;         // B_hi + B_lo bytes at the start of a stage (2 * Npad * 128)
    uint32_t box_bytes;       // one x box (aligned to 1024 in the stage)
    uint32_t box_tx;          // bytes one x box delivers
    uint32_t stage_bytes;
    int Hi;
    float *part;              // [splits][n_tiles*128][Npad]
    float *pdb;               // [splits][Npad]
    unsigned long long *trace;  // DP_WG_TRACE: per-K-block timestamps of CTA 0
    int dbg;                  // DP_WG_DBG: 2 no MMA, 8 no x boxes, 32 no converter work,
                              // 64 contiguous K ranges
};

#define WG_TRACE(A, KL, SLOT, COND)                                               \
    do {                                                                          \
        if ((A).trace && (COND) && blockIdx.x == 0 && (KL) < 256)                 \
            (A).trace[(KL) * 16 + (SLOT)] = clock64();                            \
    } while (0)

// first tap row i and number of tap rows touched by the tile group starting at tile0
__host__ __device__ inline void wg_i_range(int rows_total, int Cpad, int l, int tile0, int G,
                                           int &i_lo, int &n_i) {
    const int r_lo = tile0 * 128;
    const int r_hi = (rows_total < (tile0 + G) * 128 ? rows_total : (tile0 + G) * 128) - 1;
    i_lo = (r_lo / Cpad) / l;
    n_i = (r_hi / Cpad) / l - i_lo + 1;
}

__global__ void __launch_bounds__(WG_THREADS, 1)
tc_wgrad_kernel(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_x1,
                const __grid_constant__ CUtensorMap tm_x2, const __grid_constant__ CUtensorMap tm_x3,
                const __grid_constant__ CUtensorMap tm_dy, const TcWgradArgs a) {
    extern __shared__ __align__(1024) unsigned char wg_smem_raw[];
    __shared__ uint64_t sfull[WG_MAX_SS], sempty[WG_MAX_SS];
    __shared__ uint64_t tfull[WG_MAX_TS], accfull;
    __shared__ uint32_t s_tmem;

    unsigned char *smem = (unsigned char *)(((uintptr_t)wg_smem_raw + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x % a.n_groups, split = blockIdx.x / a.n_groups;
    const int tile0 = g * a.G;
    const int G = min(a.G, a.n_tiles - tile0);
    // K blocks of split s: interleaved s, s + splits, ... (default) or, with DP_WG_DBG & 64,
    // one contiguous range
    const bool contig = (a.dbg & 64) != 0;
    const long long kb_first = contig ? a.kb_total * split / a.splits : split;
    const int kb_step = contig ? 1 : a.splits;
    const int nkb = contig ? (int)(a.kb_total * (split + 1) / a.splits - kb_first)
                           : (int)((a.kb_total - split + a.splits - 1) / a.splits);
    const int acc_cols = 2 * a.Npad;
    const int L = a.L4 * 4;
    int i_lo, n_i;
    wg_i_range(a.rows_total, a.Cpad, a.l, tile0, G, i_lo, n_i);

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.SS; ++s) {
            ptx::mbar_init(&sfull[s], 1);
            ptx::mbar_init(&sempty[s], 1);
        }
        for (int s = 0; s < a.TS; ++s) {
            ptx::mbar_init(&tfull[s], 4);
        }
        ptx::mbar_init(&accfull, 1);
        ptx::mbar_fence_init();
    }
    if (warp == WG_TMA_WARP && lane == 0) {
        ptx::tma_prefetch_desc(&tm_dy);
        ptx::tma_prefetch_desc(&tm_x0);
    }
    if (warp == WG_MMA_WARP) ptx::tmem_alloc<512>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t a_base = tmem + (uint32_t)(a.G * acc_cols);

    if (warp == WG_TMA_WARP) {
        // ================================ TMA producer ================================
        // The whole warp walks the loop (it must reconverge before the final barrier);
        // lane 0 issues the boxes.
        const uint32_t tx = (uint32_t)a.n_b * a.box_tx + (uint32_t)a.Npad * 128u;
        for (int kl = 0; kl < nkb; ++kl) {
            const int s = kl % a.SS;
            ptx::mbar_wait(&sempty[s], ((kl / a.SS) & 1) ^ 1);
            if (lane == 0) {
                const long long kb = kb_first + (long long)kl * kb_step;
                const int vb = (int)(kb % a.nvb);
                const long long tt = kb / a.nvb;
                const int u = (int)(tt % a.Ho);
                const int img = (int)(tt / a.Ho);
                const int v0 = vb * 32;
                const int hh = img * a.Hi + u;
                unsigned char *st = smem + (size_t)s * a.stage_bytes;
                WG_TRACE(a, kl, 0, true);
                ptx::mbar_expect_tx(&sfull[s], (a.dbg & 8) ? (uint32_t)a.Npad * 128u : tx);
                ptx::tma_load_4d(st, &tm_dy, v0, u, 0, img, &sfull[s]);
                unsigned char *sa = st + a.b_bytes;
                if (a.dbg & 8) {
                    // bring-up: dy only
                } else if (a.tap_mode) {
                    ptx::tma_load_5d(sa, &tm_x0, v0, 0, 0, i_lo, hh, &sfull[s]);
                } else {
                    for (int b = 0, slot = 0; b < 4; ++b) {
                        if (!(a.shift_mask & (1 << b))) continue;
                        const CUtensorMap *m = b == 0 ? &tm_x0 : b == 1 ? &tm_x1 : b == 2 ? &tm_x2
                                                                                          : &tm_x3;
                        ptx::tma_load_4d(sa + (size_t)slot * a.box_bytes, m, v0, 0, i_lo, hh,
                                         &sfull[s]);
                        ++slot;
                    }
                }
            }
            __syncwarp();
        }
    } else if (warp == WG_MMA_WARP) {
        // ================================ MMA issuer ================================
        // One wait and one commit per K block (4 slices x G tiles x 2 MMAs): the issuing
        // thread's wait / commit / fence sequence costs ~600 cycles of serial latency,
        // so it is amortised over a whole K block rather than paid per K=8 slice.
        const uint32_t idesc_2n = ptx::idesc_tf32(128, 2 * a.Npad);
        const uint32_t idesc_n = ptx::idesc_tf32(128, a.Npad);
        const uint32_t smem_base = ptx::smem_u32(smem);
        // ring positions kept incrementally: this thread's loop is the critical path
        int s = 0, ts = 0;
        uint32_t tph = 0;
        for (int kl = 0; kl < nkb; ++kl) {
            const uint32_t bhi = smem_base + (uint32_t)s * a.stage_bytes;
            ptx::mbar_wait(&tfull[ts], tph);
            ptx::tc_fence_after();
            WG_TRACE(a, kl, 8, lane == 0);
            if (ptx::elect_one()) {
                const uint32_t abase = a_base + (uint32_t)(ts * a.G * WG_KSTEPS * 16);
                for (int ks = 0; ks < WG_KSTEPS; ++ks) {
                    const uint64_t dstack = ptx::smem_desc_sw128(bhi + ks * 32);
                    for (int t = 0; t < ((a.dbg & 2) ? 0 : G); ++t) {
                        const uint32_t dcol = tmem + (uint32_t)(t * acc_cols);
                        const uint32_t ahi = abase + (uint32_t)((ks * a.G + t) * 16), alo = ahi + 8;
                        ptx::mma_tf32_ts(dcol, ahi, dstack, idesc_2n, (kl | ks) > 0);
                        ptx::mma_tf32_ts(dcol, alo, dstack, idesc_n, 1);
                    }
                }
                // ONE commit per K block (a tcgen05.commit costs the issuing thread ~200-300
                // cycles): sempty[s] also tells the converters that TMEM stage ts is free
                // again -- they wait for the K block TS earlier (see below)
                ptx::mma_commit(&sempty[s]);
            }
            __syncwarp();
            WG_TRACE(a, kl, 9, lane == 0);
            if (++s == a.SS) s = 0;
            if (++ts == a.TS) {
                ts = 0;
                tph ^= 1;
            }
        }
        if (ptx::elect_one()) ptx::mma_commit(&accfull);
        __syncwarp();
    } else {
        // ================================ converters ================================
        const int q = warp & 3, grp = warp >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const int r = q * 32 + lane;  // row inside a tile == TMEM lane
        // byte offset of this row's 32-float line / window inside a stage's A area (-1 =
        // zero row) and its swizzle phase (tap mode: SWIZZLE_128B lines; halo: none)
        int rowoff[WG_MAX_G], rowsw[WG_MAX_G];
#pragma unroll
        for (int t = 0; t < WG_MAX_G; ++t) {
            const int rr = (tile0 + t) * 128 + r;
            int o = -1, sw = 0;
            if (t < G && rr < a.rows_total) {
                const int tap = rr / a.Cpad, c = rr - tap * a.Cpad;
                if (c < a.C) {
                    const int i = tap / a.l, j = tap - (tap / a.l) * a.l;
                    if (a.tap_mode) {
                        const int line = ((i - i_lo) * a.C + c) * a.l + j;
                        o = line * 128;
                        sw = line & 7;
                    } else {
                        const int jd = j * a.d, b = jd & 3;
                        const int slot = __popc(a.shift_mask & ((1 << b) - 1));
                        o = slot * (int)a.box_bytes + (((i - i_lo) * a.C + c) * L + (jd - b)) * 4;
                    }
                }
            }
            rowoff[t] = o;
            rowsw[t] = sw;
        }
        const int nrow_chunks = a.Npad * 8;  // 16-byte chunks of the B_hi tile
        const int dbn = a.Npad / 16;         // B rows per group-0 thread
        float dbacc[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) dbacc[m] = 0.f;
        // group p converts K blocks kl = p, p + 2, ...: B_lo + db, then all 4 slices of every
        // tile into TMEM stage kl % TS, one arrive per warp
        for (int kl = grp; kl < nkb; kl += 2) {
            const int s = kl % a.SS;
            const int ts = kl % a.TS;
            ptx::mbar_wait(&sfull[s], (kl / a.SS) & 1);
            WG_TRACE(a, kl, 2, q == 0 && lane == 0);
            unsigned char *st = smem + (size_t)s * a.stage_bytes;
            {
                // B_lo = B_hi - trunc(B_hi) (elementwise; the swizzle is preserved) + db
                const float4 *bh = reinterpret_cast<const float4 *>(st);
                float4 *bl = reinterpret_cast<float4 *>(st + (uint32_t)a.Npad * 128);
                const int tid = q * 32 + lane;  // 0..127 within the group
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    if (m >= dbn) break;
                    const int idx = tid + 128 * m;
                    if (idx >= nrow_chunks) break;
                    float4 v = bh[idx];
                    dbacc[m] += (v.x + v.y) + (v.z + v.w);
                    bl[idx] = make_float4(ptx::tf32_lo(v.x), ptx::tf32_lo(v.y),
                                          ptx::tf32_lo(v.z), ptx::tf32_lo(v.w));
                }
                ptx::fence_proxy_async_smem();
                WG_TRACE(a, kl, 3, q == 0 && lane == 0);
            }
            const unsigned char *sa = st + a.b_bytes;
            if (kl >= a.TS) {
                // TMEM stage ts was last used by K block kl - TS; its MMAs are done when
                // that block's SMEM stage is released (SS >= TS, so the parity is exact)
                const int kp = kl - a.TS;
                ptx::mbar_wait(&sempty[kp % a.SS], (kp / a.SS) & 1);
            }
            ptx::tc_fence_after();
            const uint32_t tbase = a_base + lane_off + (uint32_t)(ts * a.G * WG_KSTEPS * 16);
#pragma unroll
            for (int ks = 0; ks < WG_KSTEPS; ++ks) {
#pragma unroll
                for (int t = 0; t < WG_MAX_G; ++t) {
                    if (t >= G || (a.dbg & 32)) break;
                    float hi[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                    if (rowoff[t] >= 0) {
                        const unsigned char *row = sa + rowoff[t];
                        const float4 p0 =
                            *reinterpret_cast<const float4 *>(row + (((2 * ks) ^ rowsw[t]) << 4));
                        const float4 p1 = *reinterpret_cast<const float4 *>(
                            row + (((2 * ks + 1) ^ rowsw[t]) << 4));
                        hi[0] = p0.x; hi[1] = p0.y; hi[2] = p0.z; hi[3] = p0.w;
                        hi[4] = p1.x; hi[5] = p1.y; hi[6] = p1.z; hi[7] = p1.w;
                    }
                    float lo[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) lo[k] = ptx::tf32_lo(hi[k]);
                    const uint32_t col = tbase + (uint32_t)((ks * a.G + t) * 16);
                    ptx::tmem_st8(col, hi);
                    ptx::tmem_st8(col + 8, lo);
                }
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tfull[ts]);
            WG_TRACE(a, kl, 4, lane == 0 && q == 0);
        }
        // ---- db partials (thread q*32+lane of each group owns B rows (tid >> 3) + 16 m)
        if (g == 0) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (m >= dbn) break;
                float v = dbacc[m];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                const int row = ((q * 32 + lane) >> 3) + 16 * m;
                if ((lane & 7) == 0 && row < a.Npad)
                    a.pdb[((size_t)split * 2 + grp) * a.Npad + row] = v;
            }
        }
        // ---- epilogue: tiles t = grp, grp + 2, ... ; lane = row
        if (nkb > 0) {
            ptx::mbar_wait_sleep(&accfull, 0);
            ptx::tc_fence_after();
        }
        const size_t rows_pad = (size_t)a.n_tiles * 128;
        for (int t = grp; t < G; t += 2) {
            const int grow = (tile0 + t) * 128 + r;
            float *dst = a.part + ((size_t)split * rows_pad + grow) * a.Npad;
            for (int o0 = 0; o0 < a.Npad; o0 += 16) {
                uint32_t h[16], l2[16];
                if (nkb > 0) {
                    const uint32_t dcol = tmem + lane_off + (uint32_t)(t * acc_cols + o0);
                    ptx::tmem_ld16(dcol, h);
                    ptx::tmem_ld16(dcol + a.Npad, l2);
                    ptx::tmem_wait_ld();
                }
#pragma unroll
                for (int k = 0; k < 16; k += 4) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (nkb > 0)
                        v = make_float4(__uint_as_float(h[k]) + __uint_as_float(l2[k]),
                                        __uint_as_float(h[k + 1]) + __uint_as_float(l2[k + 1]),
                                        __uint_as_float(h[k + 2]) + __uint_as_float(l2[k + 2]),
                                        __uint_as_float(h[k + 3]) + __uint_as_float(l2[k + 3]));
                    *reinterpret_cast<float4 *>(dst + o0 + k) = v;
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == WG_MMA_WARP) ptx::tmem_dealloc<512>(tmem);
}

// dw[o,c,i,j] = sum_s part[s][(i*l+j)*Cpad + c][o], db[o] = sum_s pdb[s][o]  (fixed order)
__global__ void tc_wgrad_reduce(const float *__restrict__ part, const float *__restrict__ pdb,
                                float *__restrict__ dw, float *__restrict__ db, int Q, int C,
                                int Cpad, int l, int Npad, int splits, int rows_pad) {
    const long long total = (long long)Q * C * l * l;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < total) {
        const int ll = l * l;
        const int o = (int)(idx / ((long long)C * ll));
        const int rem = (int)(idx - (long long)o * C * ll);
        const int c = rem / ll, tap = rem - (rem / ll) * ll;
        const size_t row = (size_t)tap * Cpad + c;
        float acc = 0.f;
        for (int s = 0; s < splits; ++s) acc += part[((size_t)s * rows_pad + row) * Npad + o];
        dw[idx] = acc;
    } else if (idx < total + Q) {
        const int o = (int)(idx - total);
        float acc = 0.f;
        for (int s = 0; s < 2 * splits; ++s) acc += pdb[(size_t)s * Npad + o];
        db[o] = acc;
    }
}

// x staging: NCHW (n, c, h, w) -> copies b in `mask`, each laid out (n, h, c, wp) and
// shifted left by b columns (dst_b[n,h,c,v] = src[n,c,h,v + b], zero at v + b >= w).
// wp = w rounded up to 4 floats, so every window start j*d - b is 16-byte aligned; the
// channels of one image row are adjacent so a K block's segments are compact.
// One thread per 4 destination floats of every copy (16-byte stores; the source reads are
// unaligned scalar loads of one row segment, shared by the copies through L1).
__global__ void __launch_bounds__(256) tc_stage_x(const float *__restrict__ src,
                                                  float *__restrict__ dst, int C, int H, int w,
                                                  int wp, int mask, long long copy_stride,
                                                  long long total_quads) {
    const int nq = wp >> 2;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total_quads;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long row = idx / nq;  // (n, c, h)
        const int v = (int)(idx - row * nq) * 4;
        const int h = (int)(row % H);
        const long long nc = row / H;
        const int c = (int)(nc % C);
        const long long n = nc / C;
        const float *s = src + row * w;
        float e[7];
#pragma unroll
        for (int t = 0; t < 7; ++t) e[t] = v + t < w ? __ldg(s + v + t) : 0.f;
        float4 *d0 = reinterpret_cast<float4 *>(dst + ((n * H + h) * C + c) * wp + v);
        int slot = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (!(mask & (1 << b))) continue;
            d0[slot * (copy_stride >> 2)] = make_float4(e[b], e[b + 1], e[b + 2], e[b + 3]);
            ++slot;
        }
    }
}

// x staging, one copy per TAP (small-cin layers of the smem-operand weight gradient):
// dst_j[n,h,c,v] = src[n,c,h,v + j*d] (zero at v + j*d >= w), (n, h, c, wp) layout; a
// single TMA box with the copy stride as its tap dimension then gathers every (c, j) line
// of a row (the residue copies need one box per residue -- tiny boxes at cin = 3, d = 1).
__global__ void __launch_bounds__(256) tc_stage_x_taps(const float *__restrict__ src,
                                                       float *__restrict__ dst, int C, int H,
                                                       int w, int wp, int l, int d,
                                                       long long copy_stride,
                                                       long long total_quads) {
    const int nq = wp >> 2;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total_quads;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long row = idx / nq;  // (n, c, h)
        const int v = (int)(idx - row * nq) * 4;
        const int h = (int)(row % H);
        const long long nc = row / H;
        const int c = (int)(nc % C);
        const long long n = nc / C;
        const float *s = src + row * w;
        float4 *d0 = reinterpret_cast<float4 *>(dst + ((n * H + h) * C + c) * wp + v);
        for (int j = 0; j < l; ++j) {
            const int o = v + j * d;
            float e[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) e[t] = o + t < w ? __ldg(s + o + t) : 0.f;
            d0[j * (copy_stride >> 2)] = make_float4(e[0], e[1], e[2], e[3]);
        }
    }
}

// dy staging: NCHW (n, o, h, w) -> (n, h, o, wp), zero pad (lm zeros left of the data, lm a
// multiple of 4, the rest right of it).  A K block's dy box then reads Npad lines wp floats
// apart instead of one line per channel plane (plane-strided boxes measured ~4x slower
// here: every line opens a different DRAM page).
__global__ void __launch_bounds__(256) tc_stage_dy(const float *__restrict__ src,
                                                   float *__restrict__ dst, int O, int H, int w,
                                                   int wp, int lm, long long total_quads,
                                                   int ws,  // ws: source row pitch
                                                   const int *exit_unless) {
    // the tf32 fallback of an fp16-split weight gradient: runs only when its range flag is set
    if (exit_unless && !*(volatile const int *)exit_unless) return;
    const int nq = wp >> 2;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total_quads;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long row = idx / nq;  // (n, o, h)
        const int v = (int)(idx - row * nq) * 4;
        const int h = (int)(row % H);
        const long long no = row / H;
        const int o = (int)(no % O);
        const long long n = no / O;
        const float *s = src + row * ws;
        float e[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int c = v + t - lm;
            e[t] = (c >= 0 && c < w) ? __ldg(s + c) : 0.f;
        }
        *reinterpret_cast<float4 *>(dst + ((n * H + h) * O + o) * wp + v) =
            make_float4(e[0], e[1], e[2], e[3]);
    }
}

static int stage_grid(long long quads) {
    long long g = (quads + 255) / 256;
    return (int)(g < 148 * 64 ? g : 148 * 64);
}

// the staged copies' tails (read by the last row's out-of-row taps, which only ever meet
// zero dy) must hold zeros, not stale NaN/Inf bit patterns: 0 * NaN would poison dw
static int stage_x_tails(float *xs, long long used_floats, long long copy_floats, int mask,
                         cudaStream_t st) {
    const int ncopies = __builtin_popcount(mask);
    for (int c = 0; c < ncopies; ++c)
        if (cudaMemsetAsync(xs + c * copy_floats + used_floats, 0,
                            (size_t)(copy_floats - used_floats) * 4, st) != cudaSuccess)
            return set_error(DP_ERR_CUDA, "weight gradient: memset of staged tails failed");
    return DP_OK;
}

// --------------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------------
static unsigned long long *g_wg_trace = nullptr;

// debugging aid (tools/wg_trace.py): copy the last traced launch's timestamps
int wg_trace_copy(void *host, size_t bytes) {
    if (!g_wg_trace) return DP_ERR_ARG;
    if (bytes > 256 * 16 * 8) bytes = 256 * 16 * 8;
    return cudaMemcpy(host, g_wg_trace, bytes, cudaMemcpyDeviceToHost) == cudaSuccess
               ? DP_OK
               : DP_ERR_CUDA;
}

struct WgPlan {
    int Cpad, Npad, rows_total, n_tiles, G, n_groups, splits, SS, TS, L4, n_b, shift_mask;
    int ho, wo, nvb, wp_x, wp_dy, max_ni;
    bool tap_mode, stage_dy;
    long long kb_total;
    size_t part_bytes, pdb_bytes, copy_bytes, x_bytes, dy_bytes, total_bytes;
    uint32_t b_bytes, box_bytes, box_tx, stage_bytes;
};

static int wg_num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

// returns false when the shape is outside the kernel's envelope (caller falls back)
static bool wg_plan(int n, int cin, int hi, int wi, int cout, int k, int d, WgPlan &p) {
    const int e = (k - 1) * d + 1;
    p.ho = hi - e + 1;
    p.wo = wi - e + 1;
    if (p.ho < 1 || p.wo < 1) return false;
    p.Npad = (cout + 15) / 16 * 16;
    if (p.Npad > 128 || cin > 256 || k > 256) return false;
    p.Cpad = (cin + 7) / 8 * 8;
    p.rows_total = k * k * p.Cpad;
    p.n_tiles = (p.rows_total + 127) / 128;
    const int acc_cols = 2 * p.Npad;
    // TMEM: G tiles of accumulators + TS stages of one K block's A (4 slices x G x 16 cols)
    int G = 512 / (acc_cols + 2 * WG_KSTEPS * 16);
    if (G > WG_MAX_G) G = WG_MAX_G;
    if (const char *e = getenv("DP_WG_G")) {  // tile-group size override (experiments)
        const int v = atoi(e);
        if (v >= 1 && v < G) G = v;
    }
    if (G < 1) return false;
    p.n_groups = (p.n_tiles + G - 1) / G;
    p.G = (p.n_tiles + p.n_groups - 1) / p.n_groups;
    int TS = (512 - p.G * acc_cols) / (p.G * WG_KSTEPS * 16);
    if (TS > WG_MAX_TS) TS = WG_MAX_TS;
    if (TS < 2) return false;
    p.TS = TS;
    p.max_ni = 0;
    for (int g = 0; g < p.n_groups; ++g) {
        const int t0 = g * p.G, G_ = std::min(p.G, p.n_tiles - t0);
        int i_lo, n_i;
        wg_i_range(p.rows_total, p.Cpad, k, t0, G_, i_lo, n_i);
        p.max_ni = std::max(p.max_ni, n_i);
    }
    p.tap_mode = (d % 4) == 0;
    p.b_bytes = 2u * (uint32_t)p.Npad * 128u;
    if (p.tap_mode) {
        p.shift_mask = 1;
        p.n_b = 1;
        p.L4 = 8;
        p.box_tx = (uint32_t)p.max_ni * cin * k * 128u;
    } else {
        // residues b = (j*d) & 3 that occur; segment length an odd multiple of 4 floats
        p.shift_mask = 0;
        for (int j = 0; j < k; ++j) p.shift_mask |= 1 << ((j * d) & 3);
        p.n_b = __builtin_popcount(p.shift_mask);
        int L4 = ((((k - 1) * d) & ~3) + 32) / 4;
        if ((L4 & 1) == 0) ++L4;
        if (L4 > WG_MAX_L4) return false;
        p.L4 = L4;
        p.box_tx = (uint32_t)p.max_ni * cin * L4 * 16u;
    }
    p.box_bytes = (p.box_tx + 1023u) & ~1023u;
    p.stage_bytes = p.b_bytes + (uint32_t)p.n_b * p.box_bytes;
    int SS = WG_SMEM_BUDGET / (int)p.stage_bytes;
    if (SS > WG_MAX_SS) SS = WG_MAX_SS;
    if (SS < 2) return false;
    p.SS = SS;
    if (p.TS > p.SS) p.TS = p.SS;  // TMEM-stage reuse is read off the SMEM-stage barriers
    p.nvb = (p.wo + 31) / 32;
    p.kb_total = (long long)n * p.ho * p.nvb;
    int sms = wg_num_sms();
    p.splits = sms / p.n_groups;
    if (p.splits < 1) p.splits = 1;
    if (p.splits > p.kb_total) p.splits = (int)p.kb_total;
    p.wp_x = (wi + 3) / 4 * 4;
    p.wp_dy = (p.wo + 3) / 4 * 4;
    p.stage_dy = p.wp_dy != p.wo;  // re-pitched (n, h, o, wp) only when rows are unaligned
    if ((long long)n * hi > (1LL << 31)) return false;
    p.part_bytes = align256((size_t)p.splits * p.n_tiles * 128 * p.Npad * 4);
    p.pdb_bytes = align256((size_t)p.splits * 2 * p.Npad * 4);  // one row per converter group
    // tap-mode boxes may read up to (l-1)*d + 32 floats past a row's end (those columns
    // only meet zero dy); pad the staged copy so the last row stays inside it
    p.copy_bytes = align256((size_t)n * cin * hi * p.wp_x * 4 + ((size_t)(k - 1) * d + 64) * 4);
    p.x_bytes = (size_t)p.n_b * p.copy_bytes;
    p.dy_bytes = p.stage_dy ? align256((size_t)n * cout * p.ho * p.wp_dy * 4) : 0;
    p.total_bytes = p.part_bytes + p.pdb_bytes + p.x_bytes + p.dy_bytes;
    return true;
}

static PFN_cuTensorMapEncodeTiled_v12000 wg_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (fn == nullptr) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    return fn;
}

static int wg_map(CUtensorMap *m, const void *base, int rank, const cuuint64_t *dims,
                  const cuuint64_t *strides_bytes, const cuuint32_t *box, bool swz,
                  bool f16 = false) {
    auto enc = wg_encode();
    if (!enc) return set_error(DP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     rank, (void *)base, dims, strides_bytes,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(DP_ERR_CUDA, "weight gradient: cuTensorMapEncodeTiled failed (%d)",
                         (int)r);
    return DP_OK;
}

// ---- helpers shared with the shared-memory-operand variant (tc_wgrad_ss.cu)
unsigned long long *wg_trace_buffer(cudaStream_t st) {
    static unsigned long long *buf = nullptr;
    if (!buf && cudaMalloc(&buf, 256 * 16 * 8) != cudaSuccess) buf = nullptr;
    if (buf) cudaMemsetAsync(buf, 0, 256 * 16 * 8, st);
    g_wg_trace = buf;
    return buf;
}
int wg_make_map(CUtensorMap *m, const void *base, int rank, const cuuint64_t *dims,
                const cuuint64_t *strides_bytes, const cuuint32_t *box, bool swz) {
    return wg_map(m, base, rank, dims, strides_bytes, box, swz);
}
int wg_make_map16(CUtensorMap *m, const void *base, int rank, const cuuint64_t *dims,
                  const cuuint64_t *strides_bytes, const cuuint32_t *box) {
    return wg_map(m, base, rank, dims, strides_bytes, box, true, true);
}

// dy staging for the fp16-split weight gradient: NCHW fp32 (row pitch ws) -> two fp16
// tensors (n, h, o, wp) hi = RN(dy), lo' = RN((dy - hi) * 2^11) (the data gradient's offset
// split), lm zeros left of each row; one thread per 8 destination halves (16-byte stores)
__global__ void __launch_bounds__(256) tc_stage_dy16(const float *__restrict__ src,
                                                     uint4 *__restrict__ dhi,
                                                     uint4 *__restrict__ dlo, int O, int H,
                                                     int w, int wp, int lm, long long total8,
                                                     int ws, int *flag) {
    const int n8 = wp >> 3;
    bool bad = false;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total8;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long row = idx / n8;  // (n, o, h)
        const int v = (int)(idx - row * n8) * 8;
        const int h = (int)(row % H);
        const long long no = row / H;
        const int o = (int)(no % O);
        const long long n = no / O;
        const float *s = src + row * ws;
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c0 = v + 2 * q - lm, c1 = c0 + 1;
            const float e0 = (c0 >= 0 && c0 < w) ? __ldg(s + c0) : 0.f;
            const float e1 = (c1 >= 0 && c1 < w) ? __ldg(s + c1) : 0.f;
            bad |= !(fabsf(e0) < ptx::F16_SPLIT_MAX) || !(fabsf(e1) < ptx::F16_SPLIT_MAX);
            ptx::f16_split2_scaled(e0, e1, hw[q], lw[q]);
        }
        const long long di = (((n * H + h) * O + o) * wp + v) >> 3;
        dhi[di] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        dlo[di] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    if (bad) atomicOr(flag, 1);
}
int wg_stage_dy16(const float *dy, void *dhi, void *dlo, int n, int cout, int ho, int wo,
                  int wp, int lm, cudaStream_t st, int src_pitch, int *flag) {
    const long long total8 = (long long)n * cout * ho * (wp / 8);
    tc_stage_dy16<<<stage_grid(total8), 256, 0, st>>>(dy, (uint4 *)dhi, (uint4 *)dlo, cout, ho,
                                                      wo, wp, lm, total8,
                                                      src_pitch > 0 ? src_pitch : wo, flag);
    return check_launch("tc_stage_dy16");
}
// x -> (hi, lo') for the fp16-split weight gradient's in-place operands (the engine splits
// an activation once in the forward pass): rows of w floats -> rows of wp >= w halves (16-byte
// rows for TMA, zero padding), one thread per 8 destination halves (16-byte stores).  With
// hs / ls: also the same padded arrays shifted left by `shift` halves (flat: hs[i] = hi[i +
// shift]) -- the second tap residue's TMA boxes must start 16-byte aligned.
__device__ __forceinline__ float split_src(const float *__restrict__ x, long long q, int w,
                                           int wp, long long total) {
    if (q >= total) return 0.f;
    const long long row = q / wp;
    const int c = (int)(q - row * wp);
    return c < w ? __ldg(x + row * w + c) : 0.f;
}
__global__ void __launch_bounds__(256) tc_split_f16(const float *__restrict__ x,
                                                    uint4 *__restrict__ hi,
                                                    uint4 *__restrict__ lo,
                                                    uint4 *__restrict__ hs,
                                                    uint4 *__restrict__ ls, int shift, int w,
                                                    int wp, long long total8) {
    const int n8 = wp >> 3;
    const bool vec = (w & 3) == 0;  // source rows 16-byte aligned
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total8;
         i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / n8;
        const int v = (int)(i - row * n8) * 8;
        const float *s = x + row * w + v;
        float e[8];
        if (vec && v + 8 <= w) {
            const float4 a = __ldg(reinterpret_cast<const float4 *>(s));
            const float4 b = __ldg(reinterpret_cast<const float4 *>(s) + 1);
            e[0] = a.x; e[1] = a.y; e[2] = a.z; e[3] = a.w;
            e[4] = b.x; e[5] = b.y; e[6] = b.z; e[7] = b.w;
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) e[q] = v + q < w ? __ldg(s + q) : 0.f;
        }
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) ptx::f16_split2_scaled(e[2 * q], e[2 * q + 1], hw[q], lw[q]);
        hi[i] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        lo[i] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        if (hs) {
#pragma unroll
            for (int q = 0; q < 8; ++q) e[q] = split_src(x, i * 8 + shift + q, w, wp, total8 * 8);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                ptx::f16_split2_scaled(e[2 * q], e[2 * q + 1], hw[q], lw[q]);
            hs[i] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            ls[i] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
    }
}
int tc_split_f16_launch(const float *x, void *hi, void *lo, void *hs, void *ls, int shift,
                        long long rows, int w, int wp, cudaStream_t st) {
    if (((uintptr_t)x & 15) || ((uintptr_t)hi & 15) || ((uintptr_t)lo & 15) ||
        ((uintptr_t)hs & 15) || ((uintptr_t)ls & 15) || (!hs != !ls))
        return set_error(DP_ERR_ARG, "fp16 split: pointers must be 16-byte aligned");
    if (hs && (shift <= 0 || shift >= 8))
        return set_error(DP_ERR_ARG, "fp16 split: shift %d outside 1..7", shift);
    if (wp < w || (wp & 7))
        return set_error(DP_ERR_ARG, "fp16 split: pitch %d must be >= %d and a multiple of 8",
                         wp, w);
    const long long total8 = rows * (wp / 8);
    if (total8 <= 0) return DP_OK;
    tc_split_f16<<<stage_grid(total8), 256, 0, st>>>(x, (uint4 *)hi, (uint4 *)lo, (uint4 *)hs,
                                                     (uint4 *)ls, shift, w, wp, total8);
    return check_launch("tc_split_f16");
}
int wg_sms() { return wg_num_sms(); }
int wg_stage_x(const float *x, float *xs, int n, int cin, int hi, int wi, int wp, int mask,
               long long copy_floats, cudaStream_t st) {
    const long long quads = (long long)n * cin * hi * (wp / 4);
    tc_stage_x<<<stage_grid(quads), 256, 0, st>>>(x, xs, cin, hi, wi, wp, mask, copy_floats, quads);
    int rc = check_launch("tc_stage_x");
    if (rc) return rc;
    return stage_x_tails(xs, quads * 4, copy_floats, mask, st);
}
int wg_stage_x_taps(const float *x, float *xs, int n, int cin, int hi, int wi, int wp, int l,
                    int d, long long copy_floats, cudaStream_t st) {
    const long long quads = (long long)n * cin * hi * (wp / 4);
    tc_stage_x_taps<<<stage_grid(quads), 256, 0, st>>>(x, xs, cin, hi, wi, wp, l, d, copy_floats,
                                                       quads);
    int rc = check_launch("tc_stage_x_taps");
    if (rc) return rc;
    for (int j = 0; j < l; ++j)
        if (cudaMemsetAsync(xs + j * copy_floats + quads * 4, 0,
                            (size_t)(copy_floats - quads * 4) * 4, st) != cudaSuccess)
            return set_error(DP_ERR_CUDA, "weight gradient: memset of staged tails failed");
    return DP_OK;
}
int wg_stage_dy(const float *dy, float *dys, int n, int cout, int ho, int wo, int wp, int lm,
                cudaStream_t st, int src_pitch, const int *exit_unless) {
    const long long quads = (long long)n * cout * ho * (wp / 4);
    // a gated fallback usually exits at once: a small grid-stride grid keeps that ~3 us
    // (the full grid measured 22 us of block launches that only read the flag)
    const int grid = exit_unless ? std::min(stage_grid(quads), 2 * wg_num_sms()) : stage_grid(quads);
    tc_stage_dy<<<grid, 256, 0, st>>>(dy, dys, cout, ho, wo, wp, lm, quads,
                                      src_pitch > 0 ? src_pitch : wo, exit_unless);
    return check_launch("tc_stage_dy");
}

// preferred variant: x tap lines read by the tensor core from a shared-memory row ring
bool ws_supported(int n, int cin, int hi, int wi, int cout, int k, int d);
size_t ws_workspace(int n, int cin, int hi, int wi, int cout, int k, int d);
int ws_conv_backward_kernel(const float *x, const float *dy, float *dw, float *db, int n,
                            int cin, int hi, int wi, int cout, int k, int d, void *ws,
                            size_t ws_bytes, cudaStream_t st, int phases, size_t x_slack,
                            int dy_pitch, const int *exit_unless = nullptr);

// Split form (engine): stage x early (phase 1, may run during the forward pass), the rest
// later (phase 2).  Only the smem-operand kernel splits; the TMEM-operand fallback stages
// everything in its single call (prepare is then a no-op).
int tc_wgrad_prepare(const float *x, int n, int cin, int hi, int wi, int cout, int k, int d,
                     void *ws, size_t ws_bytes, cudaStream_t st) {
    if (!ws_supported(n, cin, hi, wi, cout, k, d)) return DP_OK;
    return ws_conv_backward_kernel(x, nullptr, nullptr, nullptr, n, cin, hi, wi, cout, k, d, ws,
                                   ws_bytes, st, 1, 0, 0);
}
int tc_conv_backward_kernel(const float *x, const float *dy, float *dw, float *db, int n,
                            int cin, int hi, int wi, int cout, int k, int d, void *ws,
                            size_t ws_bytes, cudaStream_t st, size_t x_slack, int dy_pitch);
int tc_conv_backward_kernel_staged(const float *x, const float *dy, float *dw, float *db, int n,
                                   int cin, int hi, int wi, int cout, int k, int d, void *ws,
                                   size_t ws_bytes, cudaStream_t st) {
    if (!ws_supported(n, cin, hi, wi, cout, k, d))
        return tc_conv_backward_kernel(x, dy, dw, db, n, cin, hi, wi, cout, k, d, ws, ws_bytes,
                                       st, 0, 0);
    return ws_conv_backward_kernel(x, dy, dw, db, n, cin, hi, wi, cout, k, d, ws, ws_bytes, st,
                                   2, 0, 0);
}

bool tc_wgrad_supported(int n, int cin, int hi, int wi, int cout, int k, int d) {
    if (ws_supported(n, cin, hi, wi, cout, k, d)) return true;
    WgPlan p;
    return wg_plan(n, cin, hi, wi, cout, k, d, p);
}

size_t tc_wgrad_workspace(int n, int cin, int hi, int wi, int cout, int k, int d) {
    if (ws_supported(n, cin, hi, wi, cout, k, d)) return ws_workspace(n, cin, hi, wi, cout, k, d);
    WgPlan p;
    if (!wg_plan(n, cin, hi, wi, cout, k, d, p)) return 0;
    return p.total_bytes;
}

int tc_conv_backward_kernel(const float *x, const float *dy, float *dw, float *db, int n,
                            int cin, int hi, int wi, int cout, int k, int d, void *ws,
                            size_t ws_bytes, cudaStream_t st, size_t x_slack, int dy_pitch) {
    if (ws_supported(n, cin, hi, wi, cout, k, d))
        return ws_conv_backward_kernel(x, dy, dw, db, n, cin, hi, wi, cout, k, d, ws, ws_bytes,
                                       st, 3, x_slack, dy_pitch);
    if (dy_pitch != 0 && dy_pitch != wi - (k - 1) * d)
        return set_error(DP_ERR_UNSUPPORTED, "weight gradient: pitched dy needs the smem kernel");
    WgPlan p;
    if (!wg_plan(n, cin, hi, wi, cout, k, d, p))
        return set_error(DP_ERR_UNSUPPORTED,
                         "tensor-core weight gradient: shape outside the kernel envelope "
                         "(cin=%d cout=%d k=%d d=%d)",
                         cin, cout, k, d);
    if (ws == nullptr || ws_bytes < p.total_bytes)
        return set_error(DP_ERR_ARG, "tensor-core weight gradient: workspace %zu < %zu bytes",
                         ws_bytes, p.total_bytes);
    if (((uintptr_t)ws & 255) != 0)
        return set_error(DP_ERR_ARG,
                         "tensor-core weight gradient: workspace must be 256-byte aligned");
    unsigned char *w8 = (unsigned char *)ws;
    TcWgradArgs a;
    a.part = (float *)w8;
    a.pdb = (float *)(w8 + p.part_bytes);
    float *xs = (float *)(w8 + p.part_bytes + p.pdb_bytes);
    const int mask = p.shift_mask;
    {
        const long long quads = (long long)n * cin * hi * (p.wp_x / 4);
        tc_stage_x<<<stage_grid(quads), 256, 0, st>>>(x, xs, cin, hi, wi, p.wp_x, mask,
                                                      (long long)(p.copy_bytes / 4), quads);
        int rt = stage_x_tails(xs, quads * 4, (long long)(p.copy_bytes / 4), mask, st);
        if (rt) return rt;
    }
    int rc = check_launch("tc_stage_x");
    if (rc) return rc;
    const bool stage_dy = p.stage_dy || ((uintptr_t)dy & 15) != 0;
    if (stage_dy && !p.stage_dy)
        return set_error(DP_ERR_ARG, "weight gradient: dy must be 16-byte aligned");
    const float *dys = dy;
    if (stage_dy) {
        float *dp_ = (float *)(w8 + p.part_bytes + p.pdb_bytes + p.x_bytes);
        const long long quads = (long long)n * cout * p.ho * (p.wp_dy / 4);
        tc_stage_dy<<<stage_grid(quads), 256, 0, st>>>(dy, dp_, cout, p.ho, p.wo, p.wp_dy, 0, quads,
                                                       p.wo, nullptr);
        rc = check_launch("tc_stage_dy");
        if (rc) return rc;
        dys = dp_;
    }
    // ---- tensor maps
    CUtensorMap mx[4], mdy;
    {
        // staged: (n, h, o, wp_dy); direct: NCHW with 16-byte rows
        const cuuint64_t rowb = (cuuint64_t)(stage_dy ? p.wp_dy : p.wo) * 4;
        cuuint64_t dims[4] = {(cuuint64_t)p.wo, (cuuint64_t)p.ho, (cuuint64_t)cout, (cuuint64_t)n};
        cuuint64_t str[3] = {stage_dy ? rowb * cout : rowb, stage_dy ? rowb : rowb * p.ho,
                             rowb * cout * p.ho};
        cuuint32_t box[4] = {32, 1, (cuuint32_t)p.Npad, 1};
        rc = wg_map(&mdy, dys, 4, dims, str, box, true);
        if (rc) return rc;
    }
    const cuuint64_t xrow = (cuuint64_t)p.wp_x * 4;          // one channel line
    const cuuint64_t ximg_row = xrow * cin;                  // one image row (all channels)
    for (int b = 0, slot = 0; b < 4; ++b) {
        const bool used = (mask >> b) & 1;
        const float *base = (const float *)((const unsigned char *)xs +
                                            (size_t)(used ? slot : 0) * p.copy_bytes);
        if (p.tap_mode) {
            // (w, j: stride d, c, i: stride d rows, row of n*hi) -- overlapping views
            cuuint64_t dims[5] = {(cuuint64_t)wi, (cuuint64_t)k, (cuuint64_t)cin, (cuuint64_t)k,
                                  (cuuint64_t)n * hi};
            cuuint64_t str[4] = {(cuuint64_t)d * 4, xrow, ximg_row * d, ximg_row};
            cuuint32_t box[5] = {32, (cuuint32_t)k, (cuuint32_t)cin, (cuuint32_t)p.max_ni, 1};
            rc = wg_map(&mx[b], base, 5, dims, str, box, true);
        } else {
            cuuint64_t dims[4] = {(cuuint64_t)p.wp_x, (cuuint64_t)cin, (cuuint64_t)k,
                                  (cuuint64_t)n * hi};
            cuuint64_t str[3] = {xrow, ximg_row * d, ximg_row};
            cuuint32_t box[4] = {(cuuint32_t)p.L4 * 4, (cuuint32_t)cin, (cuuint32_t)p.max_ni, 1};
            rc = wg_map(&mx[b], base, 4, dims, str, box, false);
        }
        if (rc) return rc;
        if (used) ++slot;
    }
    a.C = cin;
    a.Cpad = p.Cpad;
    a.l = k;
    a.d = d;
    a.Q = cout;
    a.Npad = p.Npad;
    a.rows_total = p.rows_total;
    a.n_tiles = p.n_tiles;
    a.G = p.G;
    a.n_groups = p.n_groups;
    a.splits = p.splits;
    a.Ho = p.ho;
    a.Wo = p.wo;
    a.nvb = p.nvb;
    a.kb_total = p.kb_total;
    a.SS = p.SS;
    a.TS = p.TS;
    a.tap_mode = p.tap_mode ? 1 : 0;
    a.L4 = p.L4;
    a.n_b = p.n_b;
    a.shift_mask = p.shift_mask;
    a.b_bytes = p.b_bytes;
    a.box_bytes = p.box_bytes;
    a.box_tx = p.box_tx;
    a.stage_bytes = p.stage_bytes;
    a.Hi = hi;
    a.trace = nullptr;
    if (getenv("DP_WG_TRACE")) {
        static unsigned long long *buf = nullptr;
        if (!buf && cudaMalloc(&buf, 256 * 16 * 8) != cudaSuccess) buf = nullptr;
        if (buf) cudaMemsetAsync(buf, 0, 256 * 16 * 8, st);
        a.trace = buf;
        g_wg_trace = buf;
    }
    a.dbg = getenv("DP_WG_DBG") ? atoi(getenv("DP_WG_DBG")) : 0;
    size_t smem = (size_t)p.SS * p.stage_bytes + 1024;
    cudaError_t e = cudaFuncSetAttribute(tc_wgrad_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tc_wgrad: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    const int grid = p.n_groups * p.splits;
    tc_wgrad_kernel<<<grid, WG_THREADS, smem, st>>>(mx[0], mx[1], mx[2], mx[3], mdy, a);
    rc = check_launch("tc_wgrad_kernel");
    if (rc) return rc;
    long long total = (long long)cout * cin * k * k + cout;
    tc_wgrad_reduce<<<ceil_div(total, 256), 256, 0, st>>>(a.part, a.pdb, dw, db, cout, cin,
                                                          p.Cpad, k, p.Npad, p.splits,
                                                          p.n_tiles * 128);
    return check_launch("tc_wgrad_reduce");
}

}  // namespace dp
