// Weight / bias gradient of the d-regularly sparse convolution on the tcgen05 tensor cores
// with BOTH operands read from shared memory (fast tier, 3xTF32) -- preferred over the
// TMEM-operand kernel in tc_wgrad.cu whenever its row ring fits.
//
//   dw[o,c,i,j] = sum_{n,u,v} dy[n,o,u,v] * x[n,c,u+i*d,v+j*d]      db[o] = sum dy[n,o,u,v]
// (reference _kernels.pyx:94-130, _kernels_py.py:54-66) as D[r, o] = sum_k A[r, k] B[o, k]:
//   k = output pixel, K blocks of 32 consecutive v of one output row u  (the long axis)
//   r = x tap line (i, residue copy, c, jj)                             -> M, tiles of 128
//   o = output channel (x J column-tap shifts, padded to 16)             -> N
//
// x tap lines.  tc_stage_x lays x out as (n, h, c, wp) copies shifted left by
// b = (j*d) & 3 for each residue b that occurs, so that for one residue copy the taps j with
// that residue sit at columns v0 + j*d - b, all multiples of 4 floats, lcm(d, 4) floats
// apart -- a legal TMA stride.  One 4-D box {32 px, taps of the residue, cin channels,
// 1 row} therefore delivers, for ONE input row, every (c, j) line of 32 pixels as a 128-byte
// SWIZZLE_128B row: exactly the canonical K-major A layout the tensor core reads (SBO = 1024,
// +32 B per K=8 slice).  All residue boxes of an input row form one ring slot of Ls lines
// (each box rounded up to 8 lines; cin * l when cin % 8 == 0).
//
// Row ring.  A CTA walks K blocks down image columns (u, u+d, u+2d, ... for one 32-px block
// and row phase u mod d).  Consecutive blocks share l-1 of their l tap rows (rows u + i*d),
// so each input row is loaded ONCE into a ring slot and serves as tap row i of l successive
// blocks; a block adds one row (a column start adds all of them).  The lo part of a row
// (x - trunc_tf32(x), for 3xTF32) is computed once into a parallel lo ring.  Block tiles
// (128 consecutive lines = parts of up to 3 slots) are contiguous because the first NM
// slots are mirrored past the ring's end.  Ring slot reuse: inside a column the slot a block
// overwrites was last read by block kl - SS (R = n_i + SS - 1 slots); a column start waits
// for the previous block (a drain every ~Ho/d blocks).
//
// Small-cin layers with several residues (c2 conv1: cin 3, d 1) stage one pre-shifted copy
// of x per tap instead (tc_stage_x_taps): a single box {32 px, l taps, cin, 1 row} per input
// row rather than one tiny box per residue (the TMA box rate was their limit).
//
// 3xTF32 per K=8 slice and tile: A_hi x [B_hi | B_lo] (N = 2 NB) + A_lo x B_hi (N = NB);
// accumulators stay in TMEM (all tiles of the CTA's group: no A staging in TMEM at all).  A
// group's last tile with <= 64 real lines runs as M = 64 (D row r in TMEM quadrant r / 16,
// lane r % 16 -- measured with tools/m64_probe.cu).
//
// Roles (one CTA per SM, 10 warps): warp 8 TMA producer, warp 9 TMEM allocator + MMA issuer,
// warps 0-7 converters (dy B_lo + db, lo lines of new rows) and the epilogue.  Split-K over
// CTAs, partials [split][line][o] summed by ws_reduce in a fixed order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>

#include "dp_common.cuh"
#include "tc_ptx.cuh"

namespace dp {

int wg_make_map(CUtensorMap *m, const void *base, int rank, const cuuint64_t *dims,
                const cuuint64_t *strides_bytes, const cuuint32_t *box, bool swz);
int wg_make_map16(CUtensorMap *m, const void *base, int rank, const cuuint64_t *dims,
                  const cuuint64_t *strides_bytes, const cuuint32_t *box);
int wg_stage_dy16(const float *dy, void *dhi, void *dlo, int n, int cout, int ho, int wo,
                  int wp, int lm, cudaStream_t st, int src_pitch, int *flag);
int wg_sms();
unsigned long long *wg_trace_buffer(cudaStream_t st);
int wg_stage_x(const float *x, float *xs, int n, int cin, int hi, int wi, int wp, int mask,
               long long copy_floats, cudaStream_t st);
int wg_stage_x_taps(const float *x, float *xs, int n, int cin, int hi, int wi, int wp, int l,
                    int d, long long copy_floats, cudaStream_t st);
int wg_stage_dy(const float *dy, float *dys, int n, int cout, int ho, int wo, int wp, int lm,
                cudaStream_t st, int src_pitch, const int *exit_unless);

constexpr int WS_CONV_WARPS = 8;
constexpr int WS_TMA_WARP = 8;
constexpr int WS_MMA_WARP = 9;
constexpr int WS_THREADS = 320;
constexpr int WS_MAX_SS = 12;
constexpr int WS_MAX_G = 16;
constexpr int WS_SMEM_BUDGET = 222 * 1024;

struct WsResidues {
    int n_b;        // residue copies used
    int b[4];       // residue of copy slot
    int n[4];       // taps in the residue
    int j0[4];      // first tap of the residue
    int line0[4];   // first line of the residue's box inside a ring slot
    int step;       // tap step inside a residue: 4 / gcd(d, 4)
    int tapcopy;    // 1: one staged copy per tap (single box per row), lines (c, j)
    int nreal0;     // real taps of residue 0 (n[0] may be padded so cin * n[0] == Ls)
};

struct WsArgs {
    int C, Cpad, l, d, Q, Npad;
    int J, sb, NB;       // dy copies per stage, their shift step (Ja*d floats, 4 | sb), N
                         // (J*Q rows rounded up to 16: B rows jb'*Q + o, zero rows past J*Q)
    int tma_mirror;      // DP_WG_TMA_MIRROR: mirror slots loaded by TMA, not the converters
    int pair;            // one 2-row x box feeds two consecutive blocks of a column
    int direct;          // x read in place from NCHW through a 5-D map (no staged copy)
    int n_tiles, G, n_groups, splits;
    int Ho, Wo, nvb, T, Hi;
    long long kb_total;  // n * nvb * d columns x T blocks
    int SS, R, NM, Ls;   // dy stages, ring slots, mirrored slots, lines per slot
    uint32_t b_bytes;    // dy stage: B_hi + B_lo (2 * NB * 128)
    uint32_t slot_bytes, box_tx_row;  // Ls * 128
    uint32_t ring_hi, ring_lo;        // shared-memory offsets
    WsResidues rs;
    float *part;  // [splits][n_tiles * 128][NB]
    float *pdb;   // [splits][Npad]
    int no_m64;   // DP_WG_NO_M64: run a short last tile as M = 128 (experiments)
    int pf;       // L2 prefetch distance in K blocks (DP_WG_PF, 0 = off)
    int f16;      // fp16-split operands: tm_x1 = x lo', tm_xp = dy lo' (offset split, 2^11)
    int dycomb;   // fp16: ONE dy box {64, Q, J, row, hl} brings B_hi and B_lo' (tm_dy; rows
                  // n*Ho + u); B_lo' then starts at row LO = J*Q (else two boxes, LO = NB)
    int LO;       // B row (and accumulator column) offset of the lo' half
    int dy_rows;  // dycomb: n * Ho folded rows (a row past Ho -- a column phase running past
                  // the image -- is sent to this out-of-range row: TMA zero fill)
    unsigned long long *trace;  // DP_WG_TRACE: per-K-block clock64 stamps of CTA 0
    const int *exit_if;         // fp16 kernel: exit when its operands tripped the range flag
    const int *exit_unless;     // its tf32 fallback: run only when they did
};

// slots: 1 producer ready, 0 TMA issue, 2 converters got the stage, 4 converters done,
// 10 MMA ready, 8 MMA got, 9 issued
#define WS_TRACE(A, KL, SLOT, COND)                                               \
    do {                                                                          \
        if ((A).trace && (COND) && blockIdx.x == 0 && (KL) < 256)                 \
            (A).trace[(KL) * 16 + (SLOT)] = clock64();                            \
    } while (0)

// Column-major K order (see header).  Bm = ring slot of the block's first tap row.
struct WsSched {
    int t, T, vb, img, phase, u, nvb, d, n_i, R, Bm;
    bool cstart;
    __device__ WsSched(const WsArgs &a, long long kb, int ni) {
        T = a.T;
        nvb = a.nvb;
        d = a.d;
        n_i = ni;
        R = a.R;
        const long long col = kb / T;
        t = (int)(kb - col * T);
        phase = (int)(col % d);
        const long long vc = col / d;
        vb = (int)(vc % nvb);
        img = (int)(vc / nvb);
        u = phase + t * d;
        Bm = 0;
        cstart = true;
    }
    __device__ void next() {
        if (++t == T) {
            t = 0;
            if (++phase == d) {
                phase = 0;
                if (++vb == nvb) {
                    vb = 0;
                    ++img;
                }
            }
        }
        u = phase + t * d;
        // inside a column the block sits one row further down the ring; a new column
        // starts on fresh slots after the previous block's n_i rows
        Bm += (t == 0) ? n_i : 1;
        while (Bm >= R) Bm -= R;
        cstart = t == 0;
    }
};

__global__ void __launch_bounds__(WS_THREADS, 1)
tc_wgrad_ss_kernel(const __grid_constant__ CUtensorMap tm_x0,
                   const __grid_constant__ CUtensorMap tm_x1,
                   const __grid_constant__ CUtensorMap tm_x2,
                   const __grid_constant__ CUtensorMap tm_x3,
                   const __grid_constant__ CUtensorMap tm_dy,
                   const __grid_constant__ CUtensorMap tm_xp, const WsArgs a) {
    extern __shared__ __align__(1024) unsigned char ws_smem_raw[];
    __shared__ uint64_t sfull[WS_MAX_SS], cfull[WS_MAX_SS], sempty[WS_MAX_SS], accfull;
    __shared__ uint32_t s_tmem;

    if ((a.exit_if && *(volatile const int *)a.exit_if) ||
        (a.exit_unless && !*(volatile const int *)a.exit_unless))
        return;  // block-uniform, before any barrier or TMEM allocation
    unsigned char *smem = (unsigned char *)(((uintptr_t)ws_smem_raw + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x % a.n_groups, split = blockIdx.x / a.n_groups;
    const int tile0 = g * a.G;
    const int G = min(a.G, a.n_tiles - tile0);
    const long long kb_first = a.kb_total * split / a.splits;
    const int nkb = (int)(a.kb_total * (split + 1) / a.splits - kb_first);
    const int acc_cols = 2 * a.NB;
    const int lines_total = a.l * a.Ls;
    const int i_lo = tile0 * 128 / a.Ls;
    const int n_i = (min((tile0 + G) * 128, lines_total) - 1) / a.Ls - i_lo + 1;
    // a last tile with <= 64 real lines runs as M = 64 (D rows r -> TMEM quadrant r / 16,
    // lane r % 16; measured, tools/m64_probe.cu): half its A reads and tensor work
    const bool tail64 = !a.no_m64 && min((tile0 + G) * 128, lines_total) - (tile0 + G - 1) * 128 <= 64;

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.SS; ++s) {
            ptx::mbar_init(&sfull[s], 1);
            ptx::mbar_init(&cfull[s], WS_CONV_WARPS);
            ptx::mbar_init(&sempty[s], 1);
        }
        ptx::mbar_init(&accfull, 1);
        ptx::mbar_fence_init();
    }
    if (warp == WS_TMA_WARP && lane == 0) {
        ptx::tma_prefetch_desc(&tm_dy);
        ptx::tma_prefetch_desc(&tm_x0);
    }
    if (warp == WS_MMA_WARP) ptx::tmem_alloc<512>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == WS_TMA_WARP) {
        // ================================ TMA producer ================================
        WsSched sc(a, kb_first, n_i);
        // a second schedule a.pf blocks ahead: its dy box and new x row are prefetched into
        // L2 so the stage's TMA loads hit L2 (the traces showed ~2400 cycles from issue to
        // stage-full with only 2-3 stages in flight on the wide layers)
        WsSched pf(a, kb_first, n_i);
        for (int q = 0; q < a.pf; ++q) pf.next();
        unsigned char *ring = smem + a.ring_hi;
        int pre = 0;  // this block's new row came with the previous block's 2-row box
        for (int kl = 0; kl < nkb; ++kl, sc.next(), pf.next()) {
            if (a.pf && lane == 0 && kl + a.pf < nkb) {
                const int pv0 = pf.vb * (a.f16 ? 64 : 32);
                const int prow = pf.u < a.Ho ? pf.img * a.Ho + pf.u : a.dy_rows;
                if (a.dycomb && a.J == 1)
                    ptx::tma_prefetch_l2_4d(&tm_dy, pv0, 0, prow, 0);
                else if (a.dycomb)
                    ptx::tma_prefetch_l2_5d(&tm_dy, pv0, 0, 0, prow, 0);
                else if (a.J == 1)
                    ptx::tma_prefetch_l2_4d(&tm_dy, pv0, pf.u, 0, pf.img);
                else
                    ptx::tma_prefetch_l2_5d(&tm_dy, pv0, 0, 0, pf.u, pf.img);
                if (a.f16 && !a.dycomb && a.J == 1)
                    ptx::tma_prefetch_l2_4d(&tm_xp, pv0, pf.u, 0, pf.img);
                else if (a.f16 && !a.dycomb)
                    ptx::tma_prefetch_l2_5d(&tm_xp, pv0, 0, 0, pf.u, pf.img);
                for (int k = pf.cstart ? 0 : n_i - 1; k < n_i; ++k) {
                    if (a.direct) {
                        // fp16: residue rb's hi / lo' views are tm_x{2rb} / tm_x{2rb+1}
                        for (int rb = 0; rb < a.rs.n_b; ++rb) {
                            const int xc = pv0 + a.rs.j0[rb] * a.d - a.rs.b[rb],
                                      xr = pf.u + (i_lo + k) * a.d;
                            ptx::tma_prefetch_l2_5d(rb ? &tm_x2 : &tm_x0, xc, 0, 0, xr, pf.img);
                            if (a.f16)
                                ptx::tma_prefetch_l2_5d(rb ? &tm_x3 : &tm_x1, xc, 0, 0, xr,
                                                        pf.img);
                        }
                        continue;
                    }
                    const int prow = pf.img * a.Hi + pf.u + (i_lo + k) * a.d;
                    for (int rb = 0; rb < a.rs.n_b; ++rb) {
                        const CUtensorMap *m = rb == 0 ? &tm_x0 : rb == 1 ? &tm_x1
                                                               : rb == 2 ? &tm_x2 : &tm_x3;
                        ptx::tma_prefetch_l2_4d(m, pv0 + a.rs.j0[rb] * a.d - a.rs.b[rb], 0, 0,
                                                prow);
                    }
                }
            }
            const int s = kl % a.SS;
            WS_TRACE(a, kl, 1, lane == 0);
            ptx::mbar_wait(&sempty[s], ((kl / a.SS) & 1) ^ 1);
            if (sc.cstart && kl > 0) {
                const int kw = kl - 1;  // column start: drain (see header)
                ptx::mbar_wait(&sempty[kw % a.SS], (kw / a.SS) & 1);
            }
            if (lane == 0) {
                const int v0 = sc.vb * (a.f16 ? 64 : 32);
                const int hh = sc.img * a.Hi + sc.u;
                const uint32_t f16x = a.f16 ? 2u : 1u;  // fp16 split: hi and lo' boxes
                const int k0 = sc.cstart ? 0 : n_i - 1;
                WS_TRACE(a, kl, 0, true);
                // TMA box count, not bytes, limits this producer: inside a column one 2-row
                // box (rows u + (n_i-1) d and u + n_i d, adjacent ring slots) feeds this
                // block and the next one
                int slotN = sc.Bm + n_i - 1;
                if (slotN >= a.R) slotN -= a.R;
                const bool skip = !sc.cstart && pre;
                const bool pair = a.pair && !sc.cstart && !pre && sc.t + 1 < a.T &&
                                  kl + 1 < nkb && slotN + 1 < a.R;
                int nbox_rows = 0;
                if (sc.cstart || !a.pair) {
                    for (int k = k0; k < n_i; ++k) {
                        int slot = sc.Bm + k;
                        if (slot >= a.R) slot -= a.R;
                        nbox_rows += (a.tma_mirror && slot < a.NM) ? 2 : 1;
                    }
                } else {
                    nbox_rows = skip ? 0 : pair ? 2 : 1;
                }
                ptx::mbar_expect_tx(&sfull[s], f16x * ((uint32_t)(a.J * a.Q) * 128u +
                                                          (uint32_t)nbox_rows * a.box_tx_row));
                if (a.f16 && !a.dycomb) {  // B_lo' straight from the staged fp16 lo' rows
                    unsigned char *bl = smem + (size_t)s * a.b_bytes + (size_t)a.NB * 128;
                    if (a.J == 1)
                        ptx::tma_load_4d(bl, &tm_xp, v0, sc.u, 0, sc.img, &sfull[s]);
                    else
                        ptx::tma_load_5d(bl, &tm_xp, v0, 0, 0, sc.u, sc.img, &sfull[s]);
                }
                const int drow = sc.u < a.Ho ? sc.img * a.Ho + sc.u : a.dy_rows;
                if (a.dycomb && a.J == 1) {  // (w, o, row, hl): hi rows then lo' rows
                    ptx::tma_load_4d(smem + (size_t)s * a.b_bytes, &tm_dy, v0, 0, drow, 0,
                                     &sfull[s]);
                } else if (a.dycomb) {       // (w, o, jb', row, hl)
                    ptx::tma_load_5d(smem + (size_t)s * a.b_bytes, &tm_dy, v0, 0, 0, drow, 0,
                                     &sfull[s]);
                } else if (a.J == 1) {
                    ptx::tma_load_4d(smem + (size_t)s * a.b_bytes, &tm_dy, v0, sc.u, 0, sc.img,
                                     &sfull[s]);
                } else {
                    // ONE box {32 px, Q, J} of the overlapping view (w, o, jb' = J-1-jb: sb
                    // floats apart, ...) of the zero-margined staged dy: rows jb'*Q + o hold
                    // dy shifted right by jb*sb for the column taps j = jb*Ja + ja
                    ptx::tma_load_5d(smem + (size_t)s * a.b_bytes, &tm_dy, v0, 0, 0, sc.u,
                                     sc.img, &sfull[s]);
                }
                if (pair)
                    ptx::tma_load_5d(ring + (size_t)slotN * a.slot_bytes, &tm_xp,
                                     v0 + a.rs.j0[0] * a.d - a.rs.b[0], 0, 0, 0,
                                     hh + (i_lo + n_i - 1) * a.d, &sfull[s]);
                pre = pair ? 1 : 0;
                for (int k = (skip || pair) ? n_i : k0; k < n_i; ++k) {
                    int slot = sc.Bm + k;
                    if (slot >= a.R) slot -= a.R;
                    const int row = hh + (i_lo + k) * a.d;
                    for (int copy = 0; copy < 2; ++copy) {
                        if (copy == 1 && (slot >= a.NM || !a.tma_mirror)) break;
                        unsigned char *dst =
                            ring + (size_t)(copy ? a.R + slot : slot) * a.slot_bytes;
                        if (a.direct) {
                            // NCHW in place: (w, jj, c, h, n); rows past Hi zero-fill.  The
                            // fp16 split may have two residues (tap offsets j*d = 0 / 4 mod 8
                            // halves): one box each, lo' rows into the lo ring
                            for (int rb = 0; rb < a.rs.n_b; ++rb) {
                                unsigned char *db_ = dst + (size_t)a.rs.line0[rb] * 128;
                                // (residue 1: a copy shifted left by its residue b, so the
                                // box start stays 16-byte aligned)
                                const int xc = v0 + a.rs.j0[rb] * a.d - a.rs.b[rb],
                                          xr = sc.u + (i_lo + k) * a.d;
                                ptx::tma_load_5d(db_, rb ? &tm_x2 : &tm_x0, xc, 0, 0, xr, sc.img,
                                                 &sfull[s]);
                                if (a.f16)
                                    ptx::tma_load_5d(db_ + (a.ring_lo - a.ring_hi),
                                                     rb ? &tm_x3 : &tm_x1, xc, 0, 0, xr, sc.img,
                                                     &sfull[s]);
                            }
                            continue;
                        }
                        for (int rb = 0; rb < a.rs.n_b; ++rb) {
                            const CUtensorMap *m = rb == 0 ? &tm_x0 : rb == 1 ? &tm_x1
                                                                   : rb == 2 ? &tm_x2 : &tm_x3;
                            ptx::tma_load_4d(dst + (size_t)a.rs.line0[rb] * 128, m,
                                             v0 + a.rs.j0[rb] * a.d - a.rs.b[rb], 0, 0, row,
                                             &sfull[s]);
                        }
                    }
                }
            }
            __syncwarp();
        }
    } else if (warp == WS_MMA_WARP) {
        // ================================ MMA issuer ================================
        // [B_hi | B_lo'] spans LO + NB rows... the stacked MMA's N: 2 NB, or 2 J Q when the
        // halves come in one box (J Q a multiple of 8)
        const int n2 = a.dycomb ? 2 * a.LO : 2 * a.NB;
        const uint32_t idesc_2n = a.f16 ? ptx::idesc_f16(128, n2) : ptx::idesc_tf32(128, 2 * a.NB);
        const uint32_t idesc_n = a.f16 ? ptx::idesc_f16(128, a.NB) : ptx::idesc_tf32(128, a.NB);
        const uint32_t idesc_2n64 =
            a.f16 ? ptx::idesc_f16(64, n2) : ptx::idesc_tf32(64, 2 * a.NB);
        const uint32_t idesc_n64 = a.f16 ? ptx::idesc_f16(64, a.NB) : ptx::idesc_tf32(64, a.NB);
        const uint32_t sbase = ptx::smem_u32(smem);
        const uint32_t hi_base = sbase + a.ring_hi, lo_base = sbase + a.ring_lo;
        // tile 0's first ring slot (relative to the block's Bm) and line inside it; later
        // tiles follow 128 lines on (incremental: this thread's loop is the critical path)
        const int line00 = tile0 * 128 - i_lo * a.Ls;
        const int slot00 = line00 / a.Ls, lin00 = line00 - slot00 * a.Ls;
        const int RL = a.R * a.Ls;  // ring lines (the mirrors follow)
        const uint64_t lo_units = (uint64_t)((a.ring_lo - a.ring_hi) >> 4);
        WsSched sc(a, kb_first, n_i);
        int s = 0;
        uint32_t ph = 0;
        for (int kl = 0; kl < nkb; ++kl, sc.next()) {
            WS_TRACE(a, kl, 10, lane == 0);
            ptx::mbar_wait(&cfull[s], ph);
            ptx::tc_fence_after();
            WS_TRACE(a, kl, 8, lane == 0);
            if (ptx::elect_one()) {
                const uint64_t bd0 = ptx::smem_desc_sw128(sbase + (uint32_t)s * a.b_bytes);
                // tile t starts at ring line P0 + 128 t: descriptor +1024 (16 KB >> 4) per
                // tile; past a slot's end its lines continue in the next slot (or the mirror
                // past the ring's end), and a tile STARTING past the end wraps (-RL lines).
                // Plain 64-bit adds on the descriptor: this thread is the critical path.
                int slot0 = sc.Bm + slot00;
                if (slot0 >= a.R) slot0 -= a.R;
                int P = slot0 * a.Ls + lin00;
                uint64_t dh = ptx::smem_desc_sw128(hi_base + (uint32_t)P * 128u);
                for (int t = 0; t < G; ++t, P += 128, dh += 1024) {
                    const uint64_t da = P >= RL ? dh - (uint64_t)(RL * 8) : dh;
                    const uint32_t dcol = tmem + (uint32_t)(t * acc_cols);
                    const bool m64 = tail64 && t == G - 1;
                    const uint32_t i2 = m64 ? idesc_2n64 : idesc_2n, i1 = m64 ? idesc_n64 : idesc_n;
                    if (a.f16) {
                        // offset split: [hi.hi | hi.lo'] + lo'.hi into the lo' half (scaled
                        // back by 2^-11 in the epilogue); K = 16 halves per 32-byte slice
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            ptx::mma_f16_ss(dcol, da + 2 * ks, bd0 + 2 * ks, i2, (kl | ks) > 0);
                            ptx::mma_f16_ss(dcol + (uint32_t)a.LO, da + lo_units + 2 * ks,
                                            bd0 + 2 * ks, i1, 1);
                        }
                    } else {
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            ptx::mma_tf32_ss(dcol, da + 2 * ks, bd0 + 2 * ks, i2, (kl | ks) > 0);
                            ptx::mma_tf32_ss(dcol, da + lo_units + 2 * ks, bd0 + 2 * ks, i1, 1);
                        }
                    }
                }
                ptx::mma_commit(&sempty[s]);
            }
            __syncwarp();
            WS_TRACE(a, kl, 9, lane == 0);
            if (++s == a.SS) {
                s = 0;
                ph ^= 1;
            }
        }
        if (ptx::elect_one()) ptx::mma_commit(&accfull);
        __syncwarp();
    } else {
        // ================================ converters ================================
        const int tid = threadIdx.x;  // 0..255
        const int nchunks = a.NB * 8;    // 16-byte chunks of the dy tiles
        const int db0 = (a.J - 1) * a.Q * 8;  // the unshifted copy (jb' = J-1): db
        const int db1 = db0 + a.Q * 8;
        // B rows past J*Q are never loaded: zero them once in every stage (combined fp16 dy
        // box: the rows past both halves)
        for (int st_ = 0; st_ < a.SS; ++st_) {
            float4 *bh = reinterpret_cast<float4 *>(smem + (size_t)st_ * a.b_bytes);
            const int z0 = (a.dycomb ? 2 : 1) * a.J * a.Q * 8, z1 = (a.dycomb ? 2 : 1) * nchunks;
            for (int idx = z0 + tid; idx < z1; idx += WS_CONV_WARPS * 32)
                bh[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float dbacc[4] = {0.f, 0.f, 0.f, 0.f};
        const int lchunks = a.Ls * 8;    // 16-byte chunks of a ring slot
        WsSched sc(a, kb_first, n_i);
        int s = 0;
        uint32_t ph = 0;
        for (int kl = 0; kl < nkb; ++kl, sc.next()) {
            ptx::mbar_wait(&sfull[s], ph);
            WS_TRACE(a, kl, 2, tid == 0);
            unsigned char *st = smem + (size_t)s * a.b_bytes;
            if (a.f16) {
                // db from the staged split: dy = hi + lo' * 2^-11 (8 halves per chunk)
                const uint4 *bh = reinterpret_cast<const uint4 *>(st);
                const uint4 *bl = reinterpret_cast<const uint4 *>(st + (uint32_t)a.LO * 128);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int idx = tid + 256 * m;
                    if (idx >= nchunks) break;
                    if (idx < db0 || idx >= db1) continue;
                    const uint4 h4 = bh[idx], l4 = bl[idx];
                    const uint32_t hw[4] = {h4.x, h4.y, h4.z, h4.w}, lw[4] = {l4.x, l4.y, l4.z, l4.w};
                    float sum = 0.f;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&hw[q]));
                        const float2 lf = __half22float2(*reinterpret_cast<const __half2 *>(&lw[q]));
                        sum += (hf.x + lf.x * (1.f / ptx::F16_LO_SCALE)) +
                               (hf.y + lf.y * (1.f / ptx::F16_LO_SCALE));
                    }
                    dbacc[m] += sum;
                }
            } else {
                // B_lo = B_hi - trunc(B_hi) (elementwise; the swizzle is preserved) + db
                const float4 *bh = reinterpret_cast<const float4 *>(st);
                float4 *bl = reinterpret_cast<float4 *>(st + (uint32_t)a.NB * 128);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int idx = tid + 256 * m;
                    if (idx >= nchunks) break;
                    const float4 v = bh[idx];
                    if (idx >= db0 && idx < db1) dbacc[m] += (v.x + v.y) + (v.z + v.w);
                    bl[idx] = make_float4(ptx::tf32_lo(v.x), ptx::tf32_lo(v.y), ptx::tf32_lo(v.z),
                                          ptx::tf32_lo(v.w));
                }
            }
            // lo lines of the rows this block added (and their mirrors)
            const int k0 = sc.cstart ? 0 : n_i - 1;
            for (int k = k0; k < n_i; ++k) {
                int slot = sc.Bm + k;
                if (slot >= a.R) slot -= a.R;
                const float4 *src =
                    reinterpret_cast<const float4 *>(smem + a.ring_hi + (size_t)slot * a.slot_bytes);
                float4 *dst = reinterpret_cast<float4 *>(smem + a.ring_lo + (size_t)slot * a.slot_bytes);
                float4 *dst2 = slot < a.NM ? reinterpret_cast<float4 *>(
                                                 smem + a.ring_lo + (size_t)(a.R + slot) * a.slot_bytes)
                                           : nullptr;
                // the hi mirror too (one TMA row request less per mirrored row: the TMA
                // unit's row rate is this kernel's feed limit)
                float4 *hm = (slot < a.NM && !a.tma_mirror)
                                 ? reinterpret_cast<float4 *>(smem + a.ring_hi +
                                                              (size_t)(a.R + slot) * a.slot_bytes)
                                 : nullptr;
                if (a.f16) {  // lo' came with the row (TMA): only the mirrors are copied
                    if (slot < a.NM)
                        for (int idx = tid; idx < lchunks; idx += WS_CONV_WARPS * 32) {
                            dst2[idx] = dst[idx];
                            if (hm) hm[idx] = src[idx];
                        }
                    continue;
                }
                for (int idx = tid; idx < lchunks; idx += WS_CONV_WARPS * 32) {
                    const float4 v = src[idx];
                    const float4 lo = make_float4(ptx::tf32_lo(v.x), ptx::tf32_lo(v.y),
                                                  ptx::tf32_lo(v.z), ptx::tf32_lo(v.w));
                    dst[idx] = lo;
                    if (dst2) dst2[idx] = lo;
                    if (hm) hm[idx] = v;
                }
            }
            WS_TRACE(a, kl, 3, tid == 0);
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&cfull[s]);
            WS_TRACE(a, kl, 4, tid == 0);
            if (++s == a.SS) {
                s = 0;
                ph ^= 1;
            }
        }
        // ---- db partials: thread tid owns dy rows (tid >> 3) + 32 m
        if (g == 0) {
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                float v = dbacc[m];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                const int row = (tid >> 3) + 32 * m - (a.J - 1) * a.Q;
                if ((lane & 7) == 0 && row >= 0 && row < a.Q)
                    a.pdb[(size_t)split * a.Npad + row] = v;
            }
        }
        // ---- epilogue: tiles t = grp, grp + 2, ...; lane = line
        const int q = warp & 3, grp = warp >> 2;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        if (nkb > 0) {
            ptx::mbar_wait_sleep(&accfull, 0);
            ptx::tc_fence_after();
        }
        const size_t rows_pad = (size_t)a.n_tiles * 128;
        for (int t = grp; t < G; t += 2) {
            const bool m64 = tail64 && t == G - 1;
            // M = 64 tile: rows live in lanes 0-15 of each quadrant (lanes 16-31 unused)
            const int grow = (tile0 + t) * 128 + (m64 ? q * 16 : q * 32) + lane;
            const bool store = !m64 || lane < 16;
            float *dstp = a.part + ((size_t)split * rows_pad + grow) * a.NB;
            for (int o0 = 0; o0 < a.NB; o0 += 16) {
                uint32_t h[16], l2[16];
                if (nkb > 0) {
                    const uint32_t dcol = tmem + lane_off + (uint32_t)(t * acc_cols + o0);
                    ptx::tmem_ld16(dcol, h);
                    ptx::tmem_ld16(dcol + a.LO, l2);
                    ptx::tmem_wait_ld();
                }
#pragma unroll
                for (int k = 0; k < 16; k += 4) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    const float ls = a.f16 ? 1.f / ptx::F16_LO_SCALE : 1.f;  // offset split
                    if (nkb > 0)
                        v = make_float4(__uint_as_float(h[k]) + __uint_as_float(l2[k]) * ls,
                                        __uint_as_float(h[k + 1]) + __uint_as_float(l2[k + 1]) * ls,
                                        __uint_as_float(h[k + 2]) + __uint_as_float(l2[k + 2]) * ls,
                                        __uint_as_float(h[k + 3]) + __uint_as_float(l2[k + 3]) * ls);
                    if (store) *reinterpret_cast<float4 *>(dstp + o0 + k) = v;
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == WS_MMA_WARP) ptx::tmem_dealloc<512>(tmem);
}

// dw[o,c,i,j] = sum_s part[s][line(i, j, c)][o], db[o] = sum_s pdb[s][o].  A block takes 32
// entries (lanes, (line, col) with col fastest: coalesced) x 8 warps; warp w sums the splits
// s = w, w + 8, ... in order, then lane sums of the 8 warps are added in warp order -- a
// fixed order (deterministic) with 8 independent load chains per entry instead of one
// (a single ~148-long chain per thread left the kernel latency bound).  Gap lines
// (residue-box padding), zero B rows and padding taps are skipped.
constexpr int WR_GROUPS = 8;
__global__ void __launch_bounds__(32 * WR_GROUPS)
    ws_reduce(const float *__restrict__ part, const float *__restrict__ pdb, float *__restrict__ dw,
              float *__restrict__ db, int Q, int C, int l, int Ls, int Npad, int J, int Ja,
              int splits, int rows_pad, WsResidues rs, const int *exit_if,
              const int *exit_unless, int ilv) {
    if ((exit_if && *(volatile const int *)exit_if) ||
        (exit_unless && !*(volatile const int *)exit_unless))
        return;
    __shared__ float red[WR_GROUPS][32];
    const long long lines = (long long)l * Ls;
    const int NB = (J * Q + 15) / 16 * 16;
    const long long total = lines * NB;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long idx = (long long)blockIdx.x * 32 + lane;
    // which entry, and where its partials live (src < 0: nothing to write)
    long long src = -1, sstride = 0, dst = -1;
    const float *in = part;
    float *out = nullptr;
    if (idx < total) {
        const int col = (int)(idx % NB);
        const long long line = idx / NB;
        int o = 0, c = 0, i = 0, j = l;
        if (col < J * Q) {  // else a zero B row
            const int jr = col / Q;
            o = col - jr * Q;
            const int jb = J - 1 - jr;  // B row blocks hold the shifts in reverse
            i = (int)(line / Ls);
            const int rem = (int)(line - (long long)i * Ls);
            int rb = -1;
            for (int r = 0; r < rs.n_b; ++r)
                if (rem >= rs.line0[r] && rem < rs.line0[r] + C * rs.n[r]) rb = r;
            if (rb >= 0) {  // else a gap line
                const int off = rem - rs.line0[rb];
                c = off / rs.n[rb];
                const int jj = off - c * rs.n[rb];
                const int ja = rs.tapcopy ? jj : rs.j0[rb] + jj * rs.step;
                j = ilv ? ja * J + jb : jb * Ja + ja;  // >= l: a padding tap
                if (rb == 0 && jj >= rs.nreal0) j = l;  // box-padding tap line
            }
        }
        if (j < l) {
            src = line * NB + col;
            sstride = (long long)rows_pad * NB;
            dst = (((long long)o * C + c) * l + i) * l + j;
            out = dw;
        }
    } else if (idx < total + Q) {
        src = idx - total;
        sstride = Npad;  // pdb: Npad wide
        dst = src;
        in = pdb;
        out = db;
    }
    float acc = 0.f;
    if (src >= 0)
        for (int sp = w; sp < splits; sp += WR_GROUPS) acc += in[(size_t)sp * sstride + src];
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0 && src >= 0) {
        float t = red[0][lane];
#pragma unroll
        for (int g = 1; g < WR_GROUPS; ++g) t += red[g][lane];
        out[dst] = t;
    }
}

// --------------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------------
struct WsPlan {
    int pair, direct, f16;
    int ilv;  // fp16 interleaved taps: j = ja*J + jb, x taps J*d apart, J staged dy copies
              // shifted by jb*d (copies, not an overlapping view: d*2 bytes is no 16-byte step)
    int J, kc, dc, sb, NB;  // J dy copies (B), kc = Ja column taps in the x lines (A), step dc = d
    int Cpad, Npad, Ls, n_tiles, G, n_groups, splits, SS, R, NM, max_ni;
    int ho, wo, nvb, T, wp_x, wp_dy, lm_dy, mask;
    bool stage_dy;
    long long kb_total;
    WsResidues rs;
    size_t part_bytes, pdb_bytes, copy_bytes, x_bytes, dy_bytes, total_bytes;
    uint32_t b_bytes, slot_bytes, box_tx_row;
};

static size_t ws_align256(size_t v) { return (v + 255) / 256 * 256; }

static bool ws_plan_j(int n, int cin, int hi, int wi, int cout, int k, int d, int Ja,
                      WsPlan &p, bool f16 = false);

// x read in place (no tc_stage_x copy): one residue at offset 0 (every tap offset j*d a
// multiple of 4 floats), 16-byte rows, no 2-row boxes (a 6th map dimension), and the caller
// guarantees that the bytes an overlapping tap view reads past the tensor's last row exist
// (x_slack).  Rows past Hi then come from TMA zero fill instead of the next image.
static void ws_try_direct(WsPlan &p, int cin, int wi, int d, size_t x_slack) {
    p.direct = 0;
    if (getenv("DP_WG_STAGE_X") || p.rs.tapcopy || p.rs.n_b != 1 || p.rs.b[0] != 0 ||
        wi % 4 != 0)
        return;
    const size_t overrun = ((size_t)(p.rs.n[0] - 1) * p.rs.step * d + 32) * 4;
    if (x_slack < overrun) return;
    p.direct = 1;
    if (p.pair) {
        p.pair = 0;
        p.rs.n[0] = p.rs.nreal0;
        p.box_tx_row = (uint32_t)cin * p.kc * 128u;
    }
    p.R = p.max_ni + p.SS - 1;
    p.total_bytes -= p.x_bytes;
    p.x_bytes = 0;
}

// Column-tap stacking: column tap j = jb*Ja + ja.  The x lines (A) cover only Ja taps ja
// (offsets ja*d), and J = ceil(k / Ja) copies of dy shifted right by jb*Ja*d sit side by
// side in the B operand (N = J * Q, rounded up to 16): J times fewer A lines -- fewer M tiles, i.e. fewer A
// reads from shared memory per useful MAC -- for wider MMAs and J dy boxes per K block.  The
// shift must be a multiple of 4 floats (a TMA box starts on a 16-byte boundary), so J > 1
// needs 4 | Ja*d (Ja = k: no stacking, the unstacked kernel).  Ja is picked by a per-K-block
// cost model of the shared-memory operand bytes (A hi + lo per tile, B per MMA) and issue
// slots; DP_WG_J=<J> forces the smallest legal Ja with that many dy copies.
static bool ws_plan(int n, int cin, int hi, int wi, int cout, int k, int d, WsPlan &p,
                    bool f16 = false) {
    if (const char *e = getenv("DP_WG_J")) {
        const int J = atoi(e);
        for (int Ja = 1; Ja <= k && J >= 1; ++Ja)
            if ((k + Ja - 1) / Ja == J && ws_plan_j(n, cin, hi, wi, cout, k, d, Ja, p, f16))
                return true;
    }
    bool ok = false;
    double best = 0;
    for (int Ja = k; Ja >= 1; --Ja) {
        WsPlan q;
        if (!ws_plan_j(n, cin, hi, wi, cout, k, d, Ja, q, f16)) continue;
        // cycles per K block (measured model): the tensor core -- an SS MMA costs
        // max(39, N/2) cycles (tools/tc_probe.cu), 2 per K=8 slice and tile, 4 slices, plus
        // the commit -- or the TMA producer, ~550 cycles per box (dy + the x boxes of the
        // new row; half an x box when two rows share one), whichever is slower
        auto mma = [](int N) { return std::max(39.0, N / 2.0); };
        const double mma_cycles = 4.0 * q.n_tiles * (mma(2 * q.NB) + mma(q.NB)) + 300.0;
        const double boxes = 1.0 + (q.pair ? 0.5 : (double)q.rs.n_b);
        double cost = std::max(mma_cycles, 550.0 * boxes);
        cost *= (double)q.nvb;  // K blocks per row grow with the (J-1) Ja d shift
        if (!ok || cost < best) {
            best = cost;
            p = q;
            ok = true;
        }
    }
    // fp16 with tap offsets in two or more 16-byte classes (c3 conv2: d = 4): the interleaved
    // mode instead -- x taps J*d apart (one class, in place), J dy copies shifted by jb*d.
    // Opt-in (DP_WG_F16_ILV=1): c3 conv2 measured 2.66 ms against 1.86 on 3xTF32 (224 TMEM
    // columns per tile leave 2-tile groups, so every K block is fed twice, plus J staging passes)
    if (f16 && (!ok || p.rs.n_b > 1 || p.rs.tapcopy) && getenv("DP_WG_F16_ILV")) {
        int g = 8;
        while (d % g) g >>= 1;
        WsPlan q;
        if (8 / g >= 2 && ws_plan_j(n, cin, hi, wi, cout, k, d, -(8 / g), q, f16) &&
            q.rs.n_b == 1 && !q.rs.tapcopy) {
            p = q;
            ok = true;
        }
    }
    return ok;
}

// f16: the fp16-split variant (x pre-split into fp16 hi / lo' NCHW tensors read in place,
// dy staged as fp16 hi / lo'; K blocks of 64 px so a 128-byte line still holds one K block):
// residues are tap offsets mod 8 halves (16 bytes), at most two (one in-place box each),
// no per-tap copies, no 2-row boxes
static bool ws_plan_j(int n, int cin, int hi, int wi, int cout, int k, int d, int Ja,
                      WsPlan &p, bool f16) {
    if (getenv("DP_WG_TMEM")) return false;  // force the TMEM-operand kernel (experiments)
    p.f16 = f16 ? 1 : 0;
    const int KB = f16 ? 64 : 32;  // pixels per K block (one 128-byte line)
    const int e = (k - 1) * d + 1;
    p.ho = hi - e + 1;
    p.wo = wi - e + 1;
    if (p.ho < 1 || p.wo < 1 || k > 64) return false;
    p.Npad = (cout + 15) / 16 * 16;
    if (p.Npad > 128) return false;
    // Ja < 0: the fp16 interleaved mode with J = -Ja dy copies (ws_plan)
    p.ilv = Ja < 0 ? 1 : 0;
    if (p.ilv) {
        if (!f16 || -Ja < 2 || -Ja > k) return false;
        Ja = (k + (-Ja) - 1) / (-Ja);  // x taps per group
    }
    if (Ja < 1 || Ja > k) return false;
    const int J = (k + Ja - 1) / Ja;
    p.J = J;
    p.NB = (J * cout + 15) / 16 * 16;
    if (2 * p.NB > 256) return false;
    p.kc = Ja;
    p.dc = p.ilv ? J * d : d;  // column step between the x lines' taps
    p.sb = p.ilv ? d : p.kc * d;
    if (J > 1 && !p.ilv && (p.sb & (f16 ? 7 : 3))) return false;
    const int kc = p.kc, dc = p.dc;
    const int RM = f16 ? 8 : 4;  // residue modulus: elements per 16 bytes
    p.Cpad = (cin + 7) / 8 * 8;
    if (p.Cpad > 256) return false;
    // lines per ring slot (one input row): residue boxes, each rounded up to 8 lines.  Small
    // channel counts with several residues would mean several tiny boxes per K block (TMA
    // issue bound, measured on c2 conv1: cin 3, d 1); those stage one copy per tap instead
    // and load a row with a single {32, l, cin} box.
    int nres = 0;
    {
        int ls = 0;
        for (int b = 0; b < RM; ++b) {
            int cnt = 0;
            for (int j = 0; j < kc; ++j) cnt += ((j * dc) % RM) == b;
            if (cnt) {
                ls += (cin * cnt + 7) / 8 * 8;
                ++nres;
            }
        }
        p.Ls = ls;
    }
    if (f16 && nres > 2) return false;
    p.rs.tapcopy = (!f16 && nres > 1 && cin * kc <= 32 && !getenv("DP_WG_RESIDUE")) ? 1 : 0;
    if (p.rs.tapcopy) p.Ls = (cin * kc + 7) / 8 * 8;
    // 2-row x boxes need one box per row whose lines fill the slot exactly (the tap
    // dimension is padded with zero-filled taps to Ls / cin)
    // (only for rows of <= 8 KB: a 2-row box of 16-KB rows measured 23 % slower, c2 conv3 J=1)
    p.pair = (!f16 && (nres == 1 || p.rs.tapcopy) && p.Ls % cin == 0 && p.Ls <= 64 &&
              !getenv("DP_WG_NOPAIR") && !getenv("DP_WG_TMA_MIRROR"))
                 ? 1
                 : 0;
    const int lines = k * p.Ls;
    p.n_tiles = (lines + 127) / 128;
    const int acc_cols = 2 * p.NB;
    p.slot_bytes = (uint32_t)p.Ls * 128u;  // multiple of 8 lines: 1024-byte aligned boxes
    p.b_bytes = 2u * (uint32_t)p.NB * 128u;
    // Tile groups: as many tiles per CTA as TMEM holds, unless the ring (hi + lo slots for
    // the group's tap rows + SS - 1 + mirrors) does not fit -- then smaller groups (fewer
    // tap rows each; every group re-reads its rows), down to one tile.
    p.SS = 0;
    int g_max = std::min(std::min(p.n_tiles, 512 / acc_cols), WS_MAX_G);
    if (const char *e = getenv("DP_WG_GMAX"))  // experiments: smaller tile groups, more stages
        g_max = std::max(1, std::min(g_max, atoi(e)));
    for (int G = g_max; G >= 1 && !p.SS; --G) {
        p.n_groups = (p.n_tiles + G - 1) / G;
        p.G = (p.n_tiles + p.n_groups - 1) / p.n_groups;
        // tap rows per group and the ring slots a 128-line tile can span
        p.max_ni = 0;
        int span = 1;
        for (int g = 0; g < p.n_groups; ++g) {
            const int t0 = g * p.G, G_ = std::min(p.G, p.n_tiles - t0);
            const int i_lo = t0 * 128 / p.Ls;
            const int n_i = (std::min((t0 + G_) * 128, lines) - 1) / p.Ls - i_lo + 1;
            p.max_ni = std::max(p.max_ni, n_i);
            for (int t = 0; t < G_; ++t) {
                const int line0 = (t0 + t) * 128 - i_lo * p.Ls;
                const int f = line0 % p.Ls;
                span = std::max(span, (f + 128 + p.Ls - 1) / p.Ls);
            }
        }
        p.NM = span - 1;
        for (int ss = WS_MAX_SS; ss >= 2; --ss) {
            const size_t need = (size_t)ss * p.b_bytes +
                                2 * (size_t)(p.max_ni + ss - 1 + p.pair + p.NM) * p.slot_bytes;
            if (need <= (size_t)WS_SMEM_BUDGET) {
                p.SS = ss;
                break;
            }
        }
    }
    if (p.SS < 2) return false;
    // a 2-row box fills the next block's slot one block early: one more slot
    p.R = p.max_ni + p.SS - 1 + p.pair;
    // residue copies: column taps jo with (jo*dc) & 3 == b, lcm(dc, 4) floats apart
    int gcd = 1;
    for (int v = RM; v >= 1; --v)
        if (dc % v == 0 && RM % v == 0) {
            gcd = v;
            break;
        }
    p.rs.step = RM / gcd;
    p.mask = 0;
    p.rs.n_b = 0;
    if (p.rs.tapcopy) {  // one "residue" holding all kc taps (copy jo pre-shifted by jo*dc)
        p.rs.n_b = 1;
        p.rs.b[0] = 0;
        p.rs.n[0] = kc;
        p.rs.j0[0] = 0;
        p.rs.line0[0] = 0;
        p.rs.step = 1;
        for (int rb = 1; rb < 4; ++rb) {
            p.rs.b[rb] = -1;
            p.rs.n[rb] = p.rs.j0[rb] = p.rs.line0[rb] = 0;
        }
    }
    int line0 = 0;
    for (int b = 0; b < RM && !p.rs.tapcopy; ++b) {
        int cnt = 0, j0 = -1;
        for (int j = 0; j < kc; ++j)
            if (((j * dc) % RM) == b) {
                if (j0 < 0) j0 = j;
                ++cnt;
            }
        if (!cnt) continue;
        if (cnt > 256) return false;
        const int rb = p.rs.n_b++;
        p.rs.b[rb] = b;
        p.rs.n[rb] = cnt;
        p.rs.j0[rb] = j0;
        p.rs.line0[rb] = line0;
        // a residue's box holds cin * cnt real lines; the next box starts on a 1024-byte
        // (8-line) boundary (SWIZZLE_128B).  The gap lines are never written: they only
        // feed their own (discarded) accumulator rows.
        line0 += (cin * cnt + 7) / 8 * 8;
        p.mask |= 1 << b;
    }
    for (int rb = p.rs.n_b; rb < 4; ++rb) {
        p.rs.b[rb] = -1;
        p.rs.n[rb] = p.rs.j0[rb] = p.rs.line0[rb] = 0;
    }
    p.rs.nreal0 = p.rs.n[0];
    if (p.pair) p.rs.n[0] = p.Ls / cin;  // padded tap count: box lines per row == Ls
    // bytes the residue boxes of one row deliver (zero-filled padding taps included)
    p.box_tx_row = (uint32_t)cin * (p.pair ? p.rs.n[0] : kc) * 128u;
    // K runs over x-aligned columns: dy shifted by up to (J-1) Ja d needs that many more
    p.nvb = (p.wo + (J - 1) * p.sb + KB - 1) / KB;
    p.T = (p.ho + d - 1) / d;
    p.kb_total = (long long)n * p.nvb * d * p.T;
    p.splits = wg_sms() / p.n_groups;
    if (p.splits < 1) p.splits = 1;
    if (p.splits > p.kb_total) p.splits = (int)p.kb_total;
    p.wp_x = (wi + 3) / 4 * 4;
    // J > 1: dy always staged, with (J-1)*sb zeros left of each row and zeros right of it up
    // to the last K block's reach, so the overlapping-view box never leaves the row
    p.lm_dy = (J - 1) * p.sb;
    p.wp_dy = J > 1 ? p.nvb * KB + p.lm_dy : (f16 ? (p.wo + 7) / 8 * 8 : (p.wo + 3) / 4 * 4);
    if (p.ilv) p.wp_dy = (p.wp_dy + 7) / 8 * 8;  // (margins of d halves: keep 16-byte rows)
    p.stage_dy = f16 || J > 1 || p.wp_dy != p.wo;
    if ((long long)n * hi > (1LL << 31)) return false;
    p.part_bytes = ws_align256((size_t)p.splits * p.n_tiles * 128 * p.NB * 4);
    p.pdb_bytes = ws_align256((size_t)p.splits * p.Npad * 4);
    // boxes read up to (kc*J-1)*d + 32 floats past a row's end (those columns meet zero dy)
    p.copy_bytes =
        ws_align256((size_t)n * cin * hi * p.wp_x * 4 + ((size_t)(kc * J - 1) * d + 64) * 4);
    p.x_bytes = f16 ? 0 : (size_t)(p.rs.tapcopy ? kc : p.rs.n_b) * p.copy_bytes;
    // f16: dy staged as two fp16 tensors (hi, lo')
    p.dy_bytes = !p.stage_dy ? 0
                 : f16 ? 2 * (p.ilv ? J : 1) * ws_align256((size_t)n * cout * p.ho * p.wp_dy * 2)
                       : ws_align256((size_t)n * cout * p.ho * p.wp_dy * 4);
    p.total_bytes = p.part_bytes + p.pdb_bytes + p.x_bytes + p.dy_bytes;
    return true;
}

// debugging aid (dp_debug_wgrad_plan): the smem-operand weight gradient's plan, 0 if
// unsupported; out = {J, Ja, NB, Ls, n_tiles, G, n_groups, splits, SS, pair, stage_dy,
// residues, tapcopy, x_bytes / 1 KiB, dy_bytes / 1 KiB, total_bytes / 1 KiB}
int ws_debug_plan(int n, int cin, int hi, int wi, int cout, int k, int d, int *out, int len) {
    WsPlan p;  // DP_WG_DEBUG_F16: the fp16-split plan
    if (!ws_plan(n, cin, hi, wi, cout, k, d, p, getenv("DP_WG_DEBUG_F16") != nullptr)) return 0;
    const int v[16] = {p.J, p.kc, p.NB, p.Ls, p.n_tiles, p.G, p.n_groups, p.splits, p.SS,
                       p.pair, p.stage_dy ? 1 : 0, p.rs.n_b, p.rs.tapcopy,
                       (int)(p.x_bytes >> 10), (int)(p.dy_bytes >> 10),
                       (int)(p.total_bytes >> 10)};
    for (int i = 0; i < len && i < 16; ++i) out[i] = v[i];
    return 1;
}

bool ws_supported(int n, int cin, int hi, int wi, int cout, int k, int d) {
    WsPlan p;
    return ws_plan(n, cin, hi, wi, cout, k, d, p);
}

size_t ws_workspace(int n, int cin, int hi, int wi, int cout, int k, int d) {
    WsPlan p;
    return ws_plan(n, cin, hi, wi, cout, k, d, p) ? p.total_bytes : 0;
}

// phases: 1 = stage x into the workspace, 2 = everything else (dy staging, kernel,
// reduction); 3 = both.  Staging x is independent of dy, so the engine runs phase 1 during
// the forward pass (side stream) and phase 2 in the backward.
int ws_conv_backward_kernel(const float *x, const float *dy, float *dw, float *db, int n,
                            int cin, int hi, int wi, int cout, int k, int d, void *ws,
                            size_t ws_bytes, cudaStream_t st, int phases, size_t x_slack,
                            int dy_pitch, const int *exit_unless) {
    WsPlan p;
    if (!ws_plan(n, cin, hi, wi, cout, k, d, p))
        return set_error(DP_ERR_UNSUPPORTED, "weight gradient (smem operands): unsupported shape");
    p.direct = 0;
    if (phases == 3 && ((uintptr_t)x & 15) == 0) ws_try_direct(p, cin, wi, d, x_slack);
    if (ws == nullptr || ws_bytes < p.total_bytes)
        return set_error(DP_ERR_ARG, "tensor-core weight gradient: workspace %zu < %zu bytes",
                         ws_bytes, p.total_bytes);
    if (((uintptr_t)ws & 255) != 0)
        return set_error(DP_ERR_ARG,
                         "tensor-core weight gradient: workspace must be 256-byte aligned");
    unsigned char *w8 = (unsigned char *)ws;
    WsArgs a;
    a.part = (float *)w8;
    a.pdb = (float *)(w8 + p.part_bytes);
    float *xs = (float *)(w8 + p.part_bytes + p.pdb_bytes);
    int rc = DP_OK;
    if ((phases & 1) && !p.direct) {
        rc = p.rs.tapcopy ? wg_stage_x_taps(x, xs, n, cin, hi, wi, p.wp_x, p.kc, p.dc,
                                            (long long)(p.copy_bytes / 4), st)
                          : wg_stage_x(x, xs, n, cin, hi, wi, p.wp_x, p.mask,
                                       (long long)(p.copy_bytes / 4), st);
        if (rc) return rc;
    }
    if (!(phases & 2)) return DP_OK;
    // dy in place when its rows are 16-byte aligned: unpadded (wo % 4 == 0) or handed over
    // with a 16-byte row pitch by the producer (dy_pitch, engine layer 0)
    const int pitch = dy_pitch > 0 ? dy_pitch : p.wo;
    const bool pitched_ok = p.J == 1 && pitch % 4 == 0 && ((uintptr_t)dy & 15) == 0;
    const bool stage_dy = (p.stage_dy && !pitched_ok) || ((uintptr_t)dy & 15) != 0;
    if (stage_dy && !p.stage_dy)
        return set_error(DP_ERR_ARG, "weight gradient: dy must be 16-byte aligned");
    const float *dys = dy;
    if (stage_dy) {
        float *dp_ = (float *)(w8 + p.part_bytes + p.pdb_bytes + p.x_bytes);
        rc = wg_stage_dy(dy, dp_, n, cout, p.ho, p.wo, p.wp_dy, p.lm_dy, st, pitch, exit_unless);
        if (rc) return rc;
        dys = dp_;
    }
    CUtensorMap mx[4], mdy;
    {
        const cuuint64_t rowb = (cuuint64_t)(stage_dy ? p.wp_dy : pitch) * 4;
        if (p.J == 1) {
            cuuint64_t dims[4] = {(cuuint64_t)p.wo, (cuuint64_t)p.ho, (cuuint64_t)cout, (cuuint64_t)n};
            cuuint64_t str[3] = {stage_dy ? rowb * cout : rowb, stage_dy ? rowb : rowb * p.ho,
                                 rowb * cout * p.ho};
            cuuint32_t box[4] = {32, 1, (cuuint32_t)cout, 1};
            rc = wg_make_map(&mdy, dys, 4, dims, str, box, true);
        } else {
            // (w, o, jb', h, n) over the staged (n, h, o, wp) rows; jb' steps sb floats
            cuuint64_t dims[5] = {(cuuint64_t)p.wp_dy, (cuuint64_t)cout, (cuuint64_t)p.J,
                                  (cuuint64_t)p.ho, (cuuint64_t)n};
            cuuint64_t str[4] = {rowb, (cuuint64_t)p.sb * 4, rowb * cout, rowb * cout * p.ho};
            cuuint32_t box[5] = {32, (cuuint32_t)cout, (cuuint32_t)p.J, 1, 1};
            rc = wg_make_map(&mdy, dys, 5, dims, str, box, true);
        }
        if (rc) return rc;
    }
    const cuuint64_t xrow = (cuuint64_t)p.wp_x * 4;  // one channel line
    const cuuint64_t ximg_row = xrow * cin;          // one image row (all channels)
    for (int rb = 0; rb < 4 && p.direct; ++rb) {
        // x in place, NCHW: (w, jj: step*d floats, c, h, n); one box = the (c, jj) lines
        cuuint64_t dims[5] = {(cuuint64_t)wi, (cuuint64_t)p.rs.nreal0, (cuuint64_t)cin,
                              (cuuint64_t)hi, (cuuint64_t)n};
        cuuint64_t str[4] = {(cuuint64_t)p.rs.step * p.dc * 4, (cuuint64_t)hi * wi * 4,
                             (cuuint64_t)wi * 4, (cuuint64_t)cin * hi * wi * 4};
        cuuint32_t box[5] = {32, (cuuint32_t)p.rs.n[0], (cuuint32_t)cin, 1, 1};
        rc = wg_make_map(&mx[rb], x, 5, dims, str, box, true);
        if (rc) return rc;
    }
    for (int rb = 0; rb < 4 && !p.direct; ++rb) {
        const int used = rb < p.rs.n_b ? rb : 0;
        const float *base = (const float *)((const unsigned char *)xs + (size_t)used * p.copy_bytes);
        // (w, jj: lcm(d, 4) floats, c, row of n*hi) -- overlapping views, one box = the
        // residue's (c, jj) lines of one input row
        cuuint64_t dims[4] = {(cuuint64_t)p.wp_x,
                              (cuuint64_t)(used == 0 ? p.rs.nreal0 : p.rs.n[used]),
                              (cuuint64_t)cin, (cuuint64_t)n * hi};
        // tap dimension: lcm(d, 4) floats inside a residue copy, or the copy stride when each
        // tap has its own pre-shifted copy
        cuuint64_t str[3] = {p.rs.tapcopy ? (cuuint64_t)p.copy_bytes : (cuuint64_t)p.rs.step * p.dc * 4,
                             xrow, ximg_row};
        cuuint32_t box[4] = {32, (cuuint32_t)p.rs.n[used], (cuuint32_t)cin, 1};
        rc = wg_make_map(&mx[rb], base, 4, dims, str, box, true);
        if (rc) return rc;
    }
    CUtensorMap mxp = mx[0];
    if (p.pair) {
        // residue 0's view with two rows d apart: (w, jj, c, q: d rows, r: rows of n*hi)
        cuuint64_t dims[5] = {(cuuint64_t)p.wp_x, (cuuint64_t)p.rs.nreal0, (cuuint64_t)cin, 2,
                              (cuuint64_t)n * hi};
        cuuint64_t str[4] = {p.rs.tapcopy ? (cuuint64_t)p.copy_bytes
                                          : (cuuint64_t)p.rs.step * p.dc * 4,
                             xrow, ximg_row * (cuuint64_t)d, ximg_row};
        cuuint32_t box[5] = {32, (cuuint32_t)p.rs.n[0], (cuuint32_t)cin, 2, 1};
        rc = wg_make_map(&mxp, xs, 5, dims, str, box, true);
        if (rc) return rc;
    }
    a.C = cin;
    a.Cpad = p.Cpad;
    a.l = k;
    a.d = d;
    a.Q = cout;
    a.Npad = p.Npad;
    a.J = p.J;
    a.sb = p.sb;
    a.NB = p.NB;
    a.tma_mirror = getenv("DP_WG_TMA_MIRROR") ? 1 : 0;
    a.f16 = 0;
    a.dycomb = 0;
    a.LO = p.NB;
    a.dy_rows = 0;
    a.pair = p.pair;
    a.direct = p.direct;
    a.n_tiles = p.n_tiles;
    a.G = p.G;
    a.n_groups = p.n_groups;
    a.splits = p.splits;
    a.Ho = p.ho;
    a.Wo = p.wo;
    a.nvb = p.nvb;
    a.T = p.T;
    a.Hi = hi;
    a.kb_total = p.kb_total;
    a.SS = p.SS;
    {
        // x read in place only (c3 conv2 1.88 -> 1.74 ms at 2-4 blocks ahead; the staged
        // small-box modes lost to the extra TMA requests: c3 conv1 1.33 -> 1.71)
        const char *e = getenv("DP_WG_PF");
        a.pf = e ? atoi(e) : (a.direct ? 3 : 0);
        if (a.pf < 0) a.pf = 0;
    }
    a.R = p.R;
    a.NM = p.NM;
    a.Ls = p.Ls;
    a.b_bytes = p.b_bytes;
    a.slot_bytes = p.slot_bytes;
    a.box_tx_row = p.box_tx_row;
    a.ring_hi = (uint32_t)p.SS * p.b_bytes;
    a.ring_lo = a.ring_hi + (uint32_t)(p.R + p.NM) * p.slot_bytes;
    a.rs = p.rs;
    a.trace = getenv("DP_WG_TRACE") && !exit_unless ? wg_trace_buffer(st) : nullptr;
    a.no_m64 = getenv("DP_WG_NO_M64") ? 1 : 0;
    a.exit_if = nullptr;
    a.exit_unless = exit_unless;
    const size_t smem = (size_t)a.ring_lo + (size_t)(p.R + p.NM) * p.slot_bytes + 1024;
    cudaError_t e = cudaFuncSetAttribute(tc_wgrad_ss_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tc_wgrad_ss: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    const int grid = p.n_groups * p.splits;
    tc_wgrad_ss_kernel<<<grid, WS_THREADS, smem, st>>>(mx[0], mx[1], mx[2], mx[3], mdy, mxp, a);
    rc = check_launch("tc_wgrad_ss_kernel");
    if (rc) return rc;
    const long long total = (long long)k * p.Ls * p.NB + cout;
    ws_reduce<<<ceil_div(total, 32), 32 * WR_GROUPS, 0, st>>>(a.part, a.pdb, dw, db, cout, cin, k, p.Ls,
                                                    p.Npad, p.J, p.kc, p.splits, p.n_tiles * 128,
                                                    p.rs, nullptr, exit_unless, 0);
    return check_launch("ws_reduce");
}

// fp16-split weight gradient: x arrives pre-split as two fp16 NCHW tensors (hi = RN(x),
// lo' = RN((x - hi) * 2^11), the caller's job -- the engine's pool forward emits them) read in
// place; dy is split here.  Same ring / schedule / epilogue as the tf32 kernel with 64-px K
// blocks (one 128-byte line of halves): half the MMAs and shared-memory operand bytes per
// pixel.  Range guard as the fp16 convolutions: the dy split flags any |dy| >= 2^15 (or not
// finite) and the tf32 kernel on the fp32 x runs instead (the caller guarantees |x| < 2^15:
// it splits only bounded activations).  Workspace: [fp16 plan | flag | tf32 plan].
// two residues (shifted copies) are opt-in, DP_WG_F16_RES2=1: measured slower than the tf32
// kernel on c3 conv2 (2.30 vs 1.83 ms: Ls 160 leaves 2 dy stages, 4 x boxes per row)
static bool ws_f16_inplace(const WsPlan &p) {
    const int max_nb = getenv("DP_WG_F16_RES2") ? 2 : 1;
    return p.rs.n_b >= 1 && p.rs.n_b <= max_nb && !p.rs.tapcopy && !p.pair;
}
static size_t ws_f16_overrun(const WsPlan &p, int d) {  // bytes the tap views read past x
    size_t m = 0;
    for (int rb = 0; rb < p.rs.n_b; ++rb)
        m = std::max(m, (size_t)(p.rs.n[rb] - 1) * p.rs.step * p.dc);
    (void)d;
    return (m + 64) * 2;
}

// the shift (halves) of the second residue's copies, 0 when one residue
int ws_shift_f16(int n, int cin, int hi, int wi, int cout, int k, int d) {
    WsPlan p;
    if (!ws_plan(n, cin, hi, wi, cout, k, d, p, true) || !ws_f16_inplace(p)) return -1;
    return p.rs.n_b > 1 ? p.rs.b[1] : 0;
}

size_t ws_workspace_f16(int n, int cin, int hi, int wi, int cout, int k, int d) {
    WsPlan p, q;
    if (!ws_plan(n, cin, hi, wi, cout, k, d, p, true) || !ws_f16_inplace(p) ||
        !ws_plan(n, cin, hi, wi, cout, k, d, q))
        return 0;
    return p.total_bytes + 256 + q.total_bytes;
}

int ws_conv_backward_kernel_f16(const float *x, size_t x_slack, const void *x_hi,
                                const void *x_lo, const void *x_hi_s, const void *x_lo_s,
                                size_t xh_slack, int xh_pitch, const float *dy, int dy_pitch,
                                float *dw, float *db, int n, int cin, int hi, int wi, int cout,
                                int k, int d, void *ws, size_t ws_bytes, cudaStream_t st) {
    WsPlan p, q;
    if (!ws_plan(n, cin, hi, wi, cout, k, d, p, true) || !ws_plan(n, cin, hi, wi, cout, k, d, q))
        return set_error(DP_ERR_UNSUPPORTED, "fp16 weight gradient: unsupported shape");
    // x in place: one residue at offset 0, 16-byte rows of halves, slack for the tap view
    const int xp = xh_pitch > 0 ? xh_pitch : wi;  // halves per row of x_hi / x_lo
    if (!ws_f16_inplace(p) || xp < wi || (xp & 7) || xh_slack < ws_f16_overrun(p, d) ||
        ((uintptr_t)x_hi & 15) || ((uintptr_t)x_lo & 15) || ((uintptr_t)x_hi_s & 15) ||
        ((uintptr_t)x_lo_s & 15))
        return set_error(DP_ERR_UNSUPPORTED, "fp16 weight gradient: x not readable in place");
    if (p.rs.n_b > 1 && (!x_hi_s || !x_lo_s))
        return set_error(DP_ERR_ARG, "fp16 weight gradient: this shape needs the shifted "
                         "copies (shift %d halves)", p.rs.b[1]);
    p.direct = 1;
    p.R = p.max_ni + p.SS - 1;
    const size_t need = p.total_bytes + 256 + q.total_bytes;
    if (ws == nullptr || ws_bytes < need || ((uintptr_t)ws & 255))
        return set_error(DP_ERR_ARG, "fp16 weight gradient: workspace %zu < %zu bytes or "
                         "misaligned", ws_bytes, need);
    unsigned char *w8 = (unsigned char *)ws;
    int *flag = (int *)(w8 + p.total_bytes);
    if (cudaMemsetAsync(flag, 0, sizeof(int), st) != cudaSuccess)
        return set_error(DP_ERR_CUDA, "fp16 weight gradient: flag reset failed");
    WsArgs a;
    a.part = (float *)w8;
    a.pdb = (float *)(w8 + p.part_bytes);
    unsigned char *dhi = w8 + p.part_bytes + p.pdb_bytes;
    unsigned char *dlo = dhi + p.dy_bytes / 2;
    const int pitch = dy_pitch > 0 ? dy_pitch : p.wo;
    int rc = DP_OK;
    const size_t copyb = ws_align256((size_t)n * cout * p.ho * p.wp_dy * 2);
    if (p.ilv) {
        // interleaved taps: J dy copies, copy jb' = dy shifted right by (J-1-jb') d (the
        // rows jb'*Q + o of B, as the overlapping view would give them)
        for (int jb = 0; jb < p.J; ++jb) {
            rc = wg_stage_dy16(dy, dhi + jb * copyb, dlo + jb * copyb, n, cout, p.ho, p.wo,
                               p.wp_dy, (p.J - 1 - jb) * p.sb, st, pitch, flag);
            if (rc) return rc;
        }
    } else {
        rc = wg_stage_dy16(dy, dhi, dlo, n, cout, p.ho, p.wo, p.wp_dy, p.lm_dy, st, pitch, flag);
        if (rc) return rc;
    }
    CUtensorMap mx[4], mdy, mdyl;
    const cuuint64_t rowb = (cuuint64_t)p.wp_dy * 2;
    for (int hl = 0; hl < 2; ++hl) {
        const void *base = hl ? (const void *)dlo : (const void *)dhi;
        CUtensorMap *m = hl ? &mdyl : &mdy;
        if (p.J == 1) {
            cuuint64_t dims[4] = {(cuuint64_t)p.wo, (cuuint64_t)p.ho, (cuuint64_t)cout, (cuuint64_t)n};
            cuuint64_t str[3] = {rowb * cout, rowb, rowb * cout * p.ho};
            cuuint32_t box[4] = {64, 1, (cuuint32_t)cout, 1};
            rc = wg_make_map16(m, base, 4, dims, str, box);
        } else {
            cuuint64_t dims[5] = {(cuuint64_t)p.wp_dy, (cuuint64_t)cout, (cuuint64_t)p.J,
                                  (cuuint64_t)p.ho, (cuuint64_t)n};
            // (interleaved taps: the J copies, copyb apart; else the overlapping view)
            cuuint64_t str[4] = {rowb, p.ilv ? (cuuint64_t)copyb : (cuuint64_t)p.sb * 2,
                                 rowb * cout, rowb * cout * p.ho};
            cuuint32_t box[5] = {64, (cuuint32_t)cout, (cuuint32_t)p.J, 1, 1};
            rc = wg_make_map16(m, base, 5, dims, str, box);
        }
        if (rc) return rc;
    }
    // one box for both halves when J*Q is a multiple of 8 (the stacked MMA's N = 2 J Q then a
    // multiple of 16): the staged rows (n, h) fold into one dimension, the hi -> lo' distance
    // is a fifth (DP_WG_DY2BOX=1: two boxes)
    const int dycomb = (!p.ilv && (p.J * cout) % 8 == 0 && !getenv("DP_WG_DY2BOX")) ? 1 : 0;
    if (dycomb) {
        const cuuint64_t hlb = (cuuint64_t)((unsigned char *)dlo - (unsigned char *)dhi);
        const cuuint64_t rows = (cuuint64_t)n * p.ho;
        if (p.J == 1) {
            cuuint64_t dims[4] = {(cuuint64_t)p.wo, (cuuint64_t)cout, rows, 2};
            cuuint64_t str[3] = {rowb, rowb * cout, hlb};
            cuuint32_t box[4] = {64, (cuuint32_t)cout, 1, 2};
            rc = wg_make_map16(&mdy, dhi, 4, dims, str, box);
        } else {
            cuuint64_t dims[5] = {(cuuint64_t)p.wp_dy, (cuuint64_t)cout, (cuuint64_t)p.J, rows, 2};
            cuuint64_t str[4] = {rowb, (cuuint64_t)p.sb * 2, rowb * cout, hlb};
            cuuint32_t box[5] = {64, (cuuint32_t)cout, (cuuint32_t)p.J, 1, 2};
            rc = wg_make_map16(&mdy, dhi, 5, dims, str, box);
        }
        if (rc) return rc;
    }
    // residue rb's views: mx[2 rb] (hi), mx[2 rb + 1] (lo')
    for (int m = 0; m < 4; ++m) {
        const int rb = std::min(m / 2, p.rs.n_b - 1), hl = m & 1;
        cuuint64_t dims[5] = {(cuuint64_t)wi, (cuuint64_t)p.rs.n[rb], (cuuint64_t)cin,
                              (cuuint64_t)hi, (cuuint64_t)n};
        // (a single-tap view's tap stride is never stepped: any multiple of 16 bytes will do)
        const cuuint64_t tap = p.rs.n[rb] > 1 ? (cuuint64_t)p.rs.step * p.dc * 2 : 16;
        cuuint64_t str[4] = {tap, (cuuint64_t)hi * xp * 2, (cuuint64_t)xp * 2,
                             (cuuint64_t)cin * hi * xp * 2};
        cuuint32_t box[5] = {64, (cuuint32_t)p.rs.n[rb], (cuuint32_t)cin, 1, 1};
        const void *base = rb ? (hl ? x_lo_s : x_hi_s) : (hl ? x_lo : x_hi);
        rc = wg_make_map16(&mx[m], base, 5, dims, str, box);
        if (rc) return rc;
    }
    a.C = cin;
    a.Cpad = p.Cpad;
    a.l = k;
    a.d = d;
    a.Q = cout;
    a.Npad = p.Npad;
    a.J = p.J;
    a.sb = p.sb;
    a.NB = p.NB;
    a.tma_mirror = 0;
    a.pair = 0;
    a.direct = 1;
    a.f16 = 1;
    a.dycomb = dycomb;
    a.LO = dycomb ? p.J * cout : p.NB;
    a.dy_rows = n * p.ho;
    a.n_tiles = p.n_tiles;
    a.G = p.G;
    a.n_groups = p.n_groups;
    a.splits = p.splits;
    a.Ho = p.ho;
    a.Wo = p.wo;
    a.nvb = p.nvb;
    a.T = p.T;
    a.Hi = hi;
    a.kb_total = p.kb_total;
    a.SS = p.SS;
    {
        const char *e = getenv("DP_WG_PF");
        a.pf = e ? atoi(e) : 3;
        if (a.pf < 0) a.pf = 0;
    }
    a.R = p.R;
    a.NM = p.NM;
    a.Ls = p.Ls;
    a.b_bytes = p.b_bytes;
    a.slot_bytes = p.slot_bytes;
    a.box_tx_row = (uint32_t)cin * p.kc * 128u;  // every residue box, real taps only
    a.ring_hi = (uint32_t)p.SS * p.b_bytes;
    a.ring_lo = a.ring_hi + (uint32_t)(p.R + p.NM) * p.slot_bytes;
    a.rs = p.rs;
    a.trace = getenv("DP_WG_TRACE") ? wg_trace_buffer(st) : nullptr;
    a.no_m64 = getenv("DP_WG_NO_M64") ? 1 : 0;
    a.exit_if = flag;
    a.exit_unless = nullptr;
    const size_t smem = (size_t)a.ring_lo + (size_t)(p.R + p.NM) * p.slot_bytes + 1024;
    cudaError_t e = cudaFuncSetAttribute(tc_wgrad_ss_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tc_wgrad_ss: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    const int grid = p.n_groups * p.splits;
    tc_wgrad_ss_kernel<<<grid, WS_THREADS, smem, st>>>(mx[0], mx[1], mx[2], mx[3], mdy, mdyl, a);
    rc = check_launch("tc_wgrad_ss_kernel (fp16)");
    if (rc) return rc;
    const long long total = (long long)k * p.Ls * p.NB + cout;
    ws_reduce<<<ceil_div(total, 32), 32 * WR_GROUPS, 0, st>>>(a.part, a.pdb, dw, db, cout, cin, k, p.Ls,
                                                    p.Npad, p.J, p.kc, p.splits, p.n_tiles * 128,
                                                    p.rs, flag, nullptr, p.ilv);
    rc = check_launch("ws_reduce");
    if (rc) return rc;
    // the tf32 fallback, every launch gated on the flag
    return ws_conv_backward_kernel(x, dy, dw, db, n, cin, hi, wi, cout, k, d,
                                   w8 + p.total_bytes + 256, q.total_bytes, st, 3, x_slack,
                                   dy_pitch, flag);
}

}  // namespace dp
