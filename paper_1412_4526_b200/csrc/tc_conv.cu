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
// Data flow per CTA (persistent, one per SM, 13 warps):
//   warps 0-7  producers, 2 groups x 4 warps: gather the A tiles of one K-step for all
//              MT M tiles straight from the NCHW map (lane = output column -> coalesced
//              128 B row segments; warp q of a group = pixel row q of every M tile =
//              TMEM lane quarter q), split hi/lo in registers and write both into a
//              TMEM stage with tcgen05.st.  Loads of the group's next K-step are issued
//              before it waits for a free stage (register double buffering).  A never
//              touches shared memory: SMEM-operand MMAs are SMEM-bandwidth bound
//              (~128 B/cycle, tools/tc_probe.cu) while A-in-TMEM MMAs run at the
//              tcgen05 floor (tools/tc_probe_ts.cu).
//   warp 12    loads all packed weights (B, K-major, hi and lo) into shared memory
//              once with bulk async copies (TMA engine), allocates TMEM, then issues
//              the MMAs (one elected lane), one stage = one K-step = MT M tiles:
//              A_hi x [B_hi|B_lo] (N = 2*Npad) + A_lo x B_hi   (Npad <= 16), or
//              A_hi x B_hi + A_hi x B_lo + A_lo x B_hi          (Npad >= 32),
//              and releases the stage with one tcgen05.commit.
//   warps 8-11 epilogue: tcgen05.ld the accumulators (double-buffered in TMEM so the
//              next tile's MMAs overlap), add bias + nonlinearity (forward) or apply
//              the upstream nonlinearity's derivative (data gradient), store NCHW.
// Synchronisation is per K-step (not per M tile): one mbarrier wait and one commit
// amortised over MT*(2..3) MMAs -- the per-item barrier round trip (~100-400 cycles)
// otherwise dominates the ~50-cycle MMA work of a skinny-N item.
#include <stdlib.h>

#include "dp_common.cuh"
#include "tc_ptx.cuh"

namespace dp {

constexpr int TC_MAX_STAGES = 16;
constexpr int TC_GROUPS = 2;          // producer groups of 4 warps (one per TMEM lane quarter)
constexpr int TC_MAX_MT = 4;          // M tiles per CTA tile
// Warp roles, ordered by scheduling priority (the SM arbiter favours the highest warp
// id): epilogue warps 0-3 (they mostly wait a whole tile), producers 4..4+4*GROUPS-1,
// the MMA issuer last.  Role warp % 4 == TMEM lane quarter for epilogue and producers.
constexpr int TC_EPI_WARP0 = 0;
constexpr int TC_PROD_WARP0 = 4;
constexpr int TC_PROD_WARPS = 4 * TC_GROUPS;
constexpr int TC_MMA_WARP = TC_PROD_WARP0 + TC_PROD_WARPS;
constexpr int TC_THREADS = (TC_MMA_WARP + 1) * 32;
constexpr int TC_MIN_STAGES = 2 * TC_GROUPS;  // each group keeps 2 K-steps in flight
static_assert(TC_PROD_WARP0 % 4 == 0, "producer warps must start on a lane-quarter boundary");
constexpr int TC_MAX_SMEM = 200 * 1024;

struct TcConvArgs {
    const float *in;     // (n, R, Hin, Win)
    const float *wpack;  // [n_ks][hi|lo][Npad x 8] K-major core-matrix layout
    const float *bias;   // (Q) for forward, nullptr for the data gradient
    float *out;          // (n, Q, Ho, Wo)
    const float *gate;   // (n, Q, Ho, Wo) nonlinearity output, or nullptr
    int R, Hin, Win, Q, Ho, Wo, l, d, pad, act, gate_kind;
    int n_rc, n_ks, Npad, MT, acc_cols, stages, tiles_x, tiles_y, total_tiles;
    uint32_t wbytes;
#ifdef DP_TC_TRACE
    unsigned long long *trace;  // per K-step timestamps of CTA 0 (tools/tc_trace.cu)
    int dbg;                    // 1: no loads, 2: no MMAs, 4: no TMEM stores
#endif
};

#ifdef DP_TC_TRACE
#define TC_TRACE(A, KS, SLOT, COND)                                               \
    do {                                                                          \
        if ((COND) && blockIdx.x == 0 && (KS) < 512) (A).trace[(KS) * 8 + (SLOT)] = clock64(); \
    } while (0)
#define TC_DBG(A, BIT) (((A).dbg & (BIT)) != 0)
#else
#define TC_TRACE(A, KS, SLOT, COND) do {} while (0)
#define TC_DBG(A, BIT) false
#endif

// --------------------------------------------------------------------------------
// weight packing: W(q, r, i, j) -> per K-step ks = (rc*l + i)*l + j two Npad x 8 tiles
// (hi = raw, lo = residual) in the K-major no-swizzle core-matrix layout:
// element (n, k) at byte (n>>3)*256 + (k>>2)*128 + (n&7)*16 + (k&3)*4.
// --------------------------------------------------------------------------------
__global__ void tc_pack_weights(const float *__restrict__ w, float *__restrict__ wp, int Q, int R,
                                int l, int Npad, int n_rc, int n_ks, int bwd) {
    int total = n_ks * 2 * Npad * 8;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += gridDim.x * blockDim.x) {
        int k = idx & 7;
        int n = (idx >> 3) % Npad;
        int hl = (idx / (8 * Npad)) & 1;
        int ks = idx / (16 * Npad);
        int j = ks % l, i = (ks / l) % l, rc = ks / (l * l);
        int c = rc * 8 + k;
        float v = 0.f;
        if (n < Q && c < R) {
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

// Epilogue nonlinearity of the fast tier: single-precision tanhf (<= 2 ulp) kept out of
// line.  The exact tier's fp64-evaluated tanh unrolled over 16 outputs bloats the kernel
// past the instruction cache and starves the producer / MMA warps (measured).
__device__ __noinline__ float tc_act(float v, int kind) {
    if (kind == DP_TANH || kind == DP_TANH_FAST) return tanhf(v);
    if (kind == DP_RELU) return dp_relu(v);
    return v;
}

// One producer warp's view: gathers A tiles (8 channels x 32 columns of one pixel row
// per M tile) from the NCHW map and commits them to TMEM stages.
//
// Every field is a register copy: addressing the kernel's parameter struct through a
// pointer turns each field read into a slow generic load (measured ~3000 cycles per
// K-step with tools/tc_trace.cu before this was fixed).  K-steps are decoded
// incrementally: group p walks KS = p, p + TC_GROUPS, ... so (tile, rc, i, j) advance
// by a fixed stride without integer division.
struct TcProducer {
    const float *in;
    int q, lane, MT, stages, total_ks;
    int n_ks, l, d, pad, Hin, Win, R, tiles_x, per_img;
    uint32_t lane_off, a_base;
    long long plane;
    // cursor of the next K-step this warp loads
    int cur_ks, cur_tile, cur_rc, cur_i, cur_j, cur_KS;
#ifdef DP_TC_TRACE
    unsigned long long *trace;
    int dbg;
#endif

    __device__ __forceinline__ void init(const TcConvArgs &args, int q_, int grp, int lane_,
                                         uint32_t a_base_, int per_img_) {
        in = args.in;
        q = q_;
        lane = lane_;
        a_base = a_base_;
        per_img = per_img_;
        MT = args.MT;
        stages = args.stages;
        n_ks = args.n_ks;
        l = args.l;
        d = args.d;
        pad = args.pad;
        Hin = args.Hin;
        Win = args.Win;
        R = args.R;
        tiles_x = args.tiles_x;
        lane_off = (uint32_t)(q * 32) << 16;
        plane = (long long)Hin * Win;
        const int my_tiles =
            (args.total_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
        total_ks = my_tiles * n_ks;
#ifdef DP_TC_TRACE
        trace = args.trace;
        dbg = args.dbg;
#endif
        // cursor at KS = grp
        cur_KS = grp;
        cur_tile = grp / n_ks;
        cur_ks = grp - cur_tile * n_ks;
        decode_ks();
    }

    __device__ __forceinline__ void decode_ks() {
        const int ll = l * l;
        cur_rc = cur_ks / ll;
        const int tap = cur_ks - cur_rc * ll;
        cur_i = tap / l;
        cur_j = tap - cur_i * l;
    }

    // advance the cursor by TC_GROUPS K-steps (cheap: carries only)
    __device__ __forceinline__ void advance() {
        cur_KS += TC_GROUPS;
        cur_ks += TC_GROUPS;
        if (cur_ks >= n_ks) {
            cur_ks -= n_ks;
            ++cur_tile;
            decode_ks();
            return;
        }
        cur_j += TC_GROUPS;
        while (cur_j >= l) {
            cur_j -= l;
            if (++cur_i == l) {
                cur_i = 0;
                ++cur_rc;
            }
        }
    }

    // load the A tiles of the cursor's K-step into v, then advance the cursor.
    // Instruction-lean: the producers' issue rate, not memory, bounds this kernel
    // (~1000 warp-instructions per K-step budget for ~235 tensor-core cycles), so the
    // 32 loads share one 64-bit base, advance by 32-bit channel strides and use
    // per-load predicates only.
    __device__ __forceinline__ void load(float (&v)[TC_MAX_MT][8]) {
        const bool live = cur_KS < total_ks;
        const int tile = blockIdx.x + cur_tile * gridDim.x;
        const int img = tile / per_img;
        const int rem = tile - img * per_img;
        const int ty = rem / tiles_x;
        const int u0 = ty * 4 * MT, v0 = (rem - ty * tiles_x) * 32;
        const int row0 = u0 + q + cur_i * d - pad;
        const int col = v0 + lane + cur_j * d - pad;
        const bool col_ok = live && col >= 0 && col < Win && !TC_DBG(*this, 1);
        const int c0 = cur_rc * 8;
        const int kmax = R - c0;  // channels of this chunk that exist (>= 1)
        const uint32_t pl = (uint32_t)plane;
        const float *base = in + ((long long)img * R + c0) * plane;
        uint32_t off = (uint32_t)(row0 * Win + col);
#pragma unroll
        for (int mt = 0; mt < TC_MAX_MT; ++mt, off += 4u * (uint32_t)Win) {
            const int row = row0 + 4 * mt;
            const bool ok = mt < MT && col_ok && row >= 0 && row < Hin;
            uint32_t o = off;
#pragma unroll
            for (int k = 0; k < 8; ++k, o += pl) {
                float t = 0.f;
                if (ok && k < kmax) t = __ldg(base + o);
                v[mt][k] = t;
            }
        }
        advance();
    }

    // K-step KS -> stage KS % stages: wait until the MMAs of K-step KS - stages finished,
    // write hi/lo of every M tile, then one arrive (per warp) on the stage's full barrier.
    __device__ __forceinline__ void commit(const float (&v)[TC_MAX_MT][8], int KS,
                                           uint64_t *empty_bar, uint64_t *full_bar) const {
        const int stage = KS % stages;
        const uint32_t phase = (uint32_t)((KS / stages) & 1);
        TC_TRACE(*this, KS, 0, lane == 0 && q == 0);
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        TC_TRACE(*this, KS, 1, lane == 0 && q == 0);
        ptx::tc_fence_after();
        const uint32_t sbase = a_base + lane_off + (uint32_t)(stage * MT * 16);
#pragma unroll
        for (int mt = 0; mt < TC_MAX_MT; ++mt) {
            if (mt >= MT) break;
            float lo[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) lo[k] = ptx::tf32_lo(v[mt][k]);
            if (!TC_DBG(*this, 4)) {
                ptx::tmem_st8(sbase + mt * 16, v[mt]);
                ptx::tmem_st8(sbase + mt * 16 + 8, lo);
            }
        }
        ptx::tmem_wait_st();
        TC_TRACE(*this, KS, 2, lane == 0 && q == 0);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&full_bar[stage]);
    }
};

template <bool STACKED, bool BWD>
__global__ void __launch_bounds__(TC_THREADS, 1) tc_conv_kernel(const TcConvArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *wsm = smem_raw;  // packed weights
    __shared__ uint64_t full_bar[TC_MAX_STAGES], empty_bar[TC_MAX_STAGES];
    __shared__ uint64_t tfull_bar[2], tempty_bar[2], w_bar;
    __shared__ uint32_t s_tmem;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int MT = a.MT;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            ptx::mbar_init(&full_bar[s], 4);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull_bar[b], 1);
            ptx::mbar_init(&tempty_bar[b], 4);
        }
        ptx::mbar_init(&w_bar, 1);
        ptx::mbar_fence_init();
    }
    if (warp == TC_MMA_WARP) ptx::tmem_alloc<512>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;
    // TMEM columns: [0, 2*MT*acc_cols) accumulators (2 tile buffers), then the A stages
    const uint32_t a_base = tmem + (uint32_t)(2 * MT * a.acc_cols);
    const int per_img = a.tiles_x * a.tiles_y;

    if (warp >= TC_PROD_WARP0 && warp < TC_PROD_WARP0 + TC_PROD_WARPS) {
        // ============================ producers ============================
        // K-steps are numbered per CTA in MMA order, KS = tile_seq * n_ks + ks; group p
        // produces KS = p, p + TC_GROUPS, ...  Striding the CTA-global KS keeps each
        // group's stage waits one parity round deep (unambiguous) and, with
        // stages >= 2 * TC_GROUPS, deadlock-free.
        TcProducer pr;
        const int grp = (warp - TC_PROD_WARP0) >> 2;
        pr.init(a, warp & 3, grp, lane, a_base, per_img);
        float va[TC_MAX_MT][8], vb[TC_MAX_MT][8];
        pr.load(va);  // K-step grp
        pr.load(vb);  // K-step grp + TC_GROUPS
        for (int KS = grp; KS < pr.total_ks; KS += 2 * TC_GROUPS) {
            pr.commit(va, KS, empty_bar, full_bar);
            TC_TRACE(a, KS, 6, lane == 0 && (warp & 3) == 0);
            pr.load(va);  // K-step KS + 2 * TC_GROUPS
            TC_TRACE(a, KS, 7, lane == 0 && (warp & 3) == 0);
            if (KS + TC_GROUPS >= pr.total_ks) break;
            pr.commit(vb, KS + TC_GROUPS, empty_bar, full_bar);
            pr.load(vb);  // K-step KS + 3 * TC_GROUPS
        }
    } else if (warp == TC_MMA_WARP) {
        // ============================ weights + MMA issuer ============================
        if (ptx::elect_one()) {
            ptx::mbar_expect_tx(&w_bar, a.wbytes);
            const unsigned char *src = reinterpret_cast<const unsigned char *>(a.wpack);
            for (uint32_t off = 0; off < a.wbytes; off += 32768u) {
                uint32_t n = a.wbytes - off < 32768u ? a.wbytes - off : 32768u;
                ptx::bulk_g2s(wsm + off, src + off, n, &w_bar);
            }
        }
        __syncwarp();
        ptx::mbar_wait(&w_bar, 0);
        const uint32_t wsm_addr = ptx::smem_u32(wsm);
        const uint32_t ks_bytes = (uint32_t)a.Npad * 64;  // hi + lo tiles
        const uint32_t idesc_n = ptx::idesc_tf32(128, a.Npad);
        const uint32_t idesc_2n = ptx::idesc_tf32(128, 2 * a.Npad);
        int stage = 0, buf = 0;
        uint32_t phase = 0, tphase = 0;
        int tseq_mma = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x, ++tseq_mma) {
            ptx::mbar_wait(&tempty_bar[buf], tphase ^ 1);
            ptx::tc_fence_after();
            const uint32_t dbase = tmem + (uint32_t)(buf * MT * a.acc_cols);
            for (int ks = 0; ks < a.n_ks; ++ks) {
                const uint32_t bhi = wsm_addr + (uint32_t)ks * ks_bytes;
                const uint64_t dhi = ptx::smem_desc(bhi, 128, 256);
                const uint64_t dlo = ptx::smem_desc(bhi + (uint32_t)a.Npad * 32, 128, 256);
                const uint32_t sbase = a_base + (uint32_t)(stage * MT * 16);
                const uint32_t acc = ks > 0;
                const int KSg = tseq_mma * a.n_ks + ks;
                TC_TRACE(a, KSg, 3, lane == 0);
                ptx::mbar_wait(&full_bar[stage], phase);
                TC_TRACE(a, KSg, 4, lane == 0);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    for (int mt = 0; mt < (TC_DBG(a, 2) ? 0 : MT); ++mt) {
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
                }
                TC_TRACE(a, KSg, 5, lane == 0);
                __syncwarp();
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
        const int q = warp & 3;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        int buf = 0;
        uint32_t tphase = 0;
        for (int tile = blockIdx.x; tile < a.total_tiles; tile += gridDim.x) {
            const int img = tile / per_img;
            const int rem = tile - img * per_img;
            const int u0 = (rem / a.tiles_x) * 4 * MT, v0 = (rem % a.tiles_x) * 32;
            const int col = v0 + lane;
            ptx::mbar_wait_sleep(&tfull_bar[buf], tphase);
            ptx::tc_fence_after();
            float *out_img = a.out + (long long)img * a.Q * a.Ho * a.Wo;
            const float *gate_img =
                a.gate ? a.gate + (long long)img * a.Q * a.Ho * a.Wo : nullptr;
            for (int mt = 0; mt < MT; ++mt) {
                const int row = u0 + 4 * mt + q;
                const bool inside = row < a.Ho && col < a.Wo;
                const uint32_t dcol = tmem + lane_off + (uint32_t)((buf * MT + mt) * a.acc_cols);
                for (int o0 = 0; o0 < a.Npad; o0 += 16) {
                    uint32_t r[16], r2[16];
                    ptx::tmem_ld16(dcol + o0, r);
                    if (STACKED) ptx::tmem_ld16(dcol + a.Npad + o0, r2);
                    ptx::tmem_wait_ld();
                    if (!inside) continue;
#pragma unroll
                    for (int t = 0; t < 16; ++t) {
                        const int o = o0 + t;
                        if (o >= a.Q) break;
                        float val = __uint_as_float(r[t]);
                        if (STACKED) val += __uint_as_float(r2[t]);
                        const long long off = ((long long)o * a.Ho + row) * a.Wo + col;
                        if (!BWD) {
                            val = tc_act(val + a.bias[o], a.act);
                        } else if (gate_img) {
                            val = gate_from_output(val, gate_img[off], a.gate_kind);
                        }
                        out_img[off] = val;
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
    int Npad, n_rc, n_ks, MT, acc_cols, stages;
    bool stacked;
    size_t wbytes;
};

// TMEM budget (512 columns): 2 * MT * acc_cols accumulator columns + stages * MT * 16
// A columns, with stages >= TC_MIN_STAGES.  DP_TC_MT overrides the M tiles per CTA tile.
static TcPlan tc_plan(int R, int Q, int l) {
    TcPlan p;
    p.Npad = (Q + 15) / 16 * 16;
    p.n_rc = (R + 7) / 8;
    p.n_ks = p.n_rc * l * l;
    p.stacked = p.Npad <= 16;
    p.acc_cols = p.stacked ? 2 * p.Npad : p.Npad;
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
        if (acc_total < 512 && st >= TC_MIN_STAGES) {
            p.MT = mt;
            p.stages = st;
            break;
        }
    }
    p.wbytes = (size_t)p.n_ks * p.Npad * 64;
    return p;
}

size_t tc_conv_workspace(int R, int Q, int l) { return tc_plan(R, Q, l).wbytes; }

bool tc_conv_supported(int R, int Q, int l) {
    TcPlan p = tc_plan(R, Q, l);
    return p.Npad <= 128 && p.MT >= 1 && p.wbytes <= (size_t)TC_MAX_SMEM;
}

static int g_num_sms = 0;

static int launch_tc(const float *in, const float *w, const float *bias, float *out,
                     const float *gate, int n, int R, int Hin, int Win, int Q, int Ho, int Wo,
                     int l, int d, int pad, int act, int gate_kind, bool bwd, void *ws,
                     size_t ws_bytes, cudaStream_t st) {
    TcPlan p = tc_plan(R, Q, l);
    if (!tc_conv_supported(R, Q, l))
        return set_error(DP_ERR_UNSUPPORTED,
                         "tensor-core conv: weights need %zu B of shared memory (R=%d Q=%d k=%d)",
                         p.wbytes, R, Q, l);
    if (ws == nullptr || ws_bytes < p.wbytes)
        return set_error(DP_ERR_ARG, "tensor-core conv: workspace %zu < %zu bytes", ws_bytes,
                         p.wbytes);
    if (((uintptr_t)ws & 15) != 0)
        return set_error(DP_ERR_ARG, "tensor-core conv: workspace must be 16-byte aligned");
    float *wp = (float *)ws;
    int total = p.n_ks * 2 * p.Npad * 8;
    tc_pack_weights<<<ceil_div(total, 256), 256, 0, st>>>(w, wp, Q, R, l, p.Npad, p.n_rc, p.n_ks,
                                                          bwd ? 1 : 0);
    int rc = check_launch("tc_pack_weights");
    if (rc) return rc;
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
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
    // fewer M tiles per CTA tile when the image is short (less padding waste); the
    // stage count is kept (fewer A columns per stage only loosens the TMEM budget)
    int rows_needed = (Ho + 3) / 4;
    if (a.MT > rows_needed) a.MT = rows_needed;
    a.acc_cols = p.acc_cols;
    a.tiles_x = ceil_div(Wo, 32);
    a.tiles_y = ceil_div(Ho, 4 * a.MT);
    long long tt = (long long)n * a.tiles_x * a.tiles_y;
    if (tt > 0x7fffffff) return set_error(DP_ERR_UNSUPPORTED, "tensor-core conv: too many tiles");
    a.total_tiles = (int)tt;
    a.wbytes = (uint32_t)p.wbytes;
    int grid = a.total_tiles < g_num_sms ? a.total_tiles : g_num_sms;
    size_t smem = p.wbytes;
    void (*kern)(const TcConvArgs);
    if (p.stacked)
        kern = bwd ? tc_conv_kernel<true, true> : tc_conv_kernel<true, false>;
    else
        kern = bwd ? tc_conv_kernel<false, true> : tc_conv_kernel<false, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
        return set_error(DP_ERR_CUDA, "tc_conv: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    kern<<<grid, TC_THREADS, smem, st>>>(a);
    return check_launch("tc_conv_kernel");
}

int tc_conv_forward(const float *x, const float *w, const float *b, float *y, int n, int cin,
                    int h, int wd, int cout, int k, int d, int act, void *ws, size_t ws_bytes,
                    cudaStream_t st) {
    int e = (k - 1) * d + 1;
    return launch_tc(x, w, b, y, nullptr, n, cin, h, wd, cout, h - e + 1, wd - e + 1, k, d, 0, act,
                     0, false, ws, ws_bytes, st);
}

int tc_conv_backward_data(const float *dy, const float *w, float *dx, int n, int cout, int ho,
                          int wo, int cin, int k, int d, const float *gate, int gate_kind,
                          void *ws, size_t ws_bytes, cudaStream_t st) {
    int e = (k - 1) * d + 1;
    return launch_tc(dy, w, nullptr, dx, gate, n, cout, ho, wo, cin, ho + e - 1, wo + e - 1, k, d,
                     e - 1, 0, gate_kind, true, ws, ws_bytes, st);
}

}  // namespace dp
