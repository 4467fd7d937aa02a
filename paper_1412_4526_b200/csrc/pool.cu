// d-regularly sparse max / average pooling, forward and backward (sm_100a).
//
// HBM-bound kernels; one thread per output (forward) or per input pixel
// (backward), consecutive threads on consecutive columns so every tap read is
// a coalesced row segment (shifted taps hit L1/L2).  Planes x pixels grid, no
// 64-bit divides (the first version's per-thread 64-bit index math made these
// kernels instruction bound at ~1 TB/s).  Results are bit-identical
// to the compiled reference backend:
//  * maxpool_forward  (_kernels.pyx:133-166): best = -inf, strict '>' scanning
//    taps row-major, so the first tap wins ties and NaN never wins; argmax
//    i*p + j.  Fused epilogue: the following nonlinearity.
//  * maxpool_backward (_kernels.pyx:169-191): the reference scatters dy in
//    row-major (u, v) order, i.e. each input pixel receives its contributions
//    in DESCENDING tap order; this kernel gathers them in exactly that order
//    (atomic-free, deterministic).  Fused epilogue: the upstream
//    nonlinearity's derivative (gate).
//  * avgpool_forward  (_kernels.pyx:194-221): acc = 0, += taps row-major, / p^2.
//  * avgpool_backward (_kernels.pyx:224-247): q = dy / p^2 gathered in
//    descending tap order.
#include <stdlib.h>

#include "dp_common.cuh"

namespace dp {

// Indexing: grid.y (and grid.z for more than 65535 planes) = plane n*C + c, grid.x covers
// the plane's Ho*Wo (or Hi*Wi) pixels; one 32-bit divide per thread gives (row, column).
// Consecutive threads are consecutive columns, so every tap read and every store is a
// coalesced row segment; a pixel's p^2 taps are re-read by neighbouring threads / rows
// from L1/L2, so DRAM sees each map about once (HBM-bound by construction).
__device__ __forceinline__ long long pool_plane() {
    return (long long)blockIdx.z * gridDim.y + blockIdx.y;
}

// Max pool: 2-D tiles, block (32, 8), each thread 4 columns 32 apart (warp accesses stay
// 128-byte row segments) so the index math and the plane/row bases are paid once per 4
// outputs -- the one-output-per-thread version was issue bound at ~1.7 TB/s.
constexpr int PT_X = 32, PT_Y = 8, PT_V = 4, PT_R = 8;  // tile: 128 columns x 64 rows

template <typename T, typename A, int P>
__global__ void __launch_bounds__(PT_X * PT_Y)
    maxpool_fwd_tile(const T *__restrict__ x, T *__restrict__ y, A *__restrict__ arg, int H,
                     int W, int Ho, int Wo, int p_rt, int d, int act, long long planes) {
    const int u0 = blockIdx.y * (PT_Y * PT_R) + threadIdx.y;
    if (u0 >= Ho) return;
    const int v0 = blockIdx.x * (PT_X * PT_V) + threadIdx.x;
    for (long long plane = blockIdx.z; plane < planes; plane += gridDim.z) {
        const T *src = x + (plane * H + u0) * (long long)W;
        T *yr = y + (plane * Ho + u0) * (long long)Wo;
        A *ar = arg + (plane * Ho + u0) * (long long)Wo;
        if (P == 2) {
            // four tap base pointers formed once and advanced PT_Y rows per step; every
            // load / store is base + immediate (per-tap index math made this ALU bound)
            const T *t0 = src + v0, *t1 = t0 + d, *t2 = t0 + d * W, *t3 = t2 + d;
            T *yo = yr + v0;
            A *ao = ar + v0;
            const long long xs = (long long)PT_Y * W, ys = (long long)PT_Y * Wo;
            int nk = 0;  // columns of this thread inside the map
#pragma unroll
            for (int k = 0; k < PT_V; ++k) nk += v0 + k * PT_X < Wo;
            for (int ry = 0; ry < PT_R; ++ry) {
                if (u0 + ry * PT_Y >= Ho) break;
                T t[PT_V][4];
#pragma unroll
                for (int k = 0; k < PT_V; ++k) {
                    if (k < nk) {
                        t[k][0] = __ldg(t0 + k * PT_X);
                        t[k][1] = __ldg(t1 + k * PT_X);
                        t[k][2] = __ldg(t2 + k * PT_X);
                        t[k][3] = __ldg(t3 + k * PT_X);
                    } else {
                        t[k][0] = t[k][1] = t[k][2] = t[k][3] = T(0);
                    }
                }
#pragma unroll
                for (int k = 0; k < PT_V; ++k) {
                    if (k >= nk) break;
                    T best = neg_inf<T>();
                    int bk = 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (t[k][q] > best) {
                            best = t[k][q];
                            bk = q;
                        }
                    yo[k * PT_X] = apply_nonlin(best, act);
                    ao[k * PT_X] = (A)bk;
                }
                t0 += xs;
                t1 += xs;
                t2 += xs;
                t3 += xs;
                yo += ys;
                ao += ys;
            }
        } else {
            const int p = p_rt;
            for (int ry = 0; ry < PT_R; ++ry) {
                const int u = u0 + ry * PT_Y;
                if (u >= Ho) break;
                const long long ro = (long long)ry * PT_Y;
                for (int k = 0; k < PT_V; ++k) {
                    const int v = v0 + k * PT_X;
                    if (v >= Wo) break;
                    const T *s0 = src + ro * W + v;
                    T best = neg_inf<T>();
                    int bk = 0;
                    for (int i = 0; i < p; ++i) {
                        const T *row = s0 + (long long)i * d * W;
                        for (int j = 0; j < p; ++j) {
                            const T xv = __ldg(row + j * d);
                            if (xv > best) {
                                best = xv;
                                bk = i * p + j;
                            }
                        }
                    }
                    yr[ro * Wo + v] = apply_nonlin(best, act);
                    ar[ro * Wo + v] = (A)bk;
                }
            }
        }
    }
}

constexpr int PB_V = 2;  // backward: 2 pixels per thread (PB_V = 4 measured slower)

template <typename T, typename A, int P>
__global__ void __launch_bounds__(PT_X * PT_Y)
    maxpool_bwd_tile(const T *__restrict__ dy, const A *__restrict__ arg, T *__restrict__ dx,
                     const T *__restrict__ gate, int Ho, int Wo, int Hi, int Wi, int p_rt, int d,
                     int gate_kind, long long planes, int Wd) {
    // Wd: dx row pitch (>= Wi; the gate keeps pitch Wi)
    const int r0 = blockIdx.y * (PT_Y * PT_R) + threadIdx.y;
    if (r0 >= Hi) return;
    const int s0 = blockIdx.x * (PT_X * PB_V) + threadIdx.x;
    for (long long plane = blockIdx.z; plane < planes; plane += gridDim.z) {
        const T *dyp = dy + plane * Ho * (long long)Wo;
        const A *ap = arg + plane * Ho * (long long)Wo;
        if (P == 2) {
            // candidate windows of input pixel (r, s): taps 3, 2, 1, 0 = outputs (r-d, s-d),
            // (r-d, s), (r, s-d), (r, s) -- the reference's scatter (row-major (u, v)) order.
            // Column checks hoisted out of the row loop; base pointers advance PT_Y rows per
            // step and are only dereferenced in range.
            bool cv1[PB_V], cv0[PB_V];
#pragma unroll
            for (int k = 0; k < PB_V; ++k) {
                const int s = s0 + k * PT_X;
                cv1[k] = s - d >= 0 && s - d < Wo;
                cv0[k] = s < Wo;
            }
            long long o1 = (long long)(r0 - d) * Wo + s0, o0 = (long long)r0 * Wo + s0;
            long long q = (plane * Hi + r0) * (long long)Wi + s0;
            long long qd = (plane * Hi + r0) * (long long)Wd + s0;
            const long long os = (long long)PT_Y * Wo, qs = (long long)PT_Y * Wi,
                            qds = (long long)PT_Y * Wd;
            for (int ry = 0; ry < PT_R; ++ry) {
                const int r = r0 + ry * PT_Y;
                if (r >= Hi) break;
                const bool u1 = r - d >= 0 && r - d < Ho, u0 = r < Ho;
                const A *a_[4] = {ap + o1 - d, ap + o1, ap + o0 - d, ap + o0};
                const T *d_[4] = {dyp + o1 - d, dyp + o1, dyp + o0 - d, dyp + o0};
                int av[PB_V][4];
                T dv[PB_V][4];
#pragma unroll
                for (int k = 0; k < PB_V; ++k) {
                    const bool ok[4] = {u1 && cv1[k], u1 && cv0[k], u0 && cv1[k], u0 && cv0[k]};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        av[k][c] = ok[c] ? (int)__ldg(a_[c] + k * PT_X) : -1;
                        dv[k][c] = ok[c] ? __ldg(d_[c] + k * PT_X) : T(0);
                    }
                }
                T *dxo = dx + qd;
                const T *go = gate ? gate + q : nullptr;
#pragma unroll
                for (int k = 0; k < PB_V; ++k) {
                    if (s0 + k * PT_X >= Wi) break;
                    T acc = T(0);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (av[k][c] == 3 - c) acc = add_rn(acc, dv[k][c]);
                    if (go) acc = gate_from_output(acc, go[k * PT_X], gate_kind);
                    dxo[k * PT_X] = acc;
                }
                o1 += os;
                o0 += os;
                q += qs;
                qd += qds;
            }
        } else {
            const int p = p_rt;
            for (int ry = 0; ry < PT_R; ++ry) {
                const int r = r0 + ry * PT_Y;
                if (r >= Hi) break;
                const long long q0 = (plane * Hi + r) * (long long)Wi;
                const long long qd0 = (plane * Hi + r) * (long long)Wd;
                for (int k = 0; k < PB_V; ++k) {
                    const int s = s0 + k * PT_X;
                    if (s >= Wi) break;
                    T acc = T(0);
                    for (int i = p - 1; i >= 0; --i) {
                        const int u = r - i * d;
                        if (u < 0 || u >= Ho) continue;
                        const A *arow = ap + (long long)u * Wo;
                        const T *drow = dyp + (long long)u * Wo;
                        for (int j = p - 1; j >= 0; --j) {
                            const int v = s - j * d;
                            if (v < 0 || v >= Wo) continue;
                            if ((int)__ldg(arow + v) == i * p + j) acc = add_rn(acc, __ldg(drow + v));
                        }
                    }
                    if (gate) acc = gate_from_output(acc, gate[q0 + s], gate_kind);
                    dx[qd0 + s] = acc;
                }
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) avgpool_fwd_kernel(const T *__restrict__ x,
                                                          T *__restrict__ y, int H, int W, int Ho,
                                                          int Wo, int p, int d, int act, long long planes) {
    const int pix = blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= Ho * Wo) return;
    const long long plane = pool_plane();
    if (plane >= planes) return;
    const int u = pix / Wo, v = pix - u * Wo;
    const T *src = x + plane * H * W + (long long)u * W + v;
    T acc = T(0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) acc = add_rn(acc, __ldg(src + (long long)i * d * W + j * d));
    y[plane * Ho * Wo + pix] = apply_nonlin(div_rn(acc, T(p * p)), act);
}

template <typename T>
__global__ void __launch_bounds__(256) avgpool_bwd_kernel(const T *__restrict__ dy,
                                                          T *__restrict__ dx,
                                                          const T *__restrict__ gate, int Ho,
                                                          int Wo, int Hi, int Wi, int p, int d,
                                                          int gate_kind, long long planes) {
    const int pix = blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= Hi * Wi) return;
    const long long plane = pool_plane();
    if (plane >= planes) return;
    const int r = pix / Wi, s = pix - r * Wi;
    const T *dyp = dy + plane * Ho * Wo;
    const T pp = T(p * p);
    T acc = T(0);
    for (int i = p - 1; i >= 0; --i) {
        const int u = r - i * d;
        if (u < 0 || u >= Ho) continue;
        for (int j = p - 1; j >= 0; --j) {
            const int v = s - j * d;
            if (v < 0 || v >= Wo) continue;
            acc = add_rn(acc, div_rn(__ldg(dyp + u * Wo + v), pp));
        }
    }
    const long long q = plane * Hi * Wi + pix;
    if (gate) acc = gate_from_output(acc, gate[q], gate_kind);
    dx[q] = acc;
}


// ---------------------------------------------------------------------------------------
// Shared-memory tiled kernels (p <= 8, halo (p-1)*d <= SP_MAX_HALO): the default path.
//
// A CTA owns one tile position of the (h, w) plane and walks planes blockIdx.z, +gridDim.z,
// ...  The staged region is 8*NR rows x 128 columns (4 columns per lane, NR rows per warp);
// the next plane's region is fetched into registers while the current plane is computed
// from shared memory, so loads stay in flight across the compute phase.  Every input
// element crosses HBM about once (the (p-1)*d halo overlap of neighbouring tiles is L2).
//
//  * max forward is SEPARABLE: row pass hm[r][v] = max_j x[r][v + j*d] (first j on ties,
//    strict '>'), then column pass y[u][v] = max_i hm[u + i*d][v] (first i).  The element
//    picked is the row-major-first maximum of the window, exactly the reference's scan
//    (_kernels.pyx:155-163: best = -inf, strict '>'; a NaN never wins, an all-NaN window
//    gives -inf / arg 0 in both), so values and argmax i*p + j are bit-identical -- with
//    2p instead of p^2 compares per output (p = 8: 16 vs 64).  The row pass of a row is
//    done by one warp, in place (all reads, __syncwarp, all writes).
//  * max backward gathers, per input pixel, the p^2 candidate outputs from the staged dy /
//    argmax tile in descending tap order (= the reference's row-major scatter order,
//    _kernels.pyx:184-191), so sums of several contributions round identically.
//  * avg forward adds the p^2 taps in row-major order (_kernels.pyx:215-220); avg backward
//    divides the staged dy by p^2 once per output (as the reference does, :242) and
//    gathers it in descending tap order, skipping out-of-map windows.
// ---------------------------------------------------------------------------------------
constexpr int SP_TW = 128;  // output (forward) / input (backward) columns per tile
constexpr int SP_TH = 32;   // output / input rows per tile
constexpr int SP_MAX_HALO = 48;

// dst[r * RW + c] = src[(gy0 + r) * Ws + gx0 + c] for r < RH, c < RW (zero outside the map);
// block (32, 8): lanes walk columns, warps walk rows, two rows of loads in flight per thread.
template <typename T>
__device__ __forceinline__ void sp_stage(T *__restrict__ dst, const T *__restrict__ src, int RH,
                                         int RW, int gy0, int gx0, int Hs, int Ws) {
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < RH; r += 16) {
        T v[2][6];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rr = r + 8 * h, gy = gy0 + rr;
            const bool rok = rr < RH && gy >= 0 && gy < Hs;
            const T *row = src + (long long)(rok ? gy : 0) * Ws;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const int c = tx + 32 * k, gx = gx0 + c;
                v[h][k] = (rok && c < RW && gx >= 0 && gx < Ws) ? __ldg(row + gx) : T(0);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rr = r + 8 * h;
            if (rr >= RH) break;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const int c = tx + 32 * k;
                if (c < RW) dst[rr * RW + c] = v[h][k];
            }
        }
    }
}

// DC > 0: the dilation as a compile-time constant (the d = 1 pool1 layers): the per-tap
// smem offsets become immediates -- ncu showed ~45 % of the d-generic kernel's issued
// instructions were index arithmetic (IMAD / ISETP / LEA), at ~220 per 32 outputs
template <typename T, typename A, int P, int DC>
__global__ void __launch_bounds__(256)
    maxpool_fwd_smem(const T *__restrict__ x, T *__restrict__ y, A *__restrict__ arg, int H,
                     int W, int Ho, int Wo, int d_rt, int act, long long planes) {
    const int d = DC > 0 ? DC : d_rt;
    extern __shared__ __align__(16) unsigned char sp_raw[];
    const int hx = (P - 1) * d, RW = SP_TW + hx, RH = SP_TH + hx;
    T *xs = reinterpret_cast<T *>(sp_raw);
    T *hs = xs + RH * RW;
    uint8_t *hj = reinterpret_cast<uint8_t *>(hs + RH * SP_TW);
    const int u0 = blockIdx.y * SP_TH, v0 = blockIdx.x * SP_TW;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (long long plane = blockIdx.z; plane < planes; plane += gridDim.z) {
        sp_stage(xs, x + plane * H * (long long)W, RH, RW, u0, v0, H, W);
        __syncthreads();
        // row pass
#pragma unroll 1
        for (int r = ty; r < RH; r += 8) {
#pragma unroll
            for (int k = 0; k < SP_TW / 32; ++k) {
                const int v = tx + 32 * k;
                const T *s = xs + r * RW + v;
                T best = neg_inf<T>();
                int bj = 0;
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const T t = s[j * d];
                    if (t > best) {
                        best = t;
                        bj = j;
                    }
                }
                hs[r * SP_TW + v] = best;
                hj[r * SP_TW + v] = (uint8_t)bj;
            }
        }
        __syncthreads();
        // column pass + stores
#pragma unroll 1
        for (int u = ty; u < SP_TH; u += 8) {
            const int gu = u0 + u;
            if (gu >= Ho) break;
            T *yr = y + (plane * Ho + gu) * (long long)Wo;
            A *ar = arg + (plane * Ho + gu) * (long long)Wo;
#pragma unroll
            for (int k = 0; k < SP_TW / 32; ++k) {
                const int v = tx + 32 * k, gv = v0 + v;
                if (gv >= Wo) break;
                T best = neg_inf<T>();
                int bi = 0;
#pragma unroll
                for (int i = 0; i < P; ++i) {
                    const T t = hs[(u + i * d) * SP_TW + v];
                    if (t > best) {
                        best = t;
                        bi = i;
                    }
                }
                yr[gv] = apply_nonlin(best, act);
                ar[gv] = (A)(bi * P + hj[(u + bi * d) * SP_TW + v]);
            }
        }
        __syncthreads();
    }
}

template <typename T, typename A, int P, int DC>
__global__ void __launch_bounds__(256)
    maxpool_bwd_smem(const T *__restrict__ dy, const A *__restrict__ arg, T *__restrict__ dx,
                     const T *__restrict__ gate, int Ho, int Wo, int Hi, int Wi, int d_rt,
                     int gate_kind, long long planes, int Wd) {
    const int d = DC > 0 ? DC : d_rt;
    extern __shared__ __align__(16) unsigned char sp_raw[];
    const int hx = (P - 1) * d, RW = SP_TW + hx, RH = SP_TH + hx;
    T *ds = reinterpret_cast<T *>(sp_raw);
    uint8_t *as = reinterpret_cast<uint8_t *>(ds + RH * RW);
    const int r0 = blockIdx.y * SP_TH, s0 = blockIdx.x * SP_TW;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (long long plane = blockIdx.z; plane < planes; plane += gridDim.z) {
        const long long po = plane * Ho * (long long)Wo;
        // stage dy and the argmax codes of outputs [r0 - hx, r0 + TH) x [s0 - hx, s0 + TW)
        // (code 255 = no window there)
        for (int r = ty; r < RH; r += 16) {
            T v[2][6];
            uint8_t c8[2][6];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr = r + 8 * h, gy = r0 - hx + rr;
                const bool rok = rr < RH && gy >= 0 && gy < Ho;
                const long long ro = po + (long long)(rok ? gy : 0) * Wo;
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const int c = tx + 32 * k, gx = s0 - hx + c;
                    const bool ok = rok && c < RW && gx >= 0 && gx < Wo;
                    v[h][k] = ok ? __ldg(dy + ro + gx) : T(0);
                    c8[h][k] = ok ? (uint8_t)__ldg(arg + ro + gx) : (uint8_t)255;
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr = r + 8 * h;
                if (rr >= RH) break;
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const int c = tx + 32 * k;
                    if (c < RW) {
                        ds[rr * RW + c] = v[h][k];
                        as[rr * RW + c] = c8[h][k];
                    }
                }
            }
        }
        __syncthreads();
#pragma unroll 1
        for (int r = ty; r < SP_TH; r += 8) {
            const int gr = r0 + r;
            if (gr >= Hi) break;
            const long long q = (plane * Hi + gr) * (long long)Wi;
            const long long qd = (plane * Hi + gr) * (long long)Wd;
            T gv[SP_TW / 32];
#pragma unroll
            for (int k = 0; k < SP_TW / 32; ++k) {
                const int gs = s0 + tx + 32 * k;
                gv[k] = (gate && gs < Wi) ? __ldg(gate + q + gs) : T(0);
            }
#pragma unroll
            for (int k = 0; k < SP_TW / 32; ++k) {
                const int s = tx + 32 * k, gs = s0 + s;
                if (gs >= Wi) break;
                T acc = T(0);
#pragma unroll
                for (int i = P - 1; i >= 0; --i) {
                    const int base = (r + hx - i * d) * RW + s + hx;
#pragma unroll
                    for (int j = P - 1; j >= 0; --j)
                        if (as[base - j * d] == i * P + j) acc = add_rn(acc, ds[base - j * d]);
                }
                if (gate) acc = gate_from_output(acc, gv[k], gate_kind);
                dx[qd + gs] = acc;
            }
        }
        __syncthreads();
    }
}

template <typename T, int P>
__global__ void __launch_bounds__(256)
    avgpool_fwd_smem(const T *__restrict__ x, T *__restrict__ y, int H, int W, int Ho, int Wo,
                     int d, int act, long long planes) {
    extern __shared__ __align__(16) unsigned char sp_raw[];
    const int hx = (P - 1) * d, RW = SP_TW + hx, RH = SP_TH + hx;
    T *xs = reinterpret_cast<T *>(sp_raw);
    const int u0 = blockIdx.y * SP_TH, v0 = blockIdx.x * SP_TW;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const T pp = T(P * P);
    for (long long plane = blockIdx.z; plane < planes; plane += gridDim.z) {
        sp_stage(xs, x + plane * H * (long long)W, RH, RW, u0, v0, H, W);
        __syncthreads();
#pragma unroll 1
        for (int u = ty; u < SP_TH; u += 8) {
            const int gu = u0 + u;
            if (gu >= Ho) break;
            T *yr = y + (plane * Ho + gu) * (long long)Wo;
#pragma unroll
            for (int k = 0; k < SP_TW / 32; ++k) {
                const int v = tx + 32 * k, gv = v0 + v;
                if (gv >= Wo) break;
                T acc = T(0);
#pragma unroll
                for (int i = 0; i < P; ++i)
#pragma unroll
                    for (int j = 0; j < P; ++j) acc = add_rn(acc, xs[(u + i * d) * RW + v + j * d]);
                yr[gv] = apply_nonlin(div_rn(acc, pp), act);
            }
        }
        __syncthreads();
    }
}

template <typename T, int P>
__global__ void __launch_bounds__(256)
    avgpool_bwd_smem(const T *__restrict__ dy, T *__restrict__ dx, const T *__restrict__ gate,
                     int Ho, int Wo, int Hi, int Wi, int d, int gate_kind, long long planes) {
    extern __shared__ __align__(16) unsigned char sp_raw[];
    const int hx = (P - 1) * d, RW = SP_TW + hx, RH = SP_TH + hx;
    T *qs = reinterpret_cast<T *>(sp_raw);
    const int r0 = blockIdx.y * SP_TH, s0 = blockIdx.x * SP_TW;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const T pp = T(P * P);
    for (long long plane = blockIdx.z; plane < planes; plane += gridDim.z) {
        sp_stage(qs, dy + plane * Ho * (long long)Wo, RH, RW, r0 - hx, s0 - hx, Ho, Wo);
        __syncthreads();
        for (int e = ty * 32 + tx; e < RH * RW; e += 256) qs[e] = div_rn(qs[e], pp);
        __syncthreads();
#pragma unroll 1
        for (int r = ty; r < SP_TH; r += 8) {
            const int gr = r0 + r;
            if (gr >= Hi) break;
            const long long q = (plane * Hi + gr) * (long long)Wi;
#pragma unroll
            for (int k = 0; k < SP_TW / 32; ++k) {
                const int s = tx + 32 * k, gs = s0 + s;
                if (gs >= Wi) break;
                // out-of-map windows are staged as +0.0: adding them leaves the accumulator's
                // bits unchanged (it starts at +0.0, and round-to-nearest never turns +0.0 + x
                // into -0.0), so every tap is added without a range check
                T acc = T(0);
#pragma unroll
                for (int i = P - 1; i >= 0; --i) {
                    const int base = (r + hx - i * d) * RW + s + hx;
#pragma unroll
                    for (int j = P - 1; j >= 0; --j) acc = add_rn(acc, qs[base - j * d]);
                }
                if (gate) acc = gate_from_output(acc, __ldg(gate + q + gs), gate_kind);
                dx[q + gs] = acc;
            }
        }
        __syncthreads();
    }
}

// the smem path: fp32, 2 <= p <= 8, halo (p-1)*d <= SP_MAX_HALO.  p = 2 max-pool FORWARD
// keeps the register kernel above (measured 3.7-4.8 vs 2.5-3.4 TB/s on the config shapes);
// p = 2 backward is faster here (3.0-4.0 vs 2.7-3.1 TB/s, profiles/r02_pool_bench.txt)
template <typename T>
static inline bool sp_use(int p, int d, bool max_fwd) {
    if (sizeof(T) != 4 || p < 2 || p > 8 || getenv("DP_POOL_GLOBAL")) return false;
    if (max_fwd && p == 2 && !getenv("DP_POOL_SMEM2")) return false;
    return (long long)(p - 1) * d <= SP_MAX_HALO;
}
static inline dim3 sp_grid(int out_w, int out_h, long long planes) {
    return dim3((unsigned)ceil_div(out_w, SP_TW), (unsigned)ceil_div(out_h, SP_TH),
                (unsigned)(planes < 65535 ? planes : 65535));
}
static inline size_t sp_smem(int p, int d, size_t esz, int extra_per_cell, bool hs) {
    const size_t hx = (size_t)(p - 1) * d, RH = SP_TH + hx, RW = SP_TW + hx;
    return RH * RW * (esz + extra_per_cell) + (hs ? RH * SP_TW * (esz + 1) : 0);
}

#define SP_P_SWITCH(P_RT, CALL) \
    switch (P_RT) {             \
        case 2: CALL(2); break; \
        case 3: CALL(3); break; \
        case 4: CALL(4); break; \
        case 5: CALL(5); break; \
        case 6: CALL(6); break; \
        case 7: CALL(7); break; \
        default: CALL(8); break; \
    }

template <typename K>
static inline int sp_launch_prep(K kern, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess)
            return set_error(DP_ERR_CUDA, "pool smem attribute: %s", cudaGetErrorString(e));
    }
    return DP_OK;
}

// grid for `planes` planes of `pixels` pixels each (planes split over y and z)
static inline dim3 pool_grid(long long planes, long long pixels) {
    unsigned gy = (unsigned)(planes < 65535 ? planes : 65535);
    unsigned gz = (unsigned)((planes + gy - 1) / gy);
    return dim3((unsigned)((pixels + 255) / 256), gy, gz);
}


// pool_stream.cu: warp-streaming fp32 / uint8-code kernels; -1 = shape not covered
int maxpool_forward_stream(const float *x, float *y, void *arg, int arg_bytes, long long planes,
                           int h, int w, int p, int d, int act, cudaStream_t st,
                           void *yh = nullptr, void *yl = nullptr, int yp = 0);
int maxpool_backward_stream(const float *dy, const void *arg, int arg_bytes, float *dx,
                            long long planes, int ho, int wo, int p, int d, int hi, int wi,
                            const float *gate, int gate_kind, int wd, cudaStream_t st);

template <typename T>
int maxpool_forward_t(const T *x, T *y, void *arg, int arg_bytes, int n, int c, int h, int w,
                      int p, int d, int act, cudaStream_t st) {
    int e = (p - 1) * d + 1;
    int ho = h - e + 1, wo = w - e + 1;
    long long planes = (long long)n * c;
    if (planes == 0 || ho <= 0 || wo <= 0) return DP_OK;
    if constexpr (sizeof(T) == 4) {
        const int rc = maxpool_forward_stream((const float *)x, (float *)y, arg, arg_bytes,
                                              planes, h, w, p, d, act, st);
        if (rc >= 0) return rc;
    }
    if constexpr (sizeof(T) == 4) if (sp_use<T>(p, d, true)) {
        const dim3 g = sp_grid(wo, ho, planes);
        const size_t smem = sp_smem(p, d, sizeof(T), 0, true);
        int rc = DP_OK;
#define SP_FWD_D(PP, DC)                                                                  \
    if (arg_bytes == 1) {                                                                 \
        rc = sp_launch_prep(maxpool_fwd_smem<T, uint8_t, PP, DC>, smem);                  \
        if (rc == DP_OK)                                                                  \
            maxpool_fwd_smem<T, uint8_t, PP, DC><<<g, dim3(32, 8), smem, st>>>(           \
                x, y, (uint8_t *)arg, h, w, ho, wo, d, act, planes);                      \
    } else {                                                                              \
        rc = sp_launch_prep(maxpool_fwd_smem<T, int32_t, PP, DC>, smem);                  \
        if (rc == DP_OK)                                                                  \
            maxpool_fwd_smem<T, int32_t, PP, DC><<<g, dim3(32, 8), smem, st>>>(           \
                x, y, (int32_t *)arg, h, w, ho, wo, d, act, planes);                      \
    }
#define SP_FWD(PP)                                                                        \
    if (d == 1) {                                                                         \
        SP_FWD_D(PP, 1)                                                                   \
    } else {                                                                              \
        SP_FWD_D(PP, 0)                                                                   \
    }
        SP_P_SWITCH(p, SP_FWD)
#undef SP_FWD
#undef SP_FWD_D
        if (rc) return rc;
        return check_launch("maxpool_fwd_smem");
    }
    dim3 blk(PT_X, PT_Y);
    dim3 g(ceil_div(wo, PT_X * PT_V), ceil_div(ho, PT_Y * PT_R),
           (unsigned)(planes < 65535 ? planes : 65535));
    if (arg_bytes == 1) {
        if (p == 2)
            maxpool_fwd_tile<T, uint8_t, 2><<<g, blk, 0, st>>>(x, y, (uint8_t *)arg, h, w, ho, wo,
                                                               p, d, act, planes);
        else
            maxpool_fwd_tile<T, uint8_t, 0><<<g, blk, 0, st>>>(x, y, (uint8_t *)arg, h, w, ho, wo,
                                                               p, d, act, planes);
    } else {
        maxpool_fwd_tile<T, int32_t, 0><<<g, blk, 0, st>>>(x, y, (int32_t *)arg, h, w, ho, wo, p,
                                                           d, act, planes);
    }
    return check_launch("maxpool_fwd_tile");
}

template <typename T>
int maxpool_backward_t(const T *dy, const void *arg, int arg_bytes, T *dx, int n, int c, int ho,
                       int wo, int p, int d, int hi, int wi, const T *gate, int gate_kind,
                       cudaStream_t st, int dx_pitch) {
    const int Wd = dx_pitch > 0 ? dx_pitch : wi;
    long long planes = (long long)n * c;
    if (planes == 0 || hi <= 0 || wi <= 0) return DP_OK;
    if constexpr (sizeof(T) == 4) {
        const int rc = maxpool_backward_stream((const float *)dy, arg, arg_bytes, (float *)dx,
                                               planes, ho, wo, p, d, hi, wi, (const float *)gate,
                                               gate_kind, Wd, st);
        if (rc >= 0) return rc;
    }
    if constexpr (sizeof(T) == 4) if (sp_use<T>(p, d, false)) {
        const dim3 g = sp_grid(wi, hi, planes);
        const size_t smem = sp_smem(p, d, sizeof(T), 1, false);
        int rc = DP_OK;
#define SP_BWD_D(PP, DC)                                                                    \
    if (arg_bytes == 1) {                                                                   \
        rc = sp_launch_prep(maxpool_bwd_smem<T, uint8_t, PP, DC>, smem);                    \
        if (rc == DP_OK)                                                                    \
            maxpool_bwd_smem<T, uint8_t, PP, DC><<<g, dim3(32, 8), smem, st>>>(             \
                dy, (const uint8_t *)arg, dx, gate, ho, wo, hi, wi, d, gate_kind, planes, Wd); \
    } else {                                                                                \
        rc = sp_launch_prep(maxpool_bwd_smem<T, int32_t, PP, DC>, smem);                    \
        if (rc == DP_OK)                                                                    \
            maxpool_bwd_smem<T, int32_t, PP, DC><<<g, dim3(32, 8), smem, st>>>(             \
                dy, (const int32_t *)arg, dx, gate, ho, wo, hi, wi, d, gate_kind, planes, Wd); \
    }
#define SP_BWD(PP)                                                                          \
    if (d == 1) {                                                                           \
        SP_BWD_D(PP, 1)                                                                     \
    } else {                                                                                \
        SP_BWD_D(PP, 0)                                                                     \
    }
        SP_P_SWITCH(p, SP_BWD)
#undef SP_BWD
#undef SP_BWD_D
        if (rc) return rc;
        return check_launch("maxpool_bwd_smem");
    }
    dim3 blk(PT_X, PT_Y);
    dim3 g(ceil_div(wi, PT_X * PB_V), ceil_div(hi, PT_Y * PT_R),
           (unsigned)(planes < 65535 ? planes : 65535));
    if (arg_bytes == 1) {
        if (p == 2)
            maxpool_bwd_tile<T, uint8_t, 2><<<g, blk, 0, st>>>(dy, (const uint8_t *)arg, dx, gate,
                                                               ho, wo, hi, wi, p, d, gate_kind,
                                                               planes, Wd);
        else
            maxpool_bwd_tile<T, uint8_t, 0><<<g, blk, 0, st>>>(dy, (const uint8_t *)arg, dx, gate,
                                                               ho, wo, hi, wi, p, d, gate_kind,
                                                               planes, Wd);
    } else {
        maxpool_bwd_tile<T, int32_t, 0><<<g, blk, 0, st>>>(dy, (const int32_t *)arg, dx, gate, ho,
                                                           wo, hi, wi, p, d, gate_kind, planes,
                                                           Wd);
    }
    return check_launch("maxpool_bwd_tile");
}

template <typename T>
int avgpool_forward_t(const T *x, T *y, int n, int c, int h, int w, int p, int d, int act,
                      cudaStream_t st) {
    int e = (p - 1) * d + 1;
    int ho = h - e + 1, wo = w - e + 1;
    long long planes = (long long)n * c;
    if (planes == 0 || ho <= 0 || wo <= 0) return DP_OK;
    if constexpr (sizeof(T) == 4) if (sp_use<T>(p, d, false)) {
        const dim3 g = sp_grid(wo, ho, planes);
        const size_t smem = sp_smem(p, d, sizeof(T), 0, false);
        int rc = DP_OK;
#define SP_AF(PP)                                                                        \
    rc = sp_launch_prep(avgpool_fwd_smem<T, PP>, smem);                                  \
    if (rc == DP_OK)                                                                     \
        avgpool_fwd_smem<T, PP><<<g, dim3(32, 8), smem, st>>>(x, y, h, w, ho, wo, d, act, \
                                                               planes);
        SP_P_SWITCH(p, SP_AF)
#undef SP_AF
        if (rc) return rc;
        return check_launch("avgpool_fwd_smem");
    }
    dim3 g = pool_grid(planes, (long long)ho * wo);
    avgpool_fwd_kernel<T><<<g, 256, 0, st>>>(x, y, h, w, ho, wo, p, d, act, planes);
    return check_launch("avgpool_fwd_kernel");
}

template <typename T>
int avgpool_backward_t(const T *dy, T *dx, int n, int c, int ho, int wo, int p, int d, int hi,
                       int wi, const T *gate, int gate_kind, cudaStream_t st) {
    long long planes = (long long)n * c;
    if (planes == 0 || hi <= 0 || wi <= 0) return DP_OK;
    if constexpr (sizeof(T) == 4) if (sp_use<T>(p, d, false)) {
        const dim3 g = sp_grid(wi, hi, planes);
        const size_t smem = sp_smem(p, d, sizeof(T), 0, false);
        int rc = DP_OK;
#define SP_AB(PP)                                                                          \
    rc = sp_launch_prep(avgpool_bwd_smem<T, PP>, smem);                                    \
    if (rc == DP_OK)                                                                       \
        avgpool_bwd_smem<T, PP><<<g, dim3(32, 8), smem, st>>>(dy, dx, gate, ho, wo, hi, wi, \
                                                               d, gate_kind, planes);
        SP_P_SWITCH(p, SP_AB)
#undef SP_AB
        if (rc) return rc;
        return check_launch("avgpool_bwd_smem");
    }
    dim3 g = pool_grid(planes, (long long)hi * wi);
    avgpool_bwd_kernel<T><<<g, 256, 0, st>>>(dy, dx, gate, ho, wo, hi, wi, p, d, gate_kind, planes);
    return check_launch("avgpool_bwd_kernel");
}

#define DP_POOL_INST(T)                                                                       \
    template int maxpool_forward_t<T>(const T *, T *, void *, int, int, int, int, int, int,   \
                                      int, int, cudaStream_t);                                \
    template int maxpool_backward_t<T>(const T *, const void *, int, T *, int, int, int, int, \
                                       int, int, int, int, const T *, int, cudaStream_t, int); \
    template int avgpool_forward_t<T>(const T *, T *, int, int, int, int, int, int, int,      \
                                      cudaStream_t);                                          \
    template int avgpool_backward_t<T>(const T *, T *, int, int, int, int, int, int, int, int, \
                                       const T *, int, cudaStream_t);
DP_POOL_INST(float)
DP_POOL_INST(double)

}  // namespace dp
