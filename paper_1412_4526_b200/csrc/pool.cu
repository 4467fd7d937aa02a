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
                     int gate_kind, long long planes) {
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
            const long long os = (long long)PT_Y * Wo, qs = (long long)PT_Y * Wi;
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
                T *dxo = dx + q;
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
            }
        } else {
            const int p = p_rt;
            for (int ry = 0; ry < PT_R; ++ry) {
                const int r = r0 + ry * PT_Y;
                if (r >= Hi) break;
                const long long q0 = (plane * Hi + r) * (long long)Wi;
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
                    dx[q0 + s] = acc;
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

// grid for `planes` planes of `pixels` pixels each (planes split over y and z)
static inline dim3 pool_grid(long long planes, long long pixels) {
    unsigned gy = (unsigned)(planes < 65535 ? planes : 65535);
    unsigned gz = (unsigned)((planes + gy - 1) / gy);
    return dim3((unsigned)((pixels + 255) / 256), gy, gz);
}


template <typename T>
int maxpool_forward_t(const T *x, T *y, void *arg, int arg_bytes, int n, int c, int h, int w,
                      int p, int d, int act, cudaStream_t st) {
    int e = (p - 1) * d + 1;
    int ho = h - e + 1, wo = w - e + 1;
    long long planes = (long long)n * c;
    if (planes == 0 || ho <= 0 || wo <= 0) return DP_OK;
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
                       cudaStream_t st) {
    long long planes = (long long)n * c;
    if (planes == 0 || hi <= 0 || wi <= 0) return DP_OK;
    dim3 blk(PT_X, PT_Y);
    dim3 g(ceil_div(wi, PT_X * PB_V), ceil_div(hi, PT_Y * PT_R),
           (unsigned)(planes < 65535 ? planes : 65535));
    if (arg_bytes == 1) {
        if (p == 2)
            maxpool_bwd_tile<T, uint8_t, 2><<<g, blk, 0, st>>>(dy, (const uint8_t *)arg, dx, gate,
                                                               ho, wo, hi, wi, p, d, gate_kind,
                                                               planes);
        else
            maxpool_bwd_tile<T, uint8_t, 0><<<g, blk, 0, st>>>(dy, (const uint8_t *)arg, dx, gate,
                                                               ho, wo, hi, wi, p, d, gate_kind,
                                                               planes);
    } else {
        maxpool_bwd_tile<T, int32_t, 0><<<g, blk, 0, st>>>(dy, (const int32_t *)arg, dx, gate, ho,
                                                           wo, hi, wi, p, d, gate_kind, planes);
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
    dim3 g = pool_grid(planes, (long long)ho * wo);
    avgpool_fwd_kernel<T><<<g, 256, 0, st>>>(x, y, h, w, ho, wo, p, d, act, planes);
    return check_launch("avgpool_fwd_kernel");
}

template <typename T>
int avgpool_backward_t(const T *dy, T *dx, int n, int c, int ho, int wo, int p, int d, int hi,
                       int wi, const T *gate, int gate_kind, cudaStream_t st) {
    long long planes = (long long)n * c;
    if (planes == 0 || hi <= 0 || wi <= 0) return DP_OK;
    dim3 g = pool_grid(planes, (long long)hi * wi);
    avgpool_bwd_kernel<T><<<g, 256, 0, st>>>(dy, dx, gate, ho, wo, hi, wi, p, d, gate_kind, planes);
    return check_launch("avgpool_bwd_kernel");
}

#define DP_POOL_INST(T)                                                                       \
    template int maxpool_forward_t<T>(const T *, T *, void *, int, int, int, int, int, int,   \
                                      int, int, cudaStream_t);                                \
    template int maxpool_backward_t<T>(const T *, const void *, int, T *, int, int, int, int, \
                                       int, int, int, int, const T *, int, cudaStream_t);     \
    template int avgpool_forward_t<T>(const T *, T *, int, int, int, int, int, int, int,      \
                                      cudaStream_t);                                          \
    template int avgpool_backward_t<T>(const T *, T *, int, int, int, int, int, int, int, int, \
                                       const T *, int, cudaStream_t);
DP_POOL_INST(float)
DP_POOL_INST(double)

}  // namespace dp
