// d-regularly sparse max / average pooling, forward and backward (sm_100a).
//
// HBM-bound kernels; one thread per output (forward) or per input pixel
// (backward), consecutive threads on consecutive columns so every tap read is
// a coalesced row segment (shifted taps hit L1/L2).  Results are bit-identical
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

template <typename T, typename A>
__global__ void maxpool_fwd_kernel(const T *__restrict__ x, T *__restrict__ y,
                                   A *__restrict__ arg, long long total, int H, int W, int Ho,
                                   int Wo, int p, int d, int act) {
    long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int v = (int)(idx % Wo);
    long long t = idx / Wo;
    int u = (int)(t % Ho);
    long long plane = t / Ho;  // n*C + c
    const T *src = x + plane * H * W + (long long)u * W + v;
    T best = neg_inf<T>();
    int bk = 0;
    for (int i = 0; i < p; ++i) {
        const T *row = src + (long long)i * d * W;
        for (int j = 0; j < p; ++j) {
            T xv = row[j * d];
            if (xv > best) {
                best = xv;
                bk = i * p + j;
            }
        }
    }
    y[idx] = apply_nonlin(best, act);
    arg[idx] = (A)bk;
}

template <typename T, typename A>
__global__ void maxpool_bwd_kernel(const T *__restrict__ dy, const A *__restrict__ arg,
                                   T *__restrict__ dx, const T *__restrict__ gate,
                                   long long total, int Ho, int Wo, int Hi, int Wi, int p, int d,
                                   int gate_kind) {
    long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int s = (int)(idx % Wi);
    long long t = idx / Wi;
    int r = (int)(t % Hi);
    long long plane = t / Hi;
    const T *dyp = dy + plane * Ho * Wo;
    const A *ap = arg + plane * Ho * Wo;
    T acc = T(0);
    for (int i = p - 1; i >= 0; --i) {
        int u = r - i * d;
        if (u < 0 || u >= Ho) continue;
        for (int j = p - 1; j >= 0; --j) {
            int v = s - j * d;
            if (v < 0 || v >= Wo) continue;
            long long o = (long long)u * Wo + v;
            if ((int)ap[o] == i * p + j) acc = add_rn(acc, dyp[o]);
        }
    }
    if (gate) acc = gate_from_output(acc, gate[idx], gate_kind);
    dx[idx] = acc;
}

template <typename T>
__global__ void avgpool_fwd_kernel(const T *__restrict__ x, T *__restrict__ y, long long total,
                                   int H, int W, int Ho, int Wo, int p, int d, int act) {
    long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int v = (int)(idx % Wo);
    long long t = idx / Wo;
    int u = (int)(t % Ho);
    long long plane = t / Ho;
    const T *src = x + plane * H * W + (long long)u * W + v;
    T acc = T(0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) acc = add_rn(acc, src[(long long)i * d * W + j * d]);
    y[idx] = apply_nonlin(div_rn(acc, T(p * p)), act);
}

template <typename T>
__global__ void avgpool_bwd_kernel(const T *__restrict__ dy, T *__restrict__ dx,
                                   const T *__restrict__ gate, long long total, int Ho, int Wo,
                                   int Hi, int Wi, int p, int d, int gate_kind) {
    long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int s = (int)(idx % Wi);
    long long t = idx / Wi;
    int r = (int)(t % Hi);
    long long plane = t / Hi;
    const T *dyp = dy + plane * Ho * Wo;
    const T pp = T(p * p);
    T acc = T(0);
    for (int i = p - 1; i >= 0; --i) {
        int u = r - i * d;
        if (u < 0 || u >= Ho) continue;
        for (int j = p - 1; j >= 0; --j) {
            int v = s - j * d;
            if (v < 0 || v >= Wo) continue;
            acc = add_rn(acc, div_rn(dyp[(long long)u * Wo + v], pp));
        }
    }
    if (gate) acc = gate_from_output(acc, gate[idx], gate_kind);
    dx[idx] = acc;
}

static inline int blocks_for(long long total) { return ceil_div(total, 256); }

template <typename T>
int maxpool_forward_t(const T *x, T *y, void *arg, int arg_bytes, int n, int c, int h, int w,
                      int p, int d, int act, cudaStream_t st) {
    int e = (p - 1) * d + 1;
    int ho = h - e + 1, wo = w - e + 1;
    long long total = (long long)n * c * ho * wo;
    if (total == 0) return DP_OK;
    if (arg_bytes == 1)
        maxpool_fwd_kernel<T, uint8_t><<<blocks_for(total), 256, 0, st>>>(
            x, y, (uint8_t *)arg, total, h, w, ho, wo, p, d, act);
    else
        maxpool_fwd_kernel<T, int32_t><<<blocks_for(total), 256, 0, st>>>(
            x, y, (int32_t *)arg, total, h, w, ho, wo, p, d, act);
    return check_launch("maxpool_fwd_kernel");
}

template <typename T>
int maxpool_backward_t(const T *dy, const void *arg, int arg_bytes, T *dx, int n, int c, int ho,
                       int wo, int p, int d, int hi, int wi, const T *gate, int gate_kind,
                       cudaStream_t st) {
    long long total = (long long)n * c * hi * wi;
    if (total == 0) return DP_OK;
    if (arg_bytes == 1)
        maxpool_bwd_kernel<T, uint8_t><<<blocks_for(total), 256, 0, st>>>(
            dy, (const uint8_t *)arg, dx, gate, total, ho, wo, hi, wi, p, d, gate_kind);
    else
        maxpool_bwd_kernel<T, int32_t><<<blocks_for(total), 256, 0, st>>>(
            dy, (const int32_t *)arg, dx, gate, total, ho, wo, hi, wi, p, d, gate_kind);
    return check_launch("maxpool_bwd_kernel");
}

template <typename T>
int avgpool_forward_t(const T *x, T *y, int n, int c, int h, int w, int p, int d, int act,
                      cudaStream_t st) {
    int e = (p - 1) * d + 1;
    int ho = h - e + 1, wo = w - e + 1;
    long long total = (long long)n * c * ho * wo;
    if (total == 0) return DP_OK;
    avgpool_fwd_kernel<T><<<blocks_for(total), 256, 0, st>>>(x, y, total, h, w, ho, wo, p, d,
                                                             act);
    return check_launch("avgpool_fwd_kernel");
}

template <typename T>
int avgpool_backward_t(const T *dy, T *dx, int n, int c, int ho, int wo, int p, int d, int hi,
                       int wi, const T *gate, int gate_kind, cudaStream_t st) {
    long long total = (long long)n * c * hi * wi;
    if (total == 0) return DP_OK;
    avgpool_bwd_kernel<T><<<blocks_for(total), 256, 0, st>>>(dy, dx, gate, total, ho, wo, hi,
                                                             wi, p, d, gate_kind);
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
