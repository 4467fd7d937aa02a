// Original (strided) network layers for the GPU patch-by-patch baseline.
//
// The dense engine replaces "run the strided patch classifier once per pixel" (reference
// oracle.py:29-262: conv_strided, maxpool_strided, avgpool_strided, scan_forward,
// patch_backward_batch).  To measure that baseline on the same B200 and to check the
// dense path against it, the patch network runs here on batches of patches:
//
//   strided max / avg pool ... oracle.py:58-91: y = tap (0,0), then taps in row-major order,
//                              max with strict `>` (first wins), avg as a running sum / p^2;
//                              int32 argmax i*p + j.
//   strided pool backward .... oracle.py:190-211 as a gather: each input pixel sums, in
//                              ascending tap order, the window deltas routed to it (the
//                              reference scatters tap by tap onto zeros: same order).
//   subsample / zero insert .. a stride-s conv = the stride-1 conv sampled every s pixels
//                              (forward) and the stride-1 backward of the zero-inserted
//                              delta (backward): exact, s^2 more MACs on those layers.
//   patch gather (pixel list)  the windows of an arbitrary pixel list (patch_backward_batch
//                              takes any pixel set, oracle.py:237-262).
//
// Stride-1 convolutions of the patch network use the dense kernels at dilation 1.
// CUDA cores, one thread per output element: the baseline's cost is in its convolutions.
#include "dp_common.cuh"
#include "../../include/denseprop_b200.h"

namespace dp {

static inline int grid1d(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148LL * 16) b = 148LL * 16;
    return (int)(b < 1 ? 1 : b);
}

template <typename T>
__global__ void pool_strided_fwd_kernel(const T *__restrict__ x, T *__restrict__ y,
                                        int32_t *__restrict__ arg, long long total, int H, int W,
                                        int Ho, int Wo, int p, int s, int is_max) {
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(o % Wo);
        const long long t = o / Wo;
        const int u = (int)(t % Ho);
        const long long plane = t / Ho;
        const T *xp = x + (plane * H + (long long)u * s) * W + (long long)v * s;
        T best = xp[0];
        int ai = 0;
        for (int i = 0; i < p; ++i)
            for (int j = 0; j < p; ++j) {
                if (i == 0 && j == 0) continue;
                const T val = xp[(long long)i * W + j];
                if (is_max) {
                    if (val > best) {
                        best = val;
                        ai = i * p + j;
                    }
                } else {
                    best = add_rn(best, val);
                }
            }
        if (is_max) {
            y[o] = best;
            arg[o] = ai;
        } else {
            y[o] = div_rn(best, T(p * p));
        }
    }
}

template <typename T>
__global__ void pool_strided_bwd_kernel(const T *__restrict__ dy, const int32_t *__restrict__ arg,
                                        T *__restrict__ dx, long long total, int Ho, int Wo,
                                        int Hi, int Wi, int p, int s, int is_max) {
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const int xx = (int)(o % Wi);
        const long long t = o / Wi;
        const int yy = (int)(t % Hi);
        const long long plane = t / Hi;
        const T *dyp = dy + plane * Ho * Wo;
        const int32_t *ap = arg ? arg + plane * Ho * Wo : nullptr;
        T acc = T(0);
        for (int i = 0; i < p; ++i) {
            const int ur = yy - i;
            if (ur < 0 || ur % s) continue;
            const int u = ur / s;
            if (u >= Ho) continue;
            for (int j = 0; j < p; ++j) {
                const int vr = xx - j;
                if (vr < 0 || vr % s) continue;
                const int v = vr / s;
                if (v >= Wo) continue;
                const long long q = (long long)u * Wo + v;
                if (is_max) {
                    if (ap[q] == i * p + j) acc = add_rn(acc, dyp[q]);
                } else {
                    acc = add_rn(acc, div_rn(dyp[q], T(p * p)));
                }
            }
        }
        dx[o] = acc;
    }
}

template <typename T>
__global__ void subsample_kernel(const T *__restrict__ x, T *__restrict__ y, long long total,
                                 int H, int W, int Ho, int Wo, int s) {
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(o % Wo);
        const long long t = o / Wo;
        const int u = (int)(t % Ho);
        const long long plane = t / Ho;
        y[o] = x[(plane * H + (long long)u * s) * W + (long long)v * s];
    }
}

template <typename T>
__global__ void zero_insert_kernel(const T *__restrict__ dy, T *__restrict__ out, long long total,
                                   int Ho, int Wo, int Hf, int Wf, int s) {
    for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const int xx = (int)(o % Wf);
        const long long t = o / Wf;
        const int yy = (int)(t % Hf);
        const long long plane = t / Hf;
        T v = T(0);
        if (yy % s == 0 && xx % s == 0 && yy / s < Ho && xx / s < Wo)
            v = dy[(plane * Ho + yy / s) * Wo + xx / s];
        out[o] = v;
    }
}

template <typename T>
__global__ void patch_gather_pixels_kernel(const T *__restrict__ x0, T *__restrict__ out,
                                           const int32_t *__restrict__ pix, long long total,
                                           int C, int Hp, int Wp, int P, int w) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int jj = (int)(i % P);
        long long t = i / P;
        const int ii = (int)(t % P);
        t /= P;
        const int c = (int)(t % C);
        const long long k = t / C;
        const int f = pix[k];
        const int y = f / w, x = f - y * w;
        out[i] = x0[((long long)c * Hp + y + ii) * Wp + x + jj];
    }
}

}  // namespace dp

using namespace dp;

static int arg_err(const char *msg) { return set_error(DP_ERR_ARG, "%s", msg); }

#define DP_ST_TRY(expr)         \
    do {                        \
        int _rc = (expr);       \
        if (_rc) return _rc;    \
    } while (0)

static int st_dtype(int dtype) {
    if (dtype != DP_F32 && dtype != DP_F64)
        return set_error(DP_ERR_ARG, "dtype must be DP_F32 or DP_F64, got %d", dtype);
    return DP_OK;
}

static int st_dims(int n, int c, int a, int b) {
    if (n < 1 || c < 1 || a < 1 || b < 1) return arg_err("dimensions must be >= 1");
    return DP_OK;
}

extern "C" {

int dp_pool_strided_forward(int dtype, int kind, const void *x, void *y, int32_t *arg, int n,
                            int c, int h, int w, int p, int s, void *stream) {
    DP_ST_TRY(st_dtype(dtype));
    DP_ST_TRY(st_dims(n, c, h, w));
    if (kind != DP_POOL_MAX && kind != DP_POOL_AVG) return arg_err("pool kind must be max or avg");
    if (p < 1 || s < 1) return arg_err("pool kernel and stride must be >= 1");
    if (h < p || w < p || (h - p) % s || (w - p) % s)
        return set_error(DP_ERR_ARG, "%dx%d/%d windows do not tile a %dx%d input exactly", p, p, s,
                         h, w);
    if (kind == DP_POOL_MAX && !arg) return arg_err("max pool needs an argmax buffer");
    const int ho = (h - p) / s + 1, wo = (w - p) / s + 1;
    const long long total = (long long)n * c * ho * wo;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DP_F32)
        pool_strided_fwd_kernel<float><<<grid1d(total), 256, 0, st>>>(
            (const float *)x, (float *)y, arg, total, h, w, ho, wo, p, s, kind == DP_POOL_MAX);
    else
        pool_strided_fwd_kernel<double><<<grid1d(total), 256, 0, st>>>(
            (const double *)x, (double *)y, arg, total, h, w, ho, wo, p, s, kind == DP_POOL_MAX);
    return check_launch("pool_strided_fwd_kernel");
}

int dp_pool_strided_backward(int dtype, int kind, const void *dy, const int32_t *arg, void *dx,
                             int n, int c, int ho, int wo, int p, int s, int hi, int wi,
                             void *stream) {
    DP_ST_TRY(st_dtype(dtype));
    DP_ST_TRY(st_dims(n, c, ho, wo));
    if (kind != DP_POOL_MAX && kind != DP_POOL_AVG) return arg_err("pool kind must be max or avg");
    if (p < 1 || s < 1) return arg_err("pool kernel and stride must be >= 1");
    if ((long long)(ho - 1) * s + p != hi || (long long)(wo - 1) * s + p != wi)
        return set_error(DP_ERR_ARG, "pool backward: %dx%d input does not match %dx%d output "
                         "of %dx%d/%d windows", hi, wi, ho, wo, p, p, s);
    if (kind == DP_POOL_MAX && !arg) return arg_err("max pool backward needs the argmax map");
    const long long total = (long long)n * c * hi * wi;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DP_F32)
        pool_strided_bwd_kernel<float><<<grid1d(total), 256, 0, st>>>(
            (const float *)dy, arg, (float *)dx, total, ho, wo, hi, wi, p, s, kind == DP_POOL_MAX);
    else
        pool_strided_bwd_kernel<double><<<grid1d(total), 256, 0, st>>>(
            (const double *)dy, arg, (double *)dx, total, ho, wo, hi, wi, p, s,
            kind == DP_POOL_MAX);
    return check_launch("pool_strided_bwd_kernel");
}

int dp_subsample(int dtype, const void *x, void *y, int n, int c, int h, int w, int s, int ho,
                 int wo, void *stream) {
    DP_ST_TRY(st_dtype(dtype));
    DP_ST_TRY(st_dims(n, c, h, w));
    if (s < 1 || ho < 1 || wo < 1 || (long long)(ho - 1) * s >= h || (long long)(wo - 1) * s >= w)
        return arg_err("subsample: output grid leaves the input");
    const long long total = (long long)n * c * ho * wo;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DP_F32)
        subsample_kernel<float><<<grid1d(total), 256, 0, st>>>((const float *)x, (float *)y,
                                                               total, h, w, ho, wo, s);
    else
        subsample_kernel<double><<<grid1d(total), 256, 0, st>>>((const double *)x, (double *)y,
                                                                total, h, w, ho, wo, s);
    return check_launch("subsample_kernel");
}

int dp_zero_insert(int dtype, const void *dy, void *out, int n, int c, int ho, int wo, int s,
                   int hf, int wf, void *stream) {
    DP_ST_TRY(st_dtype(dtype));
    DP_ST_TRY(st_dims(n, c, ho, wo));
    if (s < 1 || (long long)(ho - 1) * s >= hf || (long long)(wo - 1) * s >= wf)
        return arg_err("zero insert: strided grid leaves the output");
    const long long total = (long long)n * c * hf * wf;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DP_F32)
        zero_insert_kernel<float><<<grid1d(total), 256, 0, st>>>((const float *)dy, (float *)out,
                                                                 total, ho, wo, hf, wf, s);
    else
        zero_insert_kernel<double><<<grid1d(total), 256, 0, st>>>(
            (const double *)dy, (double *)out, total, ho, wo, hf, wf, s);
    return check_launch("zero_insert_kernel");
}

int dp_patch_gather_pixels(int dtype, const void *x0, void *out, int c, int hp, int wp, int patch,
                           const int32_t *pixels, int64_t count, void *stream) {
    DP_ST_TRY(st_dtype(dtype));
    if (c < 1 || patch < 1) return arg_err("channels and patch must be >= 1");
    const int w = wp - patch + 1, h = hp - patch + 1;
    if (w < 1 || h < 1) return arg_err("patch gather: padded map smaller than the patch");
    if (count < 0 || (count > 0 && !pixels)) return arg_err("patch gather: bad pixel list");
    const long long total = count * c * patch * patch;
    if (total == 0) return DP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == DP_F32)
        patch_gather_pixels_kernel<float><<<grid1d(total), 256, 0, st>>>(
            (const float *)x0, (float *)out, pixels, total, c, hp, wp, patch, w);
    else
        patch_gather_pixels_kernel<double><<<grid1d(total), 256, 0, st>>>(
            (const double *)x0, (double *)out, pixels, total, c, hp, wp, patch, w);
    return check_launch("patch_gather_pixels_kernel");
}

}  // extern "C"
