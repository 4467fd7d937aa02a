// Elementwise kernels: nonlinearity, error-map mask / loss, pad, crop, SGD.
//
// nonlin fwd/bwd ... reference forward.py:69-76 / backward.py:172-182 (numpy
//                    there, outside the kernel boundary); relu and identity
//                    are bit-exact, tanh within 2 ulp of numpy.
// mask / loss ...... backward.py:110-118 (keep the selected pixels across all
//                    channels, zero the rest) fused with the squared-error
//                    delta output - target (cli.py:218).  A dense bitmap: the
//                    cost is independent of the number of selected pixels
//                    (tests/test_acceptance.py:144-158).
// pad / crop ....... forward.py:96-98 (pad_rect with (lead, trail) margins),
//                    backward.py:218-222 (crop of the input delta).
#include "dp_common.cuh"

namespace dp {

template <typename T>
__global__ void nonlin_fwd_kernel(const T *x, T *y, long long n, int kind) {  // may alias
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = apply_nonlin(x[i], kind);
}

template <typename T>
__global__ void nonlin_bwd_kernel(const T *dy, const T *__restrict__ x, T *dx, long long n,
                                  int kind, int x_is_output) {
    // dy and dx may alias (the engine gates a delta in place): no __restrict__ on them
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        T t = x[i];
        if (!x_is_output && kind == DP_TANH) t = dp_tanh(t);
        if (!x_is_output && kind == DP_TANH_FAST) t = dp_tanh_fast(t);
        dx[i] = gate_from_output(dy[i], t, kind);
    }
}

// One thread per 4 pixels of one image: the mask is read once, the channels loop with
// 16-byte stores (zeros for unmasked pixels -- a and target are only read where the mask is
// set); the per-element 64-bit index divisions of the first version made it ALU bound.
template <typename T>
__global__ void mask_delta_kernel(const T *__restrict__ a, const T *__restrict__ target,
                                  const uint8_t *__restrict__ mask, T *__restrict__ out,
                                  long long nquads, int C, long long HW) {
    const long long qpi = HW >> 2;  // quads per image (HW % 4 == 0 on this path)
    for (long long qd = (long long)blockIdx.x * blockDim.x + threadIdx.x; qd < nquads;
         qd += (long long)gridDim.x * blockDim.x) {
        const long long img = qd / qpi;
        const long long px = (qd - img * qpi) * 4;
        const uchar4 m = *reinterpret_cast<const uchar4 *>(mask + img * HW + px);
        const bool any = m.x | m.y | m.z | m.w;
        const long long base = img * C * HW + px;
        for (int c = 0; c < C; ++c) {
            const long long i = base + (long long)c * HW;
            T v[4] = {T(0), T(0), T(0), T(0)};
            if (any) {
                const uint8_t mm[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (mm[e]) v[e] = target ? add_rn(a[i + e], -target[i + e]) : a[i + e];
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) out[i + e] = v[e];
        }
    }
}

template <typename T>
__global__ void mask_delta_scalar_kernel(const T *__restrict__ a, const T *__restrict__ target,
                                         const uint8_t *__restrict__ mask, T *__restrict__ out,
                                         long long npix, int C, long long HW) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (long long)gridDim.x * blockDim.x) {
        const long long img = p / HW, px = p - img * HW;
        const bool on = mask[p];
        for (int c = 0; c < C; ++c) {
            const long long i = (img * C + c) * HW + px;
            out[i] = on ? (target ? add_rn(a[i], -target[i]) : a[i]) : T(0);
        }
    }
}

// One block-row of threads per destination row (plane, yy): one division per row instead of
// two 64-bit divisions per element.
template <typename T>
__global__ void pad_kernel(const T *__restrict__ src, T *__restrict__ dst, long long rows,
                           int h, int w, int Hp, int Wp, int top, int left) {
    for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
        const long long plane = r / Hp;
        const int yy = (int)(r - plane * Hp);
        const int sy = yy - top;
        const bool rin = sy >= 0 && sy < h;
        const T *srow = src + (plane * h + (rin ? sy : 0)) * (long long)w;
        T *drow = dst + r * (long long)Wp;
        for (int xx = threadIdx.x; xx < Wp; xx += blockDim.x) {
            const int sx = xx - left;
            drow[xx] = (rin && sx >= 0 && sx < w) ? srow[sx] : T(0);
        }
    }
}

template <typename T>
__global__ void crop_kernel(const T *__restrict__ src, T *__restrict__ dst, long long total,
                            int hs, int ws, int top, int left, int h, int w) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int xx = (int)(i % w);
        long long t = i / w;
        int yy = (int)(t % h);
        long long plane = t / h;
        dst[i] = src[(plane * hs + yy + top) * ws + xx + left];
    }
}

template <typename T>
__global__ void sgd_kernel(T *__restrict__ p, const T *__restrict__ g, long long n, T lr) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        p[i] = add_rn(p[i], -mul_rn(lr, g[i]));  // numpy p - lr*g: no FMA contraction
}

static inline int grid_for(long long n) {
    long long b = (n + 255) / 256;
    if (b > 148LL * 32) b = 148LL * 32;
    return (int)(b < 1 ? 1 : b);
}

template <typename T>
int nonlin_forward_t(const T *x, T *y, long long n, int kind, cudaStream_t st) {
    if (n == 0) return DP_OK;
    nonlin_fwd_kernel<T><<<grid_for(n), 256, 0, st>>>(x, y, n, kind);
    return check_launch("nonlin_fwd_kernel");
}

template <typename T>
int nonlin_backward_t(const T *dy, const T *x, T *dx, long long n, int kind, int x_is_output,
                      cudaStream_t st) {
    if (n == 0) return DP_OK;
    nonlin_bwd_kernel<T><<<grid_for(n), 256, 0, st>>>(dy, x, dx, n, kind, x_is_output);
    return check_launch("nonlin_bwd_kernel");
}

template <typename T>
int mask_delta_t(const T *a, const T *target, const uint8_t *mask, T *out, int n, int c, int h,
                 int w, cudaStream_t st) {
    const long long HW = (long long)h * w;
    if ((long long)n * c * HW == 0) return DP_OK;
    const bool aligned = HW % 4 == 0 && ((uintptr_t)mask & 3) == 0;
    if (aligned) {
        const long long nq = (long long)n * HW / 4;
        mask_delta_kernel<T><<<grid_for(nq), 256, 0, st>>>(a, target, mask, out, nq, c, HW);
    } else {
        const long long np = (long long)n * HW;
        mask_delta_scalar_kernel<T><<<grid_for(np), 256, 0, st>>>(a, target, mask, out, np, c,
                                                                  HW);
    }
    return check_launch("mask_delta_kernel");
}

template <typename T>
int pad_t(const T *src, T *dst, int n, int c, int h, int w, int top, int bottom, int left,
          int right, cudaStream_t st) {
    int Hp = h + top + bottom, Wp = w + left + right;
    long long total = (long long)n * c * Hp * Wp;
    if (total == 0) return DP_OK;
    const long long rows = (long long)n * c * Hp;
    const long long g = rows < 148LL * 64 ? rows : 148LL * 64;
    pad_kernel<T><<<(int)g, 128, 0, st>>>(src, dst, rows, h, w, Hp, Wp, top, left);
    return check_launch("pad_kernel");
}

template <typename T>
int crop_t(const T *src, T *dst, int n, int c, int hs, int ws, int top, int left, int h, int w,
           cudaStream_t st) {
    long long total = (long long)n * c * h * w;
    if (total == 0) return DP_OK;
    crop_kernel<T><<<grid_for(total), 256, 0, st>>>(src, dst, total, hs, ws, top, left, h, w);
    return check_launch("crop_kernel");
}

// Per-pixel softmax cross-entropy over the q output channels (the
// 8-class labelling loss; the reference itself only has the squared-error delta,
// cli.py:218, so this is parity-unpinned and checked against torch fp64 autograd):
//   p = softmax(logits[n, :, y, x]),  loss = -log p[label],  delta = p - onehot(label)
// where mask[n,y,x] != 0 and label != 255 (ignore); zero delta / loss elsewhere.
template <typename T>
__global__ void softmax_xent_kernel(const T *__restrict__ logits, const uint8_t *__restrict__ labels,
                                    const uint8_t *__restrict__ mask, T *__restrict__ delta,
                                    T *__restrict__ loss, long long npix, int q, long long hw) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < npix;
         i += (long long)gridDim.x * blockDim.x) {
        const long long img = i / hw, px = i - img * hw;
        const T *z = logits + img * q * hw + px;
        T *dz = delta + img * q * hw + px;
        const int lab = labels[i];
        const bool on = (!mask || mask[i]) && lab < q;
        if (!on) {
            for (int c = 0; c < q; ++c) dz[c * hw] = T(0);
            if (loss) loss[i] = T(0);
            continue;
        }
        T m = z[0];
        for (int c = 1; c < q; ++c) m = z[c * hw] > m ? z[c * hw] : m;
        T s = T(0);
        for (int c = 0; c < q; ++c) s += exp(z[c * hw] - m);
        const T inv = T(1) / s;
        for (int c = 0; c < q; ++c) dz[c * hw] = exp(z[c * hw] - m) * inv - (c == lab ? T(1) : T(0));
        if (loss) loss[i] = log(s) - (z[lab * hw] - m);
    }
}

template <typename T>
int softmax_xent_t(const T *logits, const uint8_t *labels, const uint8_t *mask, T *delta, T *loss,
                   int n, int q, int h, int w, cudaStream_t st) {
    const long long npix = (long long)n * h * w;
    if (npix == 0) return DP_OK;
    softmax_xent_kernel<T><<<grid_for(npix), 256, 0, st>>>(logits, labels, mask, delta, loss, npix,
                                                           q, (long long)h * w);
    return check_launch("softmax_xent_kernel");
}

// Patch gather for the patch-by-patch baseline (reference oracle.py scan_forward:145-164 runs
// the strided classifier on one patch per pixel): out[k, c, i, j] = x0[img, c, y+i, x+j] with
// (y, x) = divmod(first + k, w) over the w-wide output grid of padded image img.
template <typename T>
__global__ void patch_gather_kernel(const T *__restrict__ x0, T *__restrict__ out,
                                    long long total, int C, int Hp, int Wp, int P, int w,
                                    long long first) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int jj = (int)(i % P);
        long long t = i / P;
        const int ii = (int)(t % P);
        t /= P;
        const int c = (int)(t % C);
        const long long k = t / C;
        const long long pix = first + k;
        const int y = (int)(pix / w), x = (int)(pix - (long long)y * w);
        out[i] = x0[((long long)c * Hp + y + ii) * Wp + x + jj];
    }
}

template <typename T>
int patch_gather_t(const T *x0, T *out, int C, int Hp, int Wp, int P, int w, long long first,
                   long long count, cudaStream_t st) {
    const long long total = count * C * P * P;
    if (total == 0) return DP_OK;
    patch_gather_kernel<T><<<grid_for(total), 256, 0, st>>>(x0, out, total, C, Hp, Wp, P, w,
                                                            first);
    return check_launch("patch_gather_kernel");
}

template <typename T>
int sgd_t(T *p, const T *g, long long n, double lr, cudaStream_t st) {
    if (n == 0) return DP_OK;
    sgd_kernel<T><<<grid_for(n), 256, 0, st>>>(p, g, n, (T)lr);
    return check_launch("sgd_kernel");
}

#define DP_EW_INST(T)                                                                         \
    template int nonlin_forward_t<T>(const T *, T *, long long, int, cudaStream_t);           \
    template int nonlin_backward_t<T>(const T *, const T *, T *, long long, int, int,         \
                                      cudaStream_t);                                          \
    template int mask_delta_t<T>(const T *, const T *, const uint8_t *, T *, int, int, int,   \
                                 int, cudaStream_t);                                          \
    template int pad_t<T>(const T *, T *, int, int, int, int, int, int, int, int,             \
                          cudaStream_t);                                                      \
    template int crop_t<T>(const T *, T *, int, int, int, int, int, int, int, int,            \
                           cudaStream_t);                                                     \
    template int sgd_t<T>(T *, const T *, long long, double, cudaStream_t);                  \
    template int patch_gather_t<T>(const T *, T *, int, int, int, int, int, long long,        \
                                   long long, cudaStream_t);                                  \
    template int softmax_xent_t<T>(const T *, const uint8_t *, const uint8_t *, T *, T *, int,  \
                                   int, int, int, cudaStream_t);
DP_EW_INST(float)
DP_EW_INST(double)

}  // namespace dp
