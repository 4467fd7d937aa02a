// Exact-tier d-regularly sparse (dilated) convolution on CUDA cores, sm_100a.
//
// One kernel serves both directions of the reference's conv data path:
//   forward        y[o,u,v]  = b[o] + sum_{c,i,j} w[o,c,i,j] * x[c, u+i*d, v+j*d]
//                  (reference _kernels.pyx:23-53)
//   data gradient  dx[c,y,x] = 0    + sum_{o,i,j} w[o,c,l-1-i,l-1-j] * dy_pad[o, y+i*d, x+j*d]
//                  (gather form, _kernels.pyx:56-91; dy zero-padded by e-1)
// Both are "out[q,u,v] = init + sum over (r,i,j) in lexicographic order of
// W(q,r,i,j) * in[r, u+i*d-pad, v+j*d-pad]" with zeros outside `in`.  Every
// output keeps that exact operation order and rounds the product and the sum
// separately (mul_rn / add_rn), so results are bit-identical to the compiled
// reference backend.  Out-of-range taps add an exact +-0.0 where the
// reference skips them; a running sum that starts at +0.0 is unchanged by it.
//
// Tiling: a CTA owns TW=32 columns x TH=16 rows x OT output channels.  For each
// reduction channel r it stages the l input row-bands it needs
// (rows u0+i*d .. +TH, cols v0 .. v0+TW+(l-1)*d) and the OT x l x l weights in
// shared memory; each thread then accumulates 4 rows x OT channels at one
// column (lane = column, so shared loads are conflict-free and global
// loads/stores are coalesced).  Nonlinearity (forward) or the upstream
// nonlinearity's derivative (backward) is applied in the epilogue.
#include "dp_common.cuh"

namespace dp {

constexpr int CONV_TW = 32;
constexpr int CONV_TH = 16;
constexpr int CONV_THREADS = 128;  // 4 warps x 4 rows each
constexpr int CONV_RPT = CONV_TH / (CONV_THREADS / CONV_TW);

template <typename T, int OT, bool BWD>
__global__ void __launch_bounds__(CONV_THREADS)
conv_direct_kernel(const T *__restrict__ in, const T *__restrict__ wt, const T *__restrict__ bias,
                   T *__restrict__ out, const T *__restrict__ gate, int R, int Q, int Hin,
                   int Win, int Ho, int Wo, int l, int d, int pad, int act, int gate_kind,
                   int tiles_x) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *s_w = reinterpret_cast<T *>(smem_raw);           // [l*l][OT]
    T *s_in = s_w + l * l * OT;                         // [l][TH][SW]
    const int SW = CONV_TW + (l - 1) * d;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x;
    const int v0 = (tile % tiles_x) * CONV_TW;
    const int u0 = (tile / tiles_x) * CONV_TH;
    const int q0 = blockIdx.y * OT;
    const long long img = blockIdx.z;
    const T *in_img = in + img * (long long)R * Hin * Win;

    T acc[OT][CONV_RPT];
#pragma unroll
    for (int o = 0; o < OT; ++o) {
        T init = T(0);
        if (!BWD && q0 + o < Q) init = bias[q0 + o];
#pragma unroll
        for (int r = 0; r < CONV_RPT; ++r) acc[o][r] = init;
    }

    const int band = CONV_TH * SW;
    const int n_in = l * band;
    const int n_w = l * l * OT;
    for (int r = 0; r < R; ++r) {
        __syncthreads();
        const T *plane = in_img + (long long)r * Hin * Win;
        for (int idx = tid; idx < n_in; idx += CONV_THREADS) {
            int i = idx / band;
            int rem = idx - i * band;
            int row = rem / SW;
            int col = rem - row * SW;
            int gy = u0 + i * d + row - pad;
            int gx = v0 + col - pad;
            T v = T(0);
            if (gy >= 0 && gy < Hin && gx >= 0 && gx < Win) v = plane[(long long)gy * Win + gx];
            s_in[idx] = v;
        }
        for (int idx = tid; idx < n_w; idx += CONV_THREADS) {
            int o = idx % OT;
            int t = idx / OT;
            int i = t / l, j = t - (t / l) * l;
            int q = q0 + o;
            T v = T(0);
            if (q < Q) {
                if (!BWD)
                    v = wt[(((long long)q * R + r) * l + i) * l + j];
                else  // w has shape (R=cout, Q=cin, l, l); rotated by 180 degrees
                    v = wt[(((long long)r * Q + q) * l + (l - 1 - i)) * l + (l - 1 - j)];
            }
            s_w[t * OT + o] = v;
        }
        __syncthreads();
        for (int i = 0; i < l; ++i) {
            const T *srow = s_in + i * band + (warp * CONV_RPT) * SW + lane;
            for (int j = 0; j < l; ++j) {
                const T *wv = s_w + (i * l + j) * OT;
                T xv[CONV_RPT];
#pragma unroll
                for (int rr = 0; rr < CONV_RPT; ++rr) xv[rr] = srow[rr * SW + j * d];
#pragma unroll
                for (int o = 0; o < OT; ++o) {
                    T wo = wv[o];
#pragma unroll
                    for (int rr = 0; rr < CONV_RPT; ++rr)
                        acc[o][rr] = add_rn(acc[o][rr], mul_rn(wo, xv[rr]));
                }
            }
        }
    }

    const int v = v0 + lane;
    if (v >= Wo) return;
    T *out_img = out + img * (long long)Q * Ho * Wo;
    const T *gate_img = gate ? gate + img * (long long)Q * Ho * Wo : nullptr;
#pragma unroll
    for (int o = 0; o < OT; ++o) {
        int q = q0 + o;
        if (q >= Q) break;
#pragma unroll
        for (int rr = 0; rr < CONV_RPT; ++rr) {
            int u = u0 + warp * CONV_RPT + rr;
            if (u >= Ho) break;
            long long off = ((long long)q * Ho + u) * Wo + v;
            T val = acc[o][rr];
            if (!BWD)
                val = apply_nonlin(val, act);
            else if (gate_img)
                val = gate_from_output(val, gate_img[off], gate_kind);
            out_img[off] = val;
        }
    }
}

template <typename T, int OT, bool BWD>
static int launch_conv(const T *in, const T *wt, const T *bias, T *out, const T *gate, int n,
                       int R, int Q, int Hin, int Win, int Ho, int Wo, int l, int d, int pad,
                       int act, int gate_kind, cudaStream_t st) {
    int SW = CONV_TW + (l - 1) * d;
    size_t smem = ((size_t)l * l * OT + (size_t)l * CONV_TH * SW) * sizeof(T);
    if (smem > 227 * 1024)
        return set_error(DP_ERR_UNSUPPORTED,
                         "conv: staged tile needs %zu bytes of shared memory (k=%d d=%d)", smem,
                         l, d);
    auto kern = conv_direct_kernel<T, OT, BWD>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess)
            return set_error(DP_ERR_CUDA, "conv: cudaFuncSetAttribute: %s",
                             cudaGetErrorString(e));
    }
    int tiles_x = ceil_div(Wo, CONV_TW);
    int tiles_y = ceil_div(Ho, CONV_TH);
    dim3 grid(tiles_x * tiles_y, ceil_div(Q, OT), n);
    if (grid.y > 65535 || n > 65535)
        return set_error(DP_ERR_UNSUPPORTED, "conv: grid too large");
    kern<<<grid, CONV_THREADS, smem, st>>>(in, wt, bias, out, gate, R, Q, Hin, Win, Ho, Wo, l,
                                           d, pad, act, gate_kind, tiles_x);
    return check_launch("conv_direct_kernel");
}

template <typename T, bool BWD>
static int dispatch_ot(const T *in, const T *wt, const T *bias, T *out, const T *gate, int n,
                       int R, int Q, int Hin, int Win, int Ho, int Wo, int l, int d, int pad,
                       int act, int gate_kind, cudaStream_t st) {
    if (Q <= 4)
        return launch_conv<T, 4, BWD>(in, wt, bias, out, gate, n, R, Q, Hin, Win, Ho, Wo, l, d,
                                      pad, act, gate_kind, st);
    if (Q <= 8)
        return launch_conv<T, 8, BWD>(in, wt, bias, out, gate, n, R, Q, Hin, Win, Ho, Wo, l, d,
                                      pad, act, gate_kind, st);
    return launch_conv<T, 16, BWD>(in, wt, bias, out, gate, n, R, Q, Hin, Win, Ho, Wo, l, d,
                                   pad, act, gate_kind, st);
}

template <typename T>
int conv_forward_t(const T *x, const T *w, const T *b, T *y, int n, int cin, int h, int wd,
                   int cout, int k, int d, int act, cudaStream_t st) {
    int e = (k - 1) * d + 1;
    return dispatch_ot<T, false>(x, w, b, y, nullptr, n, cin, cout, h, wd, h - e + 1,
                                 wd - e + 1, k, d, 0, act, 0, st);
}

template <typename T>
int conv_backward_data_t(const T *dy, const T *w, T *dx, int n, int cout, int ho, int wo,
                         int cin, int k, int d, const T *gate, int gate_kind, cudaStream_t st) {
    int e = (k - 1) * d + 1;
    return dispatch_ot<T, true>(dy, w, nullptr, dx, gate, n, cout, cin, ho, wo, ho + e - 1,
                                wo + e - 1, k, d, e - 1, 0, gate_kind, st);
}

template int conv_forward_t<float>(const float *, const float *, const float *, float *, int,
                                   int, int, int, int, int, int, int, cudaStream_t);
template int conv_forward_t<double>(const double *, const double *, const double *, double *,
                                    int, int, int, int, int, int, int, int, cudaStream_t);
template int conv_backward_data_t<float>(const float *, const float *, float *, int, int, int,
                                         int, int, int, int, const float *, int, cudaStream_t);
template int conv_backward_data_t<double>(const double *, const double *, double *, int, int,
                                          int, int, int, int, int, const double *, int,
                                          cudaStream_t);

}  // namespace dp
