// extern "C" entry points declared in include/denseprop_b200.h.
//
// Argument validation mirrors the reference wrappers (forward.py:27-38,
// backward.py:136-146, 154-155): bad shapes are rejected before any launch
// with DP_ERR_ARG and a message in dp_last_error().  The dp_host_* forms are
// the drop-in replacements for the 7 `backend.kernels()` functions: they copy
// host buffers to the device on a per-thread stream, run the batched kernel
// with n = 1, copy the result back and synchronise.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "dp_common.cuh"

namespace dp {
size_t ws_workspace_f16(int n, int cin, int hi, int wi, int cout, int k, int d);
int tc_split_f16_launch(const float *x, void *hi, void *lo, void *hs, void *ls, int shift,
                        long long rows, int w, int wp, cudaStream_t st);
int maxpool_forward_stream(const float *x, float *y, void *arg, int arg_bytes, long long planes,
                           int h, int w, int p, int d, int act, cudaStream_t st, void *yh,
                           void *yl, int yp);
int ws_shift_f16(int n, int cin, int hi, int wi, int cout, int k, int d);
int ws_conv_backward_kernel_f16(const float *x, size_t x_slack, const void *x_hi,
                                const void *x_lo, const void *x_hi_s, const void *x_lo_s,
                                size_t xh_slack, int xh_pitch, const float *dy, int dy_pitch,
                                float *dw, float *db, int n, int cin, int hi, int wi, int cout,
                                int k, int d, void *ws, size_t ws_bytes, cudaStream_t st);

// ---- kernels (defined in conv_direct.cu, conv_wgrad.cu, pool.cu, elementwise.cu)
template <typename T>
int conv_forward_t(const T *, const T *, const T *, T *, int, int, int, int, int, int, int, int,
                   cudaStream_t);
template <typename T>
int conv_backward_data_t(const T *, const T *, T *, int, int, int, int, int, int, int,
                         const T *, int, cudaStream_t);
template <typename T>
int conv_backward_kernel_t(const T *, const T *, T *, T *, int, int, int, int, int, int, int,
                           void *, size_t, cudaStream_t);
size_t wgrad_workspace_bytes(int elem, int n, int cin, int hi, int wi, int cout, int k, int d);
template <typename T>
int conv_backward_kernel_seq_t(const T *x, const T *dy, T *dw, T *db, int cin, int hi, int wi,
                               int cout, int k, int d, cudaStream_t st);
size_t tc_conv_workspace(int R, int Q, int l);
size_t tc_conv_fwd_workspace(int n, int cin, int h, int w, int cout, int k, int d);
size_t tc_conv_bwd_workspace(int n, int cout, int ho, int wo, int cin, int k, int d);
bool tc_conv_supported(int R, int Q, int l, int d);
int tc_conv_forward(const float *, const float *, const float *, float *, int, int, int, int, int,
                    int, int, int, void *, size_t, cudaStream_t, int flags);
int tc_conv_backward_data(const float *, const float *, float *, int, int, int, int, int, int,
                          int, const float *, int, void *, size_t, cudaStream_t);
bool tc_wgrad_supported(int, int, int, int, int, int, int);
int wg_trace_copy(void *, size_t);
int tc_trace_copy(void *, size_t);
int ws_debug_plan(int n, int cin, int hi, int wi, int cout, int k, int d, int *out, int len);
size_t tc_wgrad_workspace(int, int, int, int, int, int, int);
int tc_wgrad_prepare(const float *, int, int, int, int, int, int, int, void *, size_t,
                     cudaStream_t);
int tc_conv_backward_kernel_staged(const float *, const float *, float *, float *, int, int, int,
                                   int, int, int, int, void *, size_t, cudaStream_t);
int tc_conv_backward_kernel(const float *, const float *, float *, float *, int, int, int, int,
                            int, int, int, void *, size_t, cudaStream_t, size_t, int);
template <typename T>
int maxpool_forward_t(const T *, T *, void *, int, int, int, int, int, int, int, int,
                      cudaStream_t);
template <typename T>
int maxpool_backward_t(const T *, const void *, int, T *, int, int, int, int, int, int, int,
                       int, const T *, int, cudaStream_t, int);
template <typename T>
int avgpool_forward_t(const T *, T *, int, int, int, int, int, int, int, cudaStream_t);
template <typename T>
int avgpool_backward_t(const T *, T *, int, int, int, int, int, int, int, int, const T *, int,
                       cudaStream_t);
template <typename T>
int nonlin_forward_t(const T *, T *, long long, int, cudaStream_t);
template <typename T>
int nonlin_backward_t(const T *, const T *, T *, long long, int, int, cudaStream_t);
template <typename T>
int mask_delta_t(const T *, const T *, const uint8_t *, T *, int, int, int, int, cudaStream_t);
template <typename T>
int pad_t(const T *, T *, int, int, int, int, int, int, int, int, cudaStream_t);
template <typename T>
int patch_gather_t(const T *x0, T *out, int C, int Hp, int Wp, int P, int w, long long first,
                   long long count, cudaStream_t st);
template <typename T>
int softmax_xent_t(const T *logits, const uint8_t *labels, const uint8_t *mask, T *delta, T *loss,
                   int n, int q, int h, int w, cudaStream_t st);
template <typename T>
int crop_t(const T *, T *, int, int, int, int, int, int, int, int, cudaStream_t);
template <typename T>
int sgd_t(T *, const T *, long long, double, cudaStream_t);

// ---- error state
static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(DP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return DP_OK;
}

static int cuda_ok(cudaError_t e, const char *what) {
    if (e != cudaSuccess) return set_error(DP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return DP_OK;
}

static inline int esize(int dtype) { return dtype == DP_F64 ? 8 : 4; }

static int check_dtype(int dtype) {
    if (dtype != DP_F32 && dtype != DP_F64)
        return set_error(DP_ERR_ARG, "dtype must be DP_F32 or DP_F64, got %d", dtype);
    return DP_OK;
}

static int check_pos(const char *what, long long v) {
    if (v < 1) return set_error(DP_ERR_ARG, "%s must be >= 1, got %lld", what, v);
    return DP_OK;
}

static int check_nonlin(int kind) {
    if (kind < DP_IDENTITY || kind > DP_TANH_FAST)
        return set_error(DP_ERR_ARG, "unknown nonlinearity code %d", kind);
    return DP_OK;
}

#define DP_TRY(expr)            \
    do {                        \
        int _rc = (expr);       \
        if (_rc) return _rc;    \
    } while (0)

static int check_window(const char *what, int h, int w, int k, int d) {
    DP_TRY(check_pos("kernel size", k));
    DP_TRY(check_pos("dilation", d));
    long long e = (long long)(k - 1) * d + 1;
    if (h < e || w < e)
        return set_error(DP_ERR_ARG, "%s: input %dx%d is smaller than the %lldx%lld dilated window",
                         what, h, w, e, e);
    return DP_OK;
}

// ---- per-thread stream + scratch for the host-pointer forms
struct HostCtx {
    cudaStream_t st = nullptr;
    ~HostCtx() {
        if (st) cudaStreamDestroy(st);
    }
};
static thread_local HostCtx g_host;

static int host_stream(cudaStream_t *out) {
    if (!g_host.st) DP_TRY(cuda_ok(cudaStreamCreateWithFlags(&g_host.st, cudaStreamNonBlocking),
                                   "cudaStreamCreate"));
    *out = g_host.st;
    return DP_OK;
}

struct DevBufs {
    cudaStream_t st;
    void *p[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int n = 0;
    explicit DevBufs(cudaStream_t s) : st(s) {}
    ~DevBufs() {
        for (int i = 0; i < n; ++i)
            if (p[i]) cudaFreeAsync(p[i], st);
        cudaStreamSynchronize(st);
    }
    int alloc(size_t bytes, void **out) {
        void *q = nullptr;
        DP_TRY(cuda_ok(cudaMallocAsync(&q, bytes ? bytes : 1, st), "cudaMallocAsync"));
        p[n++] = q;
        *out = q;
        return DP_OK;
    }
    int up(const void *host, size_t bytes, void **out) {
        DP_TRY(alloc(bytes, out));
        return cuda_ok(cudaMemcpyAsync(*out, host, bytes, cudaMemcpyHostToDevice, st), "H2D");
    }
};

static int down(void *host, const void *dev, size_t bytes, cudaStream_t st) {
    DP_TRY(cuda_ok(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st), "D2H"));
    return DP_OK;
}

static int finish(cudaStream_t st) { return cuda_ok(cudaStreamSynchronize(st), "sync"); }

#define DP_DISPATCH(dtype, CALL_F, CALL_D) ((dtype) == DP_F64 ? (CALL_D) : (CALL_F))

}  // namespace dp

using namespace dp;

extern "C" {

const char *dp_last_error(void) { return g_err; }
int dp_abi_version(void) { return DP_ABI_VERSION; }
int dp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return n;
}

// ============================== device-pointer forms ==============================

int dp_conv_forward(int dtype, const void *x, const void *wt, const void *b, void *y, int n,
                    int cin, int h, int w, int cout, int k, int d, int nonlin, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_nonlin(nonlin));
    DP_TRY(check_window("dilated conv", h, w, k, d));
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       conv_forward_t<float>((const float *)x, (const float *)wt,
                                             (const float *)b, (float *)y, n, cin, h, w, cout,
                                             k, d, nonlin, st),
                       conv_forward_t<double>((const double *)x, (const double *)wt,
                                              (const double *)b, (double *)y, n, cin, h, w,
                                              cout, k, d, nonlin, st));
}

int dp_conv_backward_data(int dtype, const void *dy, const void *wt, void *dx, int n, int cout,
                          int ho, int wo, int cin, int k, int d, const void *gate,
                          int gate_kind, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("delta height", ho));
    DP_TRY(check_pos("delta width", wo));
    DP_TRY(check_pos("kernel size", k));
    DP_TRY(check_pos("dilation", d));
    DP_TRY(check_nonlin(gate_kind));
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       conv_backward_data_t<float>((const float *)dy, (const float *)wt,
                                                   (float *)dx, n, cout, ho, wo, cin, k, d,
                                                   (const float *)gate, gate_kind, st),
                       conv_backward_data_t<double>((const double *)dy, (const double *)wt,
                                                    (double *)dx, n, cout, ho, wo, cin, k, d,
                                                    (const double *)gate, gate_kind, st));
}

size_t dp_conv_fast_workspace(int reduce_channels, int out_channels, int k) {
    if (reduce_channels < 1 || out_channels < 1 || k < 1) return 0;
    return tc_conv_workspace(reduce_channels, out_channels, k);
}

size_t dp_conv_forward_fast_workspace(int n, int cin, int h, int w, int cout, int k, int d) {
    if (n < 1 || cin < 1 || cout < 1 || check_window("dilated conv", h, w, k, d)) return 0;
    return tc_conv_fwd_workspace(n, cin, h, w, cout, k, d);
}

size_t dp_conv_backward_data_fast_workspace(int n, int cout, int ho, int wo, int cin, int k,
                                            int d) {
    if (n < 1 || cin < 1 || cout < 1 || ho < 1 || wo < 1 || k < 1 || d < 1) return 0;
    return tc_conv_bwd_workspace(n, cout, ho, wo, cin, k, d);
}

int dp_conv_fast_supported(int reduce_channels, int out_channels, int k, int d) {
    if (reduce_channels < 1 || out_channels < 1 || k < 1 || d < 1) return 0;
    return tc_conv_supported(reduce_channels, out_channels, k, d) ? 1 : 0;
}

int dp_conv_forward_fast(const float *x, const float *wt, const float *b, float *y, int n,
                         int cin, int h, int w, int cout, int k, int d, int nonlin,
                         void *workspace, size_t workspace_bytes, void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_nonlin(nonlin));
    DP_TRY(check_window("dilated conv", h, w, k, d));
    return tc_conv_forward(x, wt, b, y, n, cin, h, w, cout, k, d, nonlin, workspace,
                           workspace_bytes, (cudaStream_t)stream, 0);
}

int dp_conv_forward_fast_ex(const float *x, const float *wt, const float *b, float *y, int n,
                            int cin, int h, int w, int cout, int k, int d, int nonlin, int flags,
                            void *workspace, size_t workspace_bytes, void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_nonlin(nonlin));
    DP_TRY(check_window("dilated conv", h, w, k, d));
    return tc_conv_forward(x, wt, b, y, n, cin, h, w, cout, k, d, nonlin, workspace,
                           workspace_bytes, (cudaStream_t)stream, flags);
}

int dp_conv_backward_data_fast(const float *dy, const float *wt, float *dx, int n, int cout,
                               int ho, int wo, int cin, int k, int d, const float *gate,
                               int gate_kind, void *workspace, size_t workspace_bytes,
                               void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("delta height", ho));
    DP_TRY(check_pos("delta width", wo));
    DP_TRY(check_pos("kernel size", k));
    DP_TRY(check_pos("dilation", d));
    DP_TRY(check_nonlin(gate_kind));
    return tc_conv_backward_data(dy, wt, dx, n, cout, ho, wo, cin, k, d, gate, gate_kind,
                                 workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t dp_conv_backward_kernel_workspace(int dtype, int n, int cin, int hi, int wi, int cout,
                                         int k, int d) {
    if (check_dtype(dtype) || n < 1 || cin < 1 || cout < 1 || check_window("wgrad", hi, wi, k, d))
        return 0;
    return wgrad_workspace_bytes(esize(dtype), n, cin, hi, wi, cout, k, d);
}

int dp_conv_backward_kernel(int dtype, const void *x, const void *dy, void *dw, void *db, int n,
                            int cin, int hi, int wi, int cout, int k, int d, void *workspace,
                            size_t workspace_bytes, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("conv backward kernel", hi, wi, k, d));
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(
        dtype,
        conv_backward_kernel_t<float>((const float *)x, (const float *)dy, (float *)dw,
                                      (float *)db, n, cin, hi, wi, cout, k, d, workspace,
                                      workspace_bytes, st),
        conv_backward_kernel_t<double>((const double *)x, (const double *)dy, (double *)dw,
                                       (double *)db, n, cin, hi, wi, cout, k, d, workspace,
                                       workspace_bytes, st));
}

int dp_conv_backward_kernel_fast_supported(int n, int cin, int hi, int wi, int cout, int k,
                                           int d) {
    if (n < 1 || cin < 1 || cout < 1 || check_window("wgrad", hi, wi, k, d)) return 0;
    return tc_wgrad_supported(n, cin, hi, wi, cout, k, d) ? 1 : 0;
}

size_t dp_conv_backward_kernel_fast_workspace(int n, int cin, int hi, int wi, int cout, int k,
                                              int d) {
    if (n < 1 || cin < 1 || cout < 1 || check_window("wgrad", hi, wi, k, d)) return 0;
    return tc_wgrad_workspace(n, cin, hi, wi, cout, k, d);
}

int dp_debug_wgrad_trace(void *host, size_t bytes) { return wg_trace_copy(host, bytes); }
int dp_debug_wgrad_plan(int n, int cin, int hi, int wi, int cout, int k, int d, int *out,
                        int len) {
    return ws_debug_plan(n, cin, hi, wi, cout, k, d, out, len);
}
int dp_debug_conv_trace(void *host, size_t bytes) { return tc_trace_copy(host, bytes); }

int dp_conv_backward_kernel_fast(const float *x, const float *dy, float *dw, float *db, int n,
                                 int cin, int hi, int wi, int cout, int k, int d,
                                 void *workspace, size_t workspace_bytes, void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("conv backward kernel", hi, wi, k, d));
    return tc_conv_backward_kernel(x, dy, dw, db, n, cin, hi, wi, cout, k, d, workspace,
                                   workspace_bytes, (cudaStream_t)stream, 0, 0);
}

int dp_conv_backward_kernel_fast_ex(const float *x, size_t x_slack_bytes, const float *dy,
                                    int dy_pitch, float *dw, float *db, int n, int cin, int hi,
                                    int wi, int cout, int k, int d, void *workspace,
                                    size_t workspace_bytes, void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("conv backward kernel", hi, wi, k, d));
    const int wo = wi - (k - 1) * d;
    if (dy_pitch != 0 && dy_pitch < wo)
        return set_error(DP_ERR_ARG, "dy row pitch %d < width %d", dy_pitch, wo);
    return tc_conv_backward_kernel(x, dy, dw, db, n, cin, hi, wi, cout, k, d, workspace,
                                   workspace_bytes, (cudaStream_t)stream, x_slack_bytes,
                                   dy_pitch);
}


size_t dp_conv_backward_kernel_fast_f16_workspace(int n, int cin, int hi, int wi, int cout,
                                                  int k, int d) {
    if (n < 1 || cin < 1 || cout < 1 || k < 1 || d < 1 || hi < (k - 1) * d + 1 ||
        wi < (k - 1) * d + 1)
        return 0;
    return dp::ws_workspace_f16(n, cin, hi, wi, cout, k, d);
}

int dp_conv_backward_kernel_fast_f16(const float *x, size_t x_slack_bytes, const void *x_hi,
                                     const void *x_lo, const void *x_hi_s, const void *x_lo_s,
                                     size_t xh_slack_bytes, int xh_pitch, const float *dy,
                                     int dy_pitch, float *dw, float *db, int n, int cin, int hi,
                                     int wi, int cout, int k, int d, void *workspace,
                                     size_t workspace_bytes, void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("conv backward kernel", hi, wi, k, d));
    const int wo = wi - (k - 1) * d;
    if (dy_pitch != 0 && dy_pitch < wo)
        return set_error(DP_ERR_ARG, "dy row pitch %d < width %d", dy_pitch, wo);
    return dp::ws_conv_backward_kernel_f16(x, x_slack_bytes, x_hi, x_lo, x_hi_s, x_lo_s,
                                           xh_slack_bytes, xh_pitch, dy,
                                           dy_pitch, dw, db, n, cin, hi, wi, cout, k, d,
                                           workspace, workspace_bytes, (cudaStream_t)stream);
}

int dp_split_f16(const float *x, void *x_hi, void *x_lo, void *x_hi_s, void *x_lo_s,
                 int shift, int64_t rows, int w, int pitch, void *stream) {
    if (rows < 0 || w < 1) return set_error(DP_ERR_ARG, "fp16 split: bad rows %lld / width %d",
                                            (long long)rows, w);
    return dp::tc_split_f16_launch(x, x_hi, x_lo, x_hi_s, x_lo_s, shift, rows, w, pitch,
                                   (cudaStream_t)stream);
}

int dp_maxpool_forward_split(const float *x, float *y, void *arg, int n, int c, int h, int w,
                             int p, int d, int nonlin, void *y_hi, void *y_lo, int y_pitch,
                             void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_nonlin(nonlin));
    DP_TRY(check_window("dilated max pool", h, w, p, d));
    if (p * p > 256) return set_error(DP_ERR_ARG, "split pool forward: uint8 codes need p*p <= 256");
    const int ho = h - (p - 1) * d, wo = w - (p - 1) * d;
    cudaStream_t st = (cudaStream_t)stream;
    // fused: the warp-streaming kernel writes the split with the output
    const int rc = dp::maxpool_forward_stream(x, y, arg, 1, (long long)n * c, h, w, p, d, nonlin,
                                              st, y_hi, y_lo, y_pitch);
    if (rc >= 0) return rc;
    DP_TRY(maxpool_forward_t<float>(x, y, arg, 1, n, c, h, w, p, d, nonlin, st));
    return dp::tc_split_f16_launch(y, y_hi, y_lo, nullptr, nullptr, 0, (long long)n * c * ho, wo,
                                   y_pitch, st);
}

int dp_conv_backward_kernel_fast_f16_shift(int n, int cin, int hi, int wi, int cout, int k,
                                           int d) {
    if (n < 1 || cin < 1 || cout < 1 || k < 1 || d < 1 || hi < (k - 1) * d + 1 ||
        wi < (k - 1) * d + 1)
        return -1;
    return dp::ws_shift_f16(n, cin, hi, wi, cout, k, d);
}

int dp_conv_backward_kernel_fast_prepare(const float *x, int n, int cin, int hi, int wi,
                                         int cout, int k, int d, void *workspace,
                                         size_t workspace_bytes, void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("conv backward kernel", hi, wi, k, d));
    return tc_wgrad_prepare(x, n, cin, hi, wi, cout, k, d, workspace, workspace_bytes,
                            (cudaStream_t)stream);
}

int dp_conv_backward_kernel_fast_staged(const float *x, const float *dy, float *dw, float *db,
                                        int n, int cin, int hi, int wi, int cout, int k, int d,
                                        void *workspace, size_t workspace_bytes, void *stream) {
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("conv backward kernel", hi, wi, k, d));
    return tc_conv_backward_kernel_staged(x, dy, dw, db, n, cin, hi, wi, cout, k, d, workspace,
                                          workspace_bytes, (cudaStream_t)stream);
}

int dp_maxpool_forward(int dtype, const void *x, void *y, void *arg, int arg_bytes, int n, int c,
                       int h, int w, int p, int d, int nonlin, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_nonlin(nonlin));
    DP_TRY(check_window("dilated max pool", h, w, p, d));
    if (arg_bytes != 4 && !(arg_bytes == 1 && p * p <= 256))
        return set_error(DP_ERR_ARG, "arg_bytes must be 4 (or 1 when p*p <= 256)");
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       maxpool_forward_t<float>((const float *)x, (float *)y, arg, arg_bytes, n,
                                                c, h, w, p, d, nonlin, st),
                       maxpool_forward_t<double>((const double *)x, (double *)y, arg, arg_bytes,
                                                 n, c, h, w, p, d, nonlin, st));
}

static int check_pool_bwd(int ho, int wo, int p, int d, int hi, int wi) {
    DP_TRY(check_pos("delta height", ho));
    DP_TRY(check_pos("delta width", wo));
    DP_TRY(check_pos("pool size", p));
    DP_TRY(check_pos("dilation", d));
    long long e = (long long)(p - 1) * d + 1;
    if (hi < ho + e - 1 || wi < wo + e - 1)
        return set_error(DP_ERR_ARG, "pool backward: input %dx%d smaller than %lldx%lld", hi, wi,
                         ho + e - 1, wo + e - 1);
    return DP_OK;
}

int dp_maxpool_backward(int dtype, const void *dy, const void *arg, int arg_bytes, void *dx,
                        int n, int c, int ho, int wo, int p, int d, int hi, int wi,
                        const void *gate, int gate_kind, void *stream) {
    return dp_maxpool_backward_pitched(dtype, dy, arg, arg_bytes, dx, wi, n, c, ho, wo, p, d,
                                       hi, wi, gate, gate_kind, stream);
}

int dp_maxpool_backward_pitched(int dtype, const void *dy, const void *arg, int arg_bytes,
                                void *dx, int dx_pitch, int n, int c, int ho, int wo, int p,
                                int d, int hi, int wi, const void *gate, int gate_kind,
                                void *stream) {
    DP_TRY(check_dtype(dtype));
    if (dx_pitch < wi) return set_error(DP_ERR_ARG, "dx row pitch %d < width %d", dx_pitch, wi);
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_nonlin(gate_kind));
    DP_TRY(check_pool_bwd(ho, wo, p, d, hi, wi));
    if (arg_bytes != 4 && arg_bytes != 1)
        return set_error(DP_ERR_ARG, "arg_bytes must be 1 or 4");
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       maxpool_backward_t<float>((const float *)dy, arg, arg_bytes, (float *)dx,
                                                 n, c, ho, wo, p, d, hi, wi,
                                                 (const float *)gate, gate_kind, st, dx_pitch),
                       maxpool_backward_t<double>((const double *)dy, arg, arg_bytes,
                                                  (double *)dx, n, c, ho, wo, p, d, hi, wi,
                                                  (const double *)gate, gate_kind, st,
                                                  dx_pitch));
}

int dp_avgpool_forward(int dtype, const void *x, void *y, int n, int c, int h, int w, int p,
                       int d, int nonlin, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_nonlin(nonlin));
    DP_TRY(check_window("dilated avg pool", h, w, p, d));
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       avgpool_forward_t<float>((const float *)x, (float *)y, n, c, h, w, p, d,
                                                nonlin, st),
                       avgpool_forward_t<double>((const double *)x, (double *)y, n, c, h, w, p,
                                                 d, nonlin, st));
}

int dp_avgpool_backward(int dtype, const void *dy, void *dx, int n, int c, int ho, int wo, int p,
                        int d, int hi, int wi, const void *gate, int gate_kind, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_nonlin(gate_kind));
    DP_TRY(check_pool_bwd(ho, wo, p, d, hi, wi));
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       avgpool_backward_t<float>((const float *)dy, (float *)dx, n, c, ho, wo, p,
                                                 d, hi, wi, (const float *)gate, gate_kind, st),
                       avgpool_backward_t<double>((const double *)dy, (double *)dx, n, c, ho, wo,
                                                  p, d, hi, wi, (const double *)gate,
                                                  gate_kind, st));
}

int dp_nonlin_forward(int dtype, const void *x, void *y, int64_t count, int kind, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_nonlin(kind));
    if (count < 0) return set_error(DP_ERR_ARG, "count must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       nonlin_forward_t<float>((const float *)x, (float *)y, count, kind, st),
                       nonlin_forward_t<double>((const double *)x, (double *)y, count, kind,
                                                st));
}

int dp_nonlin_backward(int dtype, const void *dy, const void *x, void *dx, int64_t count,
                       int kind, int x_is_output, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_nonlin(kind));
    if (count < 0) return set_error(DP_ERR_ARG, "count must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       nonlin_backward_t<float>((const float *)dy, (const float *)x,
                                                (float *)dx, count, kind, x_is_output, st),
                       nonlin_backward_t<double>((const double *)dy, (const double *)x,
                                                 (double *)dx, count, kind, x_is_output, st));
}

int dp_mask_delta(int dtype, const void *a, const void *target, const uint8_t *mask, void *out,
                  int n, int c, int h, int w, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_pos("height", h));
    DP_TRY(check_pos("width", w));
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       mask_delta_t<float>((const float *)a, (const float *)target, mask,
                                           (float *)out, n, c, h, w, st),
                       mask_delta_t<double>((const double *)a, (const double *)target, mask,
                                            (double *)out, n, c, h, w, st));
}

int dp_pad(int dtype, const void *src, void *dst, int n, int c, int h, int w, int top,
           int bottom, int left, int right, void *stream) {
    DP_TRY(check_dtype(dtype));
    if (top < 0 || bottom < 0 || left < 0 || right < 0)
        return set_error(DP_ERR_ARG, "padding margins must be >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       pad_t<float>((const float *)src, (float *)dst, n, c, h, w, top, bottom,
                                    left, right, st),
                       pad_t<double>((const double *)src, (double *)dst, n, c, h, w, top,
                                     bottom, left, right, st));
}

int dp_crop(int dtype, const void *src, void *dst, int n, int c, int hs, int ws, int top,
            int left, int h, int w, void *stream) {
    DP_TRY(check_dtype(dtype));
    if (top < 0 || left < 0 || top + h > hs || left + w > ws)
        return set_error(DP_ERR_ARG, "crop window leaves the %dx%d map", hs, ws);
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       crop_t<float>((const float *)src, (float *)dst, n, c, hs, ws, top, left,
                                     h, w, st),
                       crop_t<double>((const double *)src, (double *)dst, n, c, hs, ws, top,
                                      left, h, w, st));
}

int dp_softmax_xent_delta(int dtype, const void *logits, const uint8_t *labels,
                          const uint8_t *mask, void *delta, void *loss, int n, int q, int h, int w,
                          void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("batch", n));
    DP_TRY(check_pos("classes", q));
    DP_TRY(check_pos("height", h));
    DP_TRY(check_pos("width", w));
    if (q > 255) return set_error(DP_ERR_ARG, "softmax xent: at most 255 classes (uint8 labels)");
    if (!logits || !labels || !delta) return set_error(DP_ERR_ARG, "softmax xent: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       softmax_xent_t<float>((const float *)logits, labels, mask, (float *)delta,
                                             (float *)loss, n, q, h, w, st),
                       softmax_xent_t<double>((const double *)logits, labels, mask,
                                              (double *)delta, (double *)loss, n, q, h, w, st));
}

int dp_patch_gather(int dtype, const void *x0, void *out, int c, int hp, int wp, int patch,
                    int w, int64_t first, int64_t count, void *stream) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_pos("patch", patch));
    DP_TRY(check_pos("width", w));
    const int h = hp - patch + 1;
    if (h < 1 || wp - patch + 1 != w)
        return set_error(DP_ERR_ARG, "patch gather: padded map %dx%d does not fit patch %d / width %d",
                         hp, wp, patch, w);
    if (first < 0 || count < 0 || first + count > (int64_t)h * w)
        return set_error(DP_ERR_ARG, "patch gather: pixel range outside the %dx%d grid", h, w);
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype,
                       patch_gather_t<float>((const float *)x0, (float *)out, c, hp, wp, patch, w,
                                             first, count, st),
                       patch_gather_t<double>((const double *)x0, (double *)out, c, hp, wp,
                                              patch, w, first, count, st));
}

int dp_sgd_update(int dtype, void *param, const void *grad, int64_t count, double lr,
                  void *stream) {
    DP_TRY(check_dtype(dtype));
    cudaStream_t st = (cudaStream_t)stream;
    return DP_DISPATCH(dtype, sgd_t<float>((float *)param, (const float *)grad, count, lr, st),
                       sgd_t<double>((double *)param, (const double *)grad, count, lr, st));
}

// ============================== host-pointer forms ==============================

int dp_host_conv_forward(int dtype, const void *x, const void *wt, const void *b, void *y,
                         int cin, int h, int w, int cout, int k, int d) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("dilated conv", h, w, k, d));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t es = esize(dtype);
    int e = (k - 1) * d + 1, ho = h - e + 1, wo = w - e + 1;
    int rc;
    {
        DevBufs B(st);
        void *dx, *dw, *db, *dy;
        DP_TRY(B.up(x, es * cin * h * w, &dx));
        DP_TRY(B.up(wt, es * cout * cin * k * k, &dw));
        DP_TRY(B.up(b, es * cout, &db));
        DP_TRY(B.alloc(es * (size_t)cout * ho * wo, &dy));
        rc = dp_conv_forward(dtype, dx, dw, db, dy, 1, cin, h, w, cout, k, d, DP_IDENTITY, st);
        if (!rc) rc = down(y, dy, es * (size_t)cout * ho * wo, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_conv_backward_data(int dtype, const void *dy, const void *wt, void *dx, int cout,
                               int ho, int wo, int cin, int k, int d) {
    DP_TRY(check_dtype(dtype));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t es = esize(dtype);
    int e = (k - 1) * d + 1, hi = ho + e - 1, wi = wo + e - 1;
    int rc;
    {
        DevBufs B(st);
        void *ddy, *dw, *ddx;
        DP_TRY(B.up(dy, es * cout * ho * wo, &ddy));
        DP_TRY(B.up(wt, es * cout * cin * k * k, &dw));
        DP_TRY(B.alloc(es * (size_t)cin * hi * wi, &ddx));
        rc = dp_conv_backward_data(dtype, ddy, dw, ddx, 1, cout, ho, wo, cin, k, d, nullptr,
                                   DP_IDENTITY, st);
        if (!rc) rc = down(dx, ddx, es * (size_t)cin * hi * wi, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_conv_backward_kernel(int dtype, const void *x, const void *dy, void *dw, void *db,
                                 int cin, int hi, int wi, int cout, int k, int d) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("in channels", cin));
    DP_TRY(check_pos("out channels", cout));
    DP_TRY(check_window("conv backward kernel", hi, wi, k, d));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t es = esize(dtype);
    int e = (k - 1) * d + 1, ho = hi - e + 1, wo = wi - e + 1;
    int rc;
    {
        // per-image drop-in: the reference's own summation order (bit-identical), not the
        // batched split-K kernel
        DevBufs B(st);
        void *ddx, *ddy, *ddw, *ddb;
        DP_TRY(B.up(x, es * cin * hi * wi, &ddx));
        DP_TRY(B.up(dy, es * cout * ho * wo, &ddy));
        DP_TRY(B.alloc(es * cout * cin * k * k, &ddw));
        DP_TRY(B.alloc(es * cout, &ddb));
        rc = dtype == DP_F32
                 ? conv_backward_kernel_seq_t<float>((const float *)ddx, (const float *)ddy,
                                                     (float *)ddw, (float *)ddb, cin, hi, wi, cout,
                                                     k, d, st)
                 : conv_backward_kernel_seq_t<double>((const double *)ddx, (const double *)ddy,
                                                      (double *)ddw, (double *)ddb, cin, hi, wi,
                                                      cout, k, d, st);
        if (!rc) rc = down(dw, ddw, es * cout * cin * k * k, st);
        if (!rc) rc = down(db, ddb, es * cout, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_maxpool_forward(int dtype, const void *x, void *y, int32_t *arg, int c, int h, int w,
                            int p, int d) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_window("dilated max pool", h, w, p, d));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t es = esize(dtype);
    int e = (p - 1) * d + 1, ho = h - e + 1, wo = w - e + 1;
    size_t nout = (size_t)c * ho * wo;
    int rc;
    {
        DevBufs B(st);
        void *dx, *dy, *da;
        DP_TRY(B.up(x, es * c * h * w, &dx));
        DP_TRY(B.alloc(es * nout, &dy));
        DP_TRY(B.alloc(4 * nout, &da));
        rc = dp_maxpool_forward(dtype, dx, dy, da, 4, 1, c, h, w, p, d, DP_IDENTITY, st);
        if (!rc) rc = down(y, dy, es * nout, st);
        if (!rc) rc = down(arg, da, 4 * nout, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_maxpool_backward(int dtype, const void *dy, const int32_t *arg, void *dx, int c,
                             int ho, int wo, int p, int d, int hi, int wi) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_pool_bwd(ho, wo, p, d, hi, wi));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t es = esize(dtype);
    size_t nout = (size_t)c * ho * wo, nin = (size_t)c * hi * wi;
    int rc;
    {
        DevBufs B(st);
        void *ddy, *da, *ddx;
        DP_TRY(B.up(dy, es * nout, &ddy));
        DP_TRY(B.up(arg, 4 * nout, &da));
        DP_TRY(B.alloc(es * nin, &ddx));
        rc = dp_maxpool_backward(dtype, ddy, da, 4, ddx, 1, c, ho, wo, p, d, hi, wi, nullptr,
                                 DP_IDENTITY, st);
        if (!rc) rc = down(dx, ddx, es * nin, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_avgpool_forward(int dtype, const void *x, void *y, int c, int h, int w, int p,
                            int d) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_window("dilated avg pool", h, w, p, d));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t es = esize(dtype);
    int e = (p - 1) * d + 1, ho = h - e + 1, wo = w - e + 1;
    size_t nout = (size_t)c * ho * wo;
    int rc;
    {
        DevBufs B(st);
        void *dx, *dy;
        DP_TRY(B.up(x, es * c * h * w, &dx));
        DP_TRY(B.alloc(es * nout, &dy));
        rc = dp_avgpool_forward(dtype, dx, dy, 1, c, h, w, p, d, DP_IDENTITY, st);
        if (!rc) rc = down(y, dy, es * nout, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_avgpool_backward(int dtype, const void *dy, void *dx, int c, int ho, int wo, int p,
                             int d, int hi, int wi) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_pos("channels", c));
    DP_TRY(check_pool_bwd(ho, wo, p, d, hi, wi));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t es = esize(dtype);
    size_t nout = (size_t)c * ho * wo, nin = (size_t)c * hi * wi;
    int rc;
    {
        DevBufs B(st);
        void *ddy, *ddx;
        DP_TRY(B.up(dy, es * nout, &ddy));
        DP_TRY(B.alloc(es * nin, &ddx));
        rc = dp_avgpool_backward(dtype, ddy, ddx, 1, c, ho, wo, p, d, hi, wi, nullptr,
                                 DP_IDENTITY, st);
        if (!rc) rc = down(dx, ddx, es * nin, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_nonlin_forward(int dtype, const void *x, void *y, int64_t count, int kind) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_nonlin(kind));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t bytes = esize(dtype) * (size_t)count;
    int rc;
    {
        DevBufs B(st);
        void *dx, *dy;
        DP_TRY(B.up(x, bytes, &dx));
        DP_TRY(B.alloc(bytes, &dy));
        rc = dp_nonlin_forward(dtype, dx, dy, count, kind, st);
        if (!rc) rc = down(y, dy, bytes, st);
    }
    return rc ? rc : finish(st);
}

int dp_host_nonlin_backward(int dtype, const void *dy, const void *x_in, void *dx, int64_t count,
                            int kind) {
    DP_TRY(check_dtype(dtype));
    DP_TRY(check_nonlin(kind));
    cudaStream_t st;
    DP_TRY(host_stream(&st));
    size_t bytes = esize(dtype) * (size_t)count;
    int rc;
    {
        DevBufs B(st);
        void *ddy, *dxin, *ddx;
        DP_TRY(B.up(dy, bytes, &ddy));
        DP_TRY(B.up(x_in, bytes, &dxin));
        DP_TRY(B.alloc(bytes, &ddx));
        rc = dp_nonlin_backward(dtype, ddy, dxin, ddx, count, kind, 0, st);
        if (!rc) rc = down(dx, ddx, bytes, st);
    }
    return rc ? rc : finish(st);
}

}  // extern "C"
