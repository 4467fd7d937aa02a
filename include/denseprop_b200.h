/*
 * denseprop_b200.h -- C ABI of the B200-native dense whole-image propagation
 * kernels (arXiv 1412.4526).  Library: paper_1412_4526_b200/libdenseprop_b200.so
 * (sm_100a, built by `python -m paper_1412_4526_b200.build` or
 * __graft_entry__.build()).
 *
 * Replaces the reference's single plugin boundary, `backend.kernels()`
 * (pkg/src/denseprop/backend.py:47-48), whose modules export 7 functions
 * (pkg/src/denseprop/_kernels.pyx:23-247, _kernels_py.py:19-126).  Each of
 * those gets two entry points here:
 *
 *   dp_host_<name>  -- drop-in form: HOST pointers, one (C,H,W) map, the
 *                      reference's argument meaning; synchronous.  This is what
 *                      a ctypes/cffi backend module binds.
 *   dp_<name>       -- device form: DEVICE pointers, a batch of n maps laid
 *                      out (n, C, H, W) C-contiguous, enqueued on `stream`
 *                      (a cudaStream_t; NULL = legacy default stream), with
 *                      fused nonlinearity / gate / mask options.  The batched
 *                      executor and the data-parallel trainer call these.
 *
 * Conventions
 *  - dtype: DP_F32 or DP_F64; every float argument of a call has that type
 *    (reference fused `floating` type, _kernels.pyx:18-20).  argmax maps are
 *    int32 at the host API (value i*p + j, _kernels.pyx:143,165); device calls
 *    may use 1-byte argmax (arg_bytes = 1) when p*p <= 256.
 *  - dilation d >= 1, kernel / pool size >= 1; extent e = (k-1)*d + 1.
 *  - Return value: DP_OK (0) or an error code; dp_last_error() (thread-local)
 *    describes the last failure.  Bad shapes / arguments give DP_ERR_ARG and
 *    leave outputs untouched (reference wrappers raise ValueError before
 *    dispatch: forward.py:33-38, backward.py:136-146).
 *  - Exactness: conv forward, conv data-gradient, both pools and relu are
 *    bit-identical to the reference's compiled backend in fp32 and fp64 (same
 *    per-entry operation order, no FMA contraction); tanh is within 2 ulp of
 *    numpy; weight/bias gradients are deterministic (fixed-order split
 *    reduction) and agree to reduction-order rounding.
 */
#ifndef DENSEPROP_B200_H
#define DENSEPROP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP_ABI_VERSION 6

enum dp_dtype { DP_F32 = 0, DP_F64 = 1 };
/* reference nonlin kinds, netspec.py:31 / forward.py:69-76 */
enum dp_nonlin { DP_IDENTITY = 0, DP_TANH = 1, DP_RELU = 2,
                 /* fast tier: single-precision tanhf (<= 2 ulp); DP_TANH evaluates in
                  * fp64 and rounds once so it stays within 2 ulp of numpy */
                 DP_TANH_FAST = 3 };
enum dp_status { DP_OK = 0, DP_ERR_ARG = 1, DP_ERR_CUDA = 2, DP_ERR_UNSUPPORTED = 3 };

const char *dp_last_error(void);
int dp_abi_version(void);
/* number of visible CUDA devices, or -1 if the runtime cannot be initialised */
int dp_device_count(void);

/* ======================= host-pointer drop-in entry points =======================
 * One feature map (C, H, W), C-contiguous, caller-owned input and output
 * buffers (outputs are written, never read).  Synchronous.
 */

/* replaces conv_forward(x, w, b, dilation, threads)  -- _kernels.pyx:23-53
 * x (cin,h,w), wt (cout,cin,k,k), b (cout) -> y (cout, h-e+1, w-e+1) */
int dp_host_conv_forward(int dtype, const void *x, const void *wt, const void *b, void *y,
                         int cin, int h, int w, int cout, int k, int d);

/* replaces conv_backward_data(dy, w, dilation, threads) -- _kernels.pyx:56-91
 * dy (cout,ho,wo), wt (cout,cin,k,k) -> dx (cin, ho+e-1, wo+e-1) */
int dp_host_conv_backward_data(int dtype, const void *dy, const void *wt, void *dx,
                               int cout, int ho, int wo, int cin, int k, int d);

/* replaces conv_backward_kernel(x, dy, kernel_size, dilation, threads) -- _kernels.pyx:94-130
 * x (cin,hi,wi), dy (cout,hi-e+1,wi-e+1) -> dw (cout,cin,k,k), db (cout) */
int dp_host_conv_backward_kernel(int dtype, const void *x, const void *dy, void *dw, void *db,
                                 int cin, int hi, int wi, int cout, int k, int d);

/* replaces maxpool_forward(x, p, dilation, threads) -- _kernels.pyx:133-166
 * x (c,h,w) -> y (c,ho,wo), arg int32 (c,ho,wo) */
int dp_host_maxpool_forward(int dtype, const void *x, void *y, int32_t *arg,
                            int c, int h, int w, int p, int d);

/* replaces maxpool_backward(dy, arg, p, dilation, hi, wi, threads) -- _kernels.pyx:169-191
 * requires hi >= ho+e-1, wi >= wo+e-1 (rows/cols beyond receive 0) */
int dp_host_maxpool_backward(int dtype, const void *dy, const int32_t *arg, void *dx,
                             int c, int ho, int wo, int p, int d, int hi, int wi);

/* replaces avgpool_forward(x, p, dilation, threads) -- _kernels.pyx:194-221 */
int dp_host_avgpool_forward(int dtype, const void *x, void *y, int c, int h, int w, int p, int d);

/* replaces avgpool_backward(dy, p, dilation, hi, wi, threads) -- _kernels.pyx:224-247 */
int dp_host_avgpool_backward(int dtype, const void *dy, void *dx, int c, int ho, int wo,
                             int p, int d, int hi, int wi);

/* nonlin_forward / nonlin_backward (forward.py:69-76, backward.py:172-182; numpy
 * in the reference, outside its boundary).  x_in is the nonlinearity INPUT. */
int dp_host_nonlin_forward(int dtype, const void *x, void *y, int64_t count, int kind);
int dp_host_nonlin_backward(int dtype, const void *dy, const void *x_in, void *dx,
                            int64_t count, int kind);

/* ========================= device-pointer batched entry points ====================== */

/* y[n,cout,ho,wo] = act(b + sum_{c,i,j} w * x), act = `nonlin` (DP_IDENTITY = none) */
int dp_conv_forward(int dtype, const void *x, const void *wt, const void *b, void *y,
                    int n, int cin, int h, int w, int cout, int k, int d, int nonlin,
                    void *stream);

/* dx[n,cin,ho+e-1,wo+e-1] = conv_backward_data(dy); if gate != NULL,
 * dx *= act'(.) where gate holds the OUTPUT of the nonlinearity `gate_kind`
 * that produced this conv's input (tanh' = 1 - t*t, relu' = t > 0). */
int dp_conv_backward_data(int dtype, const void *dy, const void *wt, void *dx,
                          int n, int cout, int ho, int wo, int cin, int k, int d,
                          const void *gate, int gate_kind, void *stream);

/* ---- fast tier: tcgen05 tensor cores, fp32 in/out, 3xTF32 products (~1e-7 relative
 * to fp32; the reference tolerance for this path is 1e-4).  Same argument meaning as
 * dp_conv_forward / dp_conv_backward_data; DP_F32 only.  `workspace` (16-byte
 * aligned, dp_conv_fast_workspace bytes) receives the packed hi/lo weights.  Returns
 * DP_ERR_UNSUPPORTED when the packed weights plus the input halo buffers (which grow with
 * the dilation d) exceed the kernel's shared-memory budget -- check
 * dp_conv_fast_supported(reduce, out, k, d) first; the caller then uses the exact
 * CUDA-core entry points. */
size_t dp_conv_fast_workspace(int reduce_channels, int out_channels, int k);
/* Shape-aware workspace (ABI 3): bytes for the fastest kernel of this exact call -- the
 * tap-stacked variant (all column taps of a tap row in one MMA; needs the input re-laid
 * out as 16-byte channel-quad records with hi/lo precomputed, ~4x the input map) when it
 * applies, else the packed weights only.  Passing at least this many bytes selects the
 * tap-stacked kernel; dp_conv_fast_workspace bytes still work (flat kernel). */
size_t dp_conv_forward_fast_workspace(int n, int cin, int h, int w, int cout, int k, int d);
size_t dp_conv_backward_data_fast_workspace(int n, int cout, int ho, int wo, int cin, int k,
                                            int d);
int dp_conv_fast_supported(int reduce_channels, int out_channels, int k, int d);
int dp_conv_forward_fast(const float *x, const float *wt, const float *b, float *y, int n,
                         int cin, int h, int w, int cout, int k, int d, int nonlin,
                         void *workspace, size_t workspace_bytes, void *stream);
/* Same with flags (ABI 5).  DP_FAST_INPUT_FP16_RANGE: the caller vouches that |x| stays well
 * inside the fp16 range (tanh outputs, images), which allows the fp16-split forward (hi =
 * RN_fp16(x), lo = RN_fp16(x - hi), kind::f16, fp32 accumulation: ~2^-22 relative, half the
 * operand feed of 3xTF32).  Without it (and in dp_conv_forward_fast) the forward is 3xTF32. */
/* DP_FAST_PACK_FWD (ABI 6, with DP_FAST_INPUT_FP16_RANGE): <= 8-channel inputs also take the
 * fp16 offset split (tap-packed) -- faster, slightly larger rounding; the engine sets it when
 * the conv feeds a tanh (relu nets amplify first-layer rounding into relu / argmax flips) */
enum dp_fast_flags { DP_FAST_INPUT_FP16_RANGE = 1, DP_FAST_PACK_FWD = 2 };
int dp_conv_forward_fast_ex(const float *x, const float *wt, const float *b, float *y, int n,
                            int cin, int h, int w, int cout, int k, int d, int nonlin, int flags,
                            void *workspace, size_t workspace_bytes, void *stream);
int dp_conv_backward_data_fast(const float *dy, const float *wt, float *dx, int n, int cout,
                               int ho, int wo, int cin, int k, int d, const float *gate,
                               int gate_kind, void *workspace, size_t workspace_bytes,
                               void *stream);

/* fast-tier weight/bias gradient: tcgen05 implicit GEMM (M = taps x channels, N = cout,
 * K = pixels of all n images), operands staged by TMA, 3xTF32 products, split-K over
 * the SMs with a fixed-order reduction (deterministic).  Same argument meaning as
 * dp_conv_backward_kernel; DP_F32 only; cout <= 128.  `workspace` must be 256-byte
 * aligned and hold dp_conv_backward_kernel_fast_workspace bytes. */
int dp_conv_backward_kernel_fast_supported(int n, int cin, int hi, int wi, int cout, int k,
                                           int d);
size_t dp_conv_backward_kernel_fast_workspace(int n, int cin, int hi, int wi, int cout, int k,
                                              int d);
int dp_conv_backward_kernel_fast(const float *x, const float *dy, float *dw, float *db, int n,
                                 int cin, int hi, int wi, int cout, int k, int d,
                                 void *workspace, size_t workspace_bytes, void *stream);
/* Same, where the caller guarantees x_slack_bytes readable bytes after x's last element
 * (ABI 5): when every tap offset is a multiple of 4 floats and W % 4 == 0 the kernel then
 * reads x in place through a 5-D tensor map (overlapping tap view: it may touch up to
 * ((taps-1)*d + 32) * 4 bytes past the end) instead of staging a re-laid-out copy.
 * dy_pitch: dy's row pitch in elements (0 = wo); a multiple of 4 lets the kernel read dy
 * in place where it would otherwise re-pitch it. */
int dp_conv_backward_kernel_fast_ex(const float *x, size_t x_slack_bytes, const float *dy,
                                    int dy_pitch, float *dw, float *db, int n, int cin, int hi,
                                    int wi, int cout, int k, int d, void *workspace,
                                    size_t workspace_bytes, void *stream);
/* fp16-split weight gradient (ABI 6): the same dw / db as dp_conv_backward_kernel_fast_ex
 * (x, x_slack_bytes, dy_pitch as there) with x also handed over pre-split as two fp16 NCHW
 * tensors x_hi = RN_fp16(x), x_lo = RN_fp16((x - x_hi) * 2^11) with rows of xh_pitch halves
 * (0: W; a multiple of 8, dp_split_f16 writes them), xh_slack_bytes readable (and finite) past
 * each, read in place (tap offsets j*d in at most two classes mod 8 halves; the second class
 * reads x_hi_s / x_lo_s, the copies shifted by _shift()'s halves, NULL when it is 0); dy is
 * split the same way into the workspace.  Products hi.hi + (hi.lo' + lo'.hi) * 2^-11 on
 * kind::f16 with 64-pixel K blocks: half the MMAs and shared-memory operand bytes of the tf32
 * kernel, and a smaller error (fp16's 11-bit hi vs tf32's).  The caller guarantees |x| < 2^15;
 * a dy element outside (-2^15, 2^15) or not finite sends the call, on the device, to the tf32
 * kernel on x.  _workspace returns 0 where the fp16 form does not apply. */
size_t dp_conv_backward_kernel_fast_f16_workspace(int n, int cin, int hi, int wi, int cout,
                                                  int k, int d);
/* x_hi = RN_fp16(x), x_lo = RN_fp16((x - x_hi) * 2^11) elementwise (the split the fp16
 * weight gradient reads): `rows` rows of w floats -> rows of `pitch` halves (pitch >= w, a
 * multiple of 8; zeros past w); 16-byte aligned pointers.  x_hi_s / x_lo_s (or NULL): the
 * same padded arrays shifted left by `shift` (1..7) halves, x_hi_s[i] = x_hi[i + shift] (ABI 6) */
int dp_split_f16(const float *x, void *x_hi, void *x_lo, void *x_hi_s, void *x_lo_s, int shift,
                 int64_t rows, int w, int pitch, void *stream);
/* dp_maxpool_forward (f32, 1-byte codes) that also writes the output's fp16 split as
 * dp_split_f16 does (rows of y_pitch halves, a multiple of 8; the pad columns are not
 * written: the caller zeroes them once) -- fused into the warp-streaming kernel where it
 * applies, else the pool then the split (ABI 6) */
int dp_maxpool_forward_split(const float *x, float *y, void *arg, int n, int c, int h, int w,
                             int p, int d, int nonlin, void *y_hi, void *y_lo, int y_pitch,
                             void *stream);
/* the shift (halves) the fp16 weight gradient's second tap residue needs its shifted copies
 * at (0: one residue, no copies; -1: the fp16 form does not apply) */
int dp_conv_backward_kernel_fast_f16_shift(int n, int cin, int hi, int wi, int cout, int k,
                                           int d);
int dp_conv_backward_kernel_fast_f16(const float *x, size_t x_slack_bytes, const void *x_hi,
                                     const void *x_lo, const void *x_hi_s, const void *x_lo_s,
                                     size_t xh_slack_bytes, int xh_pitch, const float *dy,
                                     int dy_pitch, float *dw, float *db, int n, int cin, int hi,
                                     int wi, int cout, int k, int d, void *workspace,
                                     size_t workspace_bytes, void *stream);
/* Split form (ABI 4): _prepare stages x (the re-laid-out / shifted copies the kernel's TMA
 * boxes read) into `workspace`; it depends on x only, so it can run as soon as x exists
 * (the engine overlaps it with the forward pass on a side stream).  _staged then runs the
 * rest on the same workspace (which must not be reused in between).  When the split does
 * not apply (fallback kernel) _prepare does nothing and _staged does everything. */
int dp_conv_backward_kernel_fast_prepare(const float *x, int n, int cin, int hi, int wi,
                                         int cout, int k, int d, void *workspace,
                                         size_t workspace_bytes, void *stream);
int dp_conv_backward_kernel_fast_staged(const float *x, const float *dy, float *dw, float *db,
                                        int n, int cin, int hi, int wi, int cout, int k, int d,
                                        void *workspace, size_t workspace_bytes, void *stream);

/* debugging aid: with DP_WG_TRACE set in the environment, the fast weight-gradient kernel
 * records per-K-block clock64() timestamps of CTA 0 (256 blocks x 16 slots); this copies
 * the last launch's record to host memory (synchronous). */
int dp_debug_wgrad_trace(void *host, size_t bytes);
/* the fast weight gradient's plan for a shape (host only, no launch): 1 and up to 16 ints
 * {J, Ja, NB, lines per ring slot, M tiles, tiles per group, groups, split-K, stages, 2-row
 * boxes, dy staged, residue copies, per-tap copies, x / dy / total workspace KiB}, or 0 when
 * the shape is unsupported */
int dp_debug_wgrad_plan(int n, int cin, int hi, int wi, int cout, int k, int d, int *out,
                        int len);
/* same for the fast forward / data-gradient kernel with DP_TC_TRACE set (1024 K-steps x 8) */
int dp_debug_conv_trace(void *host, size_t bytes);

/* workspace bytes for dp_conv_backward_kernel at this shape */
size_t dp_conv_backward_kernel_workspace(int dtype, int n, int cin, int hi, int wi,
                                         int cout, int k, int d);
/* dw[cout,cin,k,k], db[cout] = sums over the n images and all pixels.
 * Deterministic: fixed split + fixed-order reduction, no float atomics. */
int dp_conv_backward_kernel(int dtype, const void *x, const void *dy, void *dw, void *db,
                            int n, int cin, int hi, int wi, int cout, int k, int d,
                            void *workspace, size_t workspace_bytes, void *stream);

/* y = act(maxpool(x)), arg = first row-major argmax (int32 or uint8 per arg_bytes) */
int dp_maxpool_forward(int dtype, const void *x, void *y, void *arg, int arg_bytes,
                       int n, int c, int h, int w, int p, int d, int nonlin, void *stream);
/* dx[n,c,hi,wi] = gather of dy at recorded taps (descending tap order), then
 * optional gate multiply as in dp_conv_backward_data */
int dp_maxpool_backward(int dtype, const void *dy, const void *arg, int arg_bytes, void *dx,
                        int n, int c, int ho, int wo, int p, int d, int hi, int wi,
                        const void *gate, int gate_kind, void *stream);
/* same, dx written with row pitch dx_pitch >= wi elements (the gate keeps pitch wi): the
 * engine hands layer 0's delta to the weight gradient in a 16-byte-aligned row pitch so the
 * kernel's TMA reads it without a re-pitch copy (ABI 5) */
int dp_maxpool_backward_pitched(int dtype, const void *dy, const void *arg, int arg_bytes,
                                void *dx, int dx_pitch, int n, int c, int ho, int wo, int p,
                                int d, int hi, int wi, const void *gate, int gate_kind,
                                void *stream);
int dp_avgpool_forward(int dtype, const void *x, void *y, int n, int c, int h, int w,
                       int p, int d, int nonlin, void *stream);
int dp_avgpool_backward(int dtype, const void *dy, void *dx, int n, int c, int ho, int wo,
                        int p, int d, int hi, int wi, const void *gate, int gate_kind,
                        void *stream);

/* elementwise nonlinearity; backward: x_is_output=0 -> x is the input
 * (reference semantics), 1 -> x is the nonlinearity's output */
int dp_nonlin_forward(int dtype, const void *x, void *y, int64_t count, int kind, void *stream);
int dp_nonlin_backward(int dtype, const void *dy, const void *x, void *dx, int64_t count,
                       int kind, int x_is_output, void *stream);

/* error-map mask / loss layer (backward.py:110-118; squared-error delta cli.py:218):
 * out[n,c,y,x] = mask[n,y,x] ? (target ? a - target : a) : 0, mask uint8 (n,h,w) */
int dp_mask_delta(int dtype, const void *a, const void *target, const uint8_t *mask, void *out,
                  int n, int c, int h, int w, void *stream);

/* zero-pad (n,c,h,w) -> (n,c,h+top+bottom,w+left+right)  (forward.py:96-98) */
int dp_pad(int dtype, const void *src, void *dst, int n, int c, int h, int w,
           int top, int bottom, int left, int right, void *stream);
/* crop window (top,left,h,w) of (n,c,hs,ws) -> (n,c,h,w)  (backward.py:218-222) */
int dp_crop(int dtype, const void *src, void *dst, int n, int c, int hs, int ws,
            int top, int left, int h, int w, void *stream);
/* per-pixel softmax cross-entropy over q classes (not in the
 * reference, whose delta is squared error): delta = softmax(logits) - onehot(label) and
 * loss = -log softmax[label] where mask (may be NULL = all) is set and label != 255
 * (ignore); zero elsewhere.  logits / delta (n, q, h, w); labels / mask uint8 (n, h, w);
 * loss (n, h, w) or NULL. */
int dp_softmax_xent_delta(int dtype, const void *logits, const uint8_t *labels,
                          const uint8_t *mask, void *delta, void *loss, int n, int q, int h, int w,
                          void *stream);
/* patch-by-patch baseline (reference oracle.py scan_forward:145-164): gather the patch x
 * patch windows of pixels [first, first+count) (row-major over the w-wide output grid) of ONE
 * zero-padded image x0 (c, hp, wp) into out (count, c, patch, patch) */
int dp_patch_gather(int dtype, const void *x0, void *out, int c, int hp, int wp, int patch,
                    int w, int64_t first, int64_t count, void *stream);
/* param = param - lr * grad, rounded as numpy rounds it (plain SGD; the reference has no
 * optimizer) */
int dp_sgd_update(int dtype, void *param, const void *grad, int64_t count, double lr,
                  void *stream);

/* ---- original strided network, for the GPU patch-by-patch baseline -------------------
 * (reference oracle.py:29-262: conv_strided / maxpool_strided / avgpool_strided,
 * scan_forward, patch_backward_batch).  Device pointers, batches of n patches. */
enum dp_pool_kind { DP_POOL_MAX = 0, DP_POOL_AVG = 1 };
/* strided pool (oracle.py:58-91): y = tap(0,0), then row-major taps; max: strict `>`
 * (first wins), int32 argmax i*p+j; avg: running sum / p^2.  Requires (h-p) % s == 0
 * (oracle.py _out_side). */
int dp_pool_strided_forward(int dtype, int kind, const void *x, void *y, int32_t *arg, int n,
                            int c, int h, int w, int p, int s, void *stream);
/* its backward (oracle.py:190-211) as a gather in ascending tap order; hi = (ho-1)*s + p */
int dp_pool_strided_backward(int dtype, int kind, const void *dy, const int32_t *arg, void *dx,
                             int n, int c, int ho, int wo, int p, int s, int hi, int wi,
                             void *stream);
/* y[u,v] = x[u*s, v*s]: a stride-s conv is the stride-1 conv sampled every s pixels */
int dp_subsample(int dtype, const void *x, void *y, int n, int c, int h, int w, int s, int ho,
                 int wo, void *stream);
/* out (n,c,hf,wf) = 0 except out[u*s, v*s] = dy[u,v]: backward of dp_subsample */
int dp_zero_insert(int dtype, const void *dy, void *out, int n, int c, int ho, int wo, int s,
                   int hf, int wf, void *stream);
/* gather the patch x patch windows of an arbitrary pixel list (flat indices y*w + x over the
 * w = wp-patch+1 wide output grid, device int32[count], caller-validated) of ONE padded
 * image x0 (c, hp, wp) into out (count, c, patch, patch) */
int dp_patch_gather_pixels(int dtype, const void *x0, void *out, int c, int hp, int wp, int patch,
                           const int32_t *pixels, int64_t count, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DENSEPROP_B200_H */
