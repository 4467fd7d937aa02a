/*
 * C/OpenMP restatement of the reference's 7 boundary kernels -- TEST
 * INFRASTRUCTURE ONLY (see oracle/__init__.py).  Used as the multi-threaded
 * CPU "port" baseline and as a checker at sizes numpy is too slow for.
 *
 * Per-entry operation order follows the compiled reference backend
 * (pkg/src/denseprop/_kernels.pyx) exactly; build with -ffp-contract=off
 * (reference pkg/setup.py:15) so no multiply-add is fused:
 *   conv_forward          _kernels.pyx:23-53   bias, then (c,i,j) taps
 *   conv_backward_data    _kernels.pyx:56-91   (o,i,j) gather, rotated kernel
 *   conv_backward_kernel  _kernels.pyx:94-130  sequential (u,v) sums per o
 *   maxpool_forward       _kernels.pyx:133-166 -inf start, strict '>'
 *   maxpool_backward      _kernels.pyx:169-191 row-major scatter per channel
 *   avgpool_forward       _kernels.pyx:194-221 acc=0, += taps, / (p*p)
 *   avgpool_backward      _kernels.pyx:224-247 q = dy/(p*p) scattered
 * Parallel loops own disjoint outputs, so thread count never changes results.
 */
#include <math.h>
#include <stddef.h>
#include <string.h>

typedef ptrdiff_t ix;

#define DEFINE_KERNELS(T, SFX)                                                   \
void ork_conv_forward_##SFX(const T *x, const T *w, const T *b, T *y, ix cin,    \
                            ix h, ix wd, ix cout, ix l, ix d, int threads) {     \
    ix e = (l - 1) * d + 1, ho = h - e + 1, wo = wd - e + 1;                      \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")            \
    for (ix n = 0; n < cout * ho; ++n) {                                         \
        ix o = n / ho, u = n % ho;                                               \
        T *yr = y + (o * ho + u) * wo;                                           \
        for (ix v = 0; v < wo; ++v) yr[v] = b[o];                                \
        for (ix c = 0; c < cin; ++c)                                             \
            for (ix i = 0; i < l; ++i) {                                         \
                const T *xr = x + (c * h + u + i * d) * wd;                      \
                for (ix j = 0; j < l; ++j) {                                     \
                    T wv = w[((o * cin + c) * l + i) * l + j];                   \
                    const T *xs = xr + j * d;                                    \
                    for (ix v = 0; v < wo; ++v) yr[v] = yr[v] + wv * xs[v];      \
                }                                                                \
            }                                                                    \
    }                                                                            \
}                                                                                \
void ork_conv_backward_data_##SFX(const T *dy, const T *w, T *dx, ix cout,       \
                                  ix ho, ix wo, ix cin, ix l, ix d,              \
                                  int threads) {                                 \
    ix e = (l - 1) * d + 1, hi = ho + e - 1, wi = wo + e - 1;                    \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")            \
    for (ix n = 0; n < cin * hi; ++n) {                                          \
        ix c = n / hi, yy = n % hi;                                              \
        T *dr = dx + (c * hi + yy) * wi;                                         \
        for (ix xx = 0; xx < wi; ++xx) dr[xx] = 0;                               \
        for (ix o = 0; o < cout; ++o)                                            \
            for (ix i = 0; i < l; ++i) {                                         \
                ix u = yy + i * d - (e - 1);                                     \
                if (u < 0 || u >= ho) continue;                                  \
                const T *dyr = dy + (o * ho + u) * wo;                           \
                for (ix j = 0; j < l; ++j) {                                     \
                    T wv = w[((o * cin + c) * l + (l - 1 - i)) * l + (l - 1 - j)];\
                    ix off = j * d - (e - 1);                                    \
                    ix lo = off >= 0 ? 0 : -off;                                 \
                    ix hi2 = (wo - off > wi) ? wi : wo - off;                    \
                    for (ix xx = lo; xx < hi2; ++xx)                             \
                        dr[xx] = dr[xx] + wv * dyr[xx + off];                    \
                }                                                                \
            }                                                                    \
    }                                                                            \
}                                                                                \
void ork_conv_backward_kernel_##SFX(const T *x, const T *dy, T *dw, T *db,       \
                                    ix cin, ix hi, ix wi, ix cout, ix ho, ix wo, \
                                    ix l, ix d, int threads) {                   \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")            \
    for (ix o = 0; o < cout; ++o) {                                              \
        const T *dyo = dy + o * ho * wo;                                         \
        T s = 0;                                                                 \
        for (ix q = 0; q < ho * wo; ++q) s = s + dyo[q];                         \
        db[o] = s;                                                               \
        for (ix c = 0; c < cin; ++c)                                             \
            for (ix i = 0; i < l; ++i)                                           \
                for (ix j = 0; j < l; ++j) {                                     \
                    T acc = 0;                                                   \
                    for (ix u = 0; u < ho; ++u) {                                \
                        const T *xr = x + (c * hi + u + i * d) * wi + j * d;     \
                        const T *dr = dyo + u * wo;                              \
                        for (ix v = 0; v < wo; ++v) acc = acc + dr[v] * xr[v];   \
                    }                                                            \
                    dw[((o * cin + c) * l + i) * l + j] = acc;                   \
                }                                                                \
    }                                                                            \
}                                                                                \
void ork_maxpool_forward_##SFX(const T *x, T *y, int *arg, ix c, ix h, ix wd,    \
                               ix p, ix d, int threads) {                        \
    ix e = (p - 1) * d + 1, ho = h - e + 1, wo = wd - e + 1;                      \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")            \
    for (ix n = 0; n < c * ho; ++n) {                                            \
        ix ch = n / ho, u = n % ho;                                              \
        for (ix v = 0; v < wo; ++v) {                                            \
            T best = (T)(-INFINITY);                                             \
            int bk = 0;                                                          \
            for (ix i = 0; i < p; ++i)                                           \
                for (ix j = 0; j < p; ++j) {                                     \
                    T xv = x[(ch * h + u + i * d) * wd + v + j * d];             \
                    if (xv > best) { best = xv; bk = (int)(i * p + j); }         \
                }                                                                \
            y[(ch * ho + u) * wo + v] = best;                                    \
            arg[(ch * ho + u) * wo + v] = bk;                                    \
        }                                                                        \
    }                                                                            \
}                                                                                \
void ork_maxpool_backward_##SFX(const T *dy, const int *arg, T *dx, ix c,        \
                                ix ho, ix wo, ix p, ix d, ix hi, ix wi,          \
                                int threads) {                                   \
    memset(dx, 0, sizeof(T) * (size_t)(c * hi * wi));                            \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")            \
    for (ix ch = 0; ch < c; ++ch)                                                \
        for (ix u = 0; u < ho; ++u)                                              \
            for (ix v = 0; v < wo; ++v) {                                        \
                ix k = arg[(ch * ho + u) * wo + v], i = k / p, j = k % p;        \
                T *t = dx + (ch * hi + u + i * d) * wi + v + j * d;              \
                *t = *t + dy[(ch * ho + u) * wo + v];                            \
            }                                                                    \
}                                                                                \
void ork_avgpool_forward_##SFX(const T *x, T *y, ix c, ix h, ix wd, ix p, ix d,  \
                               int threads) {                                    \
    ix e = (p - 1) * d + 1, ho = h - e + 1, wo = wd - e + 1;                      \
    T pp = (T)(p * p);                                                           \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")            \
    for (ix n = 0; n < c * ho; ++n) {                                            \
        ix ch = n / ho, u = n % ho;                                              \
        for (ix v = 0; v < wo; ++v) {                                            \
            T acc = 0;                                                           \
            for (ix i = 0; i < p; ++i)                                           \
                for (ix j = 0; j < p; ++j)                                       \
                    acc = acc + x[(ch * h + u + i * d) * wd + v + j * d];        \
            y[(ch * ho + u) * wo + v] = acc / pp;                                \
        }                                                                        \
    }                                                                            \
}                                                                                \
void ork_avgpool_backward_##SFX(const T *dy, T *dx, ix c, ix ho, ix wo, ix p,    \
                                ix d, ix hi, ix wi, int threads) {               \
    T pp = (T)(p * p);                                                           \
    memset(dx, 0, sizeof(T) * (size_t)(c * hi * wi));                            \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")            \
    for (ix ch = 0; ch < c; ++ch)                                                \
        for (ix u = 0; u < ho; ++u)                                              \
            for (ix v = 0; v < wo; ++v) {                                        \
                T q = dy[(ch * ho + u) * wo + v] / pp;                           \
                for (ix i = 0; i < p; ++i)                                       \
                    for (ix j = 0; j < p; ++j) {                                 \
                        T *t = dx + (ch * hi + u + i * d) * wi + v + j * d;      \
                        *t = *t + q;                                             \
                    }                                                            \
            }                                                                    \
}

DEFINE_KERNELS(float, f32)
DEFINE_KERNELS(double, f64)
