// Pipeline trace of the tensor-core conv kernel (CTA 0): per K-step clock64 stamps of
// producer group (empty-wait start/end, TMEM stores retired) and MMA warp (full-wait
// start/end, MMAs issued).  Builds tc_conv.cu with DP_TC_TRACE into a standalone binary.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DDP_TC_TRACE -I include \
//      -o tools/tc_trace tools/tc_trace.cu paper_1412_4526_b200/csrc/tc_conv.cu stub
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdarg.h>
#include <vector>

#define DP_TC_TRACE 1
#include "../paper_1412_4526_b200/csrc/tc_conv.cu"

namespace dp {
int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vprintf(fmt, ap);
    va_end(ap);
    printf("\n");
    return code;
}
int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("%s: %s\n", what, cudaGetErrorString(e));
    return e != cudaSuccess;
}
}  // namespace dp

int main(int argc, char **argv) {
    int N = 16, ci = 16, co = 32, k = 5, d = 2, H = 278, dbg = 0, rows = 60;
    if (argc > 1) sscanf(argv[1], "%d,%d,%d,%d,%d,%d", &N, &ci, &co, &k, &d, &H);
    if (argc > 2) dbg = atoi(argv[2]);
    if (argc > 3) rows = atoi(argv[3]);
    int e = (k - 1) * d + 1, Ho = H - e + 1;
    size_t nx = (size_t)N * ci * H * H, ny = (size_t)N * co * Ho * Ho;
    float *x, *w, *b, *y;
    unsigned long long *tr;
    cudaMalloc(&x, nx * 4);
    cudaMalloc(&w, (size_t)co * ci * k * k * 4);
    cudaMalloc(&b, co * 4);
    cudaMalloc(&y, ny * 4);
    cudaMalloc(&tr, 512 * 8 * 8);
    cudaMemset(x, 0, nx * 4);
    cudaMemset(w, 0, (size_t)co * ci * k * k * 4);
    cudaMemset(b, 0, co * 4);
    cudaMemset(tr, 0, 512 * 8 * 8);
    size_t wsb = dp::tc_conv_workspace(ci, co, k);
    void *ws;
    cudaMalloc(&ws, wsb);
    // reuse the library launcher but inject the trace pointer through a patched copy
    dp::TcPlan p = dp::tc_plan(ci, co, k);
    dp::tc_pack_weights<<<64, 256>>>(w, (float *)ws, co, ci, k, p.Npad, p.n_rc, p.n_ks, 0);
    dp::TcConvArgs a{};
    a.in = x; a.wpack = (float *)ws; a.bias = b; a.out = y; a.gate = nullptr;
    a.R = ci; a.Hin = H; a.Win = H; a.Q = co; a.Ho = Ho; a.Wo = Ho; a.l = k; a.d = d; a.pad = 0;
    a.act = 0; a.gate_kind = 0; a.n_rc = p.n_rc; a.n_ks = p.n_ks; a.Npad = p.Npad; a.MT = p.MT;
    a.stages = p.stages; a.acc_cols = p.acc_cols; a.tiles_x = (Ho + 31) / 32;
    a.tiles_y = (Ho + 4 * a.MT - 1) / (4 * a.MT); a.total_tiles = N * a.tiles_x * a.tiles_y;
    a.wbytes = (uint32_t)p.wbytes; a.trace = tr; a.dbg = dbg;
    auto kern = p.stacked ? dp::tc_conv_kernel<true, false> : dp::tc_conv_kernel<false, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.wbytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<148, dp::TC_THREADS, p.wbytes>>>(a);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dbg=%d MT=%d stages=%d n_ks=%d tiles=%d: %.3f ms\n", dbg, a.MT, a.stages, a.n_ks, a.total_tiles, ms);
    std::vector<unsigned long long> t(512 * 8);
    cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = t[3];
    printf("KS: prod[wait_start wait_end st_done after_commit after_load] mma[wait_start wait_end issued]\n");
    for (int ks = 0; ks < rows; ++ks) {
        long long v[8];
        for (int s = 0; s < 8; ++s) v[s] = t[ks * 8 + s] ? (long long)(t[ks * 8 + s] - t0) : -1;
        printf("%3d: %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld\n", ks, v[0], v[1], v[2],
               v[6], v[7], v[3], v[4], v[5]);
    }
    return 0;
}
