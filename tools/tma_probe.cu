// TMA bring-up probe: 4-D tiled loads with / without 128B swizzle, checked on the host.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1412_4526_b200/csrc/tc_ptx.cuh"

using namespace dp;

__global__ void probe(const __grid_constant__ CUtensorMap tm, float *out, int c0, int c1, int nbytes,
                      int mode) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    __shared__ uint64_t bar;
    unsigned char *sm = (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ptx::mbar_expect_tx(&bar, nbytes);
        if (mode == 0) ptx::tma_load_4d(sm, &tm, c0, c1, 0, 0, &bar);
    }
    ptx::mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < nbytes / 4; i += blockDim.x) out[i] = ((float *)sm)[i];
}

int main(int argc, char **argv) {
    int swz = argc > 1 ? atoi(argv[1]) : 1;
    int cx = argc > 2 ? atoi(argv[2]) : 40;
    int W = 75, H = 70, C = 3, N = 2, WP = 76;
    std::vector<float> h((size_t)N * C * H * WP);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 1 << 16);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    printf("entry point: %d q=%d fn=%p\n", (int)e, (int)q, fn);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
    cuuint64_t str[3] = {(cuuint64_t)WP * 4, (cuuint64_t)WP * 4 * H, (cuuint64_t)WP * 4 * H * C};
    cuuint32_t box[4] = {32, 1, 8, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    probe<<<1, 128, 8192>>>(m, o, cx, 5, 32 * 8 * 4, 0);
    e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    std::vector<float> res(256);
    cudaMemcpy(res.data(), o, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < 8; ++row)
        for (int k = 0; k < 32; ++k) {
            int chunk = k / 4;
            int pchunk = swz ? (chunk ^ (row & 7)) : chunk;
            float got = res[row * 32 + pchunk * 4 + (k & 3)];
            int v = cx + k;
            float want = (row < C && v < W) ? h[((size_t)row * H + 5) * WP + v] : 0.f;
            if (got != want && bad++ < 5) printf("row %d k %d got %g want %g\n", row, k, got, want);
        }
    printf("swz=%d bad=%d\n", swz, bad);
    return 0;
}
