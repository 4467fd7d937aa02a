// Probe: tcgen05.mma kind::tf32, cta_group::1, M=64, N=16, K=8, A and B from SMEM (K-major,
// SWIZZLE_NONE).  A[m][k] = m + 1 (k = 0 only), B[n][k] = (n == 0) -> D[m][0] = m + 1.  Dumps
// every TMEM lane's column 0 so the M=64 row -> lane mapping can be read off.
#include <cstdio>
#include <cstdint>
#include "../paper_1412_4526_b200/csrc/tc_ptx.cuh"
using namespace dp;

__global__ void probe(float *out) {
    __shared__ __align__(1024) float sa[64 * 8];
    __shared__ __align__(1024) float sb[16 * 8];
    __shared__ uint64_t bar;
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // K-major SWIZZLE_NONE core matrices: (m>>3)*256 + (k>>2)*128 + (m&7)*16 + (k&3)*4 bytes
    for (int m = tid; m < 64; m += blockDim.x)
        for (int k = 0; k < 8; ++k)
            sa[((m >> 3) * 256 + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4) / 4] = k == 0 ? (float)(m + 1) : 0.f;
    for (int n = tid; n < 16; n += blockDim.x)
        for (int k = 0; k < 8; ++k)
            sb[((n >> 3) * 256 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4) / 4] = (k == 0 && n == 0) ? 1.f : 0.f;
    if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::mbar_fence_init(); }
    ptx::fence_proxy_async_smem();
    if (warp == 0) ptx::tmem_alloc<32>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;
    // zero the accumulator columns first (all 128 lanes, 16 columns)
    {
        float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const uint32_t lo = (uint32_t)(warp * 32) << 16;
        ptx::tmem_st8(tmem + lo, z);
        ptx::tmem_st8(tmem + lo + 8, z);
        ptx::tmem_wait_st();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) {
        if (ptx::elect_one()) {
            const uint64_t da = ptx::smem_desc(ptx::smem_u32(sa), 128, 256);
            const uint64_t db = ptx::smem_desc(ptx::smem_u32(sb), 128, 256);
            ptx::mma_tf32_ss(tmem, da, db, ptx::idesc_tf32(64, 16), 0);
            ptx::mma_commit(&bar);
        }
        __syncwarp();
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    uint32_t r[16];
    ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), r);
    ptx::tmem_wait_ld();
    out[warp * 32 + lane] = __uint_as_float(r[0]);
    out[128 + warp * 32 + lane] = __uint_as_float(r[1]);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<32>(tmem);
}

int main() {
    float *d, h[256];
    cudaMalloc(&d, 256 * 4);
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 256 * 4, cudaMemcpyDeviceToHost);
    for (int q = 0; q < 4; ++q) {
        printf("quadrant %d col0:", q);
        for (int l = 0; l < 32; ++l) printf(" %g", h[q * 32 + l]);
        printf("\n");
    }
    return 0;
}
