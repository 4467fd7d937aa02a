// Handshake latency probe: ping-pong between two warps through mbarriers, with
// (a) mbarrier.try_wait, (b) mbarrier.test_wait spin, (c) the "pong" side arriving via
// tcgen05.commit (no MMA in flight) instead of a plain arrive.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/sync_probe tools/sync_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "../paper_1412_4526_b200/csrc/tc_ptx.cuh"
using namespace dp;

__device__ __forceinline__ void wait_test(uint64_t *b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(ptx::smem_u32(b)), "r"(parity) : "memory");
    }
}

__global__ void pingpong(int iters, int mode, unsigned long long *out) {
    __shared__ uint64_t ping, pong;
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&ping, 1);
        ptx::mbar_init(&pong, 1);
        ptx::mbar_fence_init();
    }
    if (warp == 1) ptx::tmem_alloc<32>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (warp == 0) {
            if (threadIdx.x == 0) ptx::mbar_arrive(&ping);
            if (mode == 1) wait_test(&pong, it & 1); else ptx::mbar_wait(&pong, it & 1);
        } else if (warp == 1) {
            if (mode == 1) wait_test(&ping, it & 1); else ptx::mbar_wait(&ping, it & 1);
            if (mode == 2) {
                ptx::tc_fence_after();
                if (ptx::elect_one()) ptx::mma_commit(&pong);
                __syncwarp();
            } else {
                if (threadIdx.x == 32) ptx::mbar_arrive(&pong);
            }
        }
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<32>(s_tmem);
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

// TMA latency: one box at a time, issue -> mbarrier completion, same box repeatedly (L2 hot)
__global__ void tma_lat(const __grid_constant__ CUtensorMap tm, int iters, int nbox, unsigned long long *out) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    __shared__ uint64_t bar;
    unsigned char *sm = (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_fence_init();
        ptx::tma_prefetch_desc(&tm);
    }
    __syncthreads();
    unsigned long long tot = 0;
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            unsigned long long t0 = clock64();
            ptx::mbar_expect_tx(&bar, nbox * 32 * 32 * 4);
            for (int b = 0; b < nbox; ++b) ptx::tma_load_4d(sm + b * 4096, &tm, 0, it % 4, 0, b, &bar);
            ptx::mbar_wait(&bar, it & 1);
            tot += clock64() - t0;
        }
        out[0] = tot / iters;
    }
}

// Skeleton of the tc_conv / tc_wgrad pipeline: 2 producer groups x 4 warps alternate K-steps,
// S stages, one MMA warp waits full / commits empty.  No data, no MMAs.
// flags: 1 producer uses tcgen05.wait::st + fences, 2 MMA uses tcgen05.commit (else arrive),
//        4 MMA thread does tcgen05.fence::after_thread_sync
__global__ void skeleton(int ksteps, int S, int flags, unsigned long long *out) {
    __shared__ uint64_t full[16], empty[16];
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 4);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_fence_init();
    }
    if (warp == 8) ptx::tmem_alloc<32>(&s_tmem);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    unsigned long long t0 = clock64();
    if (warp < 8) {
        const int grp = warp >> 2;
        for (int KS = grp; KS < ksteps; KS += 2) {
            const int st = KS % S;
            ptx::mbar_wait(&empty[st], ((KS / S) & 1) ^ 1);
            if (flags & 1) {
                ptx::tc_fence_after();
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&full[st]);
        }
    } else if (warp == 8) {
        for (int KS = 0; KS < ksteps; ++KS) {
            const int st = KS % S;
            ptx::mbar_wait(&full[st], (KS / S) & 1);
            if (flags & 4) ptx::tc_fence_after();
            if (flags & 2) {
                if (ptx::elect_one()) ptx::mma_commit(&empty[st]);
                __syncwarp();
            } else if (lane == 0) {
                ptx::mbar_arrive(&empty[st]);
            }
        }
    }
    unsigned long long t1 = clock64();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 8) ptx::tmem_dealloc<32>(s_tmem);
    if (threadIdx.x == 256) out[blockIdx.x] = (t1 - t0) / ksteps;
}

int main() {
    unsigned long long *d, h;
    cudaMalloc(&d, 8);
    const char *names[] = {"try_wait ping-pong", "test_wait spin ping-pong", "pong via tcgen05.commit"};
    for (int mode = 0; mode < 3; ++mode) {
        pingpong<<<1, 64>>>(1000, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-28s: %llu cycles per round trip (%s)\n", names[mode], h, cudaGetErrorString(e));
    }
    float *buf;
    cudaMalloc(&buf, 64 << 20);
    cudaMemset(buf, 0, 64 << 20);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m;
    // (w=272, h=270, c=32, n=8), box {32, 1, 32, 1}: a dy-like box, 32 lines a plane apart
    cuuint64_t dims[4] = {272, 270, 32, 8};
    cuuint64_t str[3] = {272 * 4, 272 * 4 * 270, 272ull * 4 * 270 * 32};
    cuuint32_t box[4] = {32, 1, 32, 1}, es[4] = {1, 1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(tma_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int nb : {1, 2, 4, 8}) {
        tma_lat<<<1, 32, 100 * 1024>>>(m, 200, nb, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("TMA %d box(es) {32,1,32} issue->complete: %llu cycles (%s)\n", nb, h, cudaGetErrorString(e));
    }
    for (int grid : {1, 148})
        for (int S : {4, 8})
            for (int flags : {0, 1, 2, 4, 7}) {
                skeleton<<<grid, 288>>>(4000, S, flags, d);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                printf("skeleton grid %3d S=%d flags=%d: %llu cycles per K-step (%s)\n", grid, S, flags, h,
                       cudaGetErrorString(e));
            }
    return 0;
}
