// Dense tcgen05 throughput on every SM, operands in shared memory (SS, K-major, no swizzle or
// SWIZZLE_128B): one CTA per SM, one thread issuing `count` back-to-back MMAs of M = 128
// rotating over 512 / N accumulators, one commit at the end; TFLOP/s from CUDA events over the whole grid.  The
// measured ceilings of the conv / weight-gradient kernels' arithmetic (kind::tf32 for 3xTF32,
// kind::f16 for the fp16 split) at the N they issue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_peak tools/mma_peak.cu
//   ./tools/mma_peak
#include <cstdio>

#include "../paper_1412_4526_b200/csrc/tc_ptx.cuh"
using namespace dp;

// A from TMEM (the "TS" form): K-major A rows in TMEM columns
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

// sw: 0 = no swizzle, 1 = SWIZZLE_128B, 2 = A from TMEM (TS), 3 = A copied smem -> TMEM
// (tcgen05.cp 128x256b) before every PAIR of TS MMAs that share it, 4 = before every one.  Accumulators rotate with
// compile-time offsets over 256 TMEM columns (N = 64: 4, 128: 2, 256: 1), the issue loop is
// unrolled by 4 (an index computation per MMA made the issuing thread the limit)
template <int N>
__global__ void __launch_bounds__(128, 1) peak(int count, int f16, int sw) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (64 * 1024) / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_fence_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&s_tmem);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = s_tmem;
    if (warp == 0) {
        // A: 128 rows, B: N rows; K-major no-swizzle core matrices (8 rows x 16 B): SBO = 128
        // between 8-row groups, LBO = one K chunk (16 B of K) of all rows
        // (sw: K-major SWIZZLE_128B, rows of 128 B in 1 KB atoms, as the weight gradient's
        // TMA boxes write them)
        const uint32_t a0 = ptx::smem_u32(sm), b0 = a0 + 16 * 1024;
        const uint64_t ad = sw == 1 ? ptx::smem_desc_sw128(a0) : ptx::smem_desc(a0, 128 * 16, 128);
        const uint64_t bd =
            sw == 1 ? ptx::smem_desc_sw128(b0) : ptx::smem_desc(b0, (uint32_t)N * 16, 128);
        const uint32_t a_tm = tmem + 448;  // A operand columns (TS form), past the accumulators
        const uint32_t idesc = f16 ? ptx::idesc_f16(128, N) : ptx::idesc_tf32(128, N);
        if (ptx::elect_one()) {
            constexpr int NACC = 256 / N;
            for (int i = 0; i < count; i += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t d = tmem + (uint32_t)((u % NACC) * N);
                    if (sw >= 3 && (sw == 4 || (u & 1) == 0))
                        cp_128x256b(a_tm + (uint32_t)((u & 2) * 4), ad);
                    if (sw >= 3 && f16)
                        mma_f16_ts(d, a_tm + (uint32_t)((u & 2) * 4), bd, idesc, 1);
                    else if (sw >= 3)
                        ptx::mma_tf32_ts(d, a_tm + (uint32_t)((u & 2) * 4), bd, idesc, 1);
                    else if (sw == 2 && f16)
                        mma_f16_ts(d, a_tm, bd, idesc, 1);
                    else if (sw == 2)
                        ptx::mma_tf32_ts(d, a_tm, bd, idesc, 1);
                    else if (f16)
                        ptx::mma_f16_ss(d, ad, bd, idesc, 1);
                    else
                        ptx::mma_tf32_ss(d, ad, bd, idesc, 1);
                }
            }
            ptx::mma_commit(&bar);
        }
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        ptx::tc_fence_after();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

int main() {
    int sms = 0, dev = 0, mhz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, dev);
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(peak<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(peak<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(peak<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int count = 20000;
    printf("{\"sms\": %d, \"points\": [\n", sms);
    bool first = true;
    for (int sw = 0; sw < 5; ++sw)
    for (int f16 = 0; f16 < 2; ++f16)
        for (int N : {64, 128, 256}) {
            const int K = f16 ? 16 : 8;
            auto kern = N == 64 ? peak<64> : N == 128 ? peak<128> : peak<256>;
            kern<<<sms, 128, smem>>>(200, f16, sw);  // warm-up
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                kern<<<sms, 128, smem>>>(count, f16, sw);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            const double flops = 2.0 * 128 * N * K * (double)count * sms;
            const double tf = flops / (best * 1e-3) / 1e12;
            const double cyc = best * 1e-3 * 1965e6 / count;  // at the max SM clock
            printf("%s {\"kind\": \"%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"operands\": \"%s\", \"layout\": \"%s\", "
                   "\"tflops\": %.1f, \"cycles_per_mma_at_1965MHz\": %.1f}",
                   first ? "" : ",\n", f16 ? "f16" : "tf32", N, K, sw >= 2 ? "TS" : "SS",
                   sw == 4 ? "TS, cp per MMA" : sw == 3 ? "TS, cp per 2 MMAs" :
                   sw == 2 ? "A in TMEM (TS)" : sw ? "sw128" : "none", tf,
                   cyc);
            first = false;
        }
    printf("\n], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
