// tcgen05 TS-mode probe: A operand in TMEM (written with tcgen05.st from registers),
// B in SMEM (K-major, no swizzle).  kind::tf32, M=128, K=8.
// Questions: is D correct with this A-in-TMEM layout (lane = row m, 8 consecutive
// 32-bit columns = K), and what does one MMA cost for N = 16..256 when the SMEM
// read is only B (the SS probe showed ~128 B/cycle SMEM-bound MMAs for small N)?
// Also times tcgen05.st of a 128 x 16 fp32 A pair (hi + lo) by 4 warps.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe_ts tools/tc_probe_ts.cu
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)(layout & 7) << 61);
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
    return pred;
}
__device__ __forceinline__ void mma_ts(uint32_t dt, uint32_t at, uint64_t bd, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dt), "r"(at),
        "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                     "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ inline uint32_t b_off(int n, int k) {
    return (n >> 3) * 256 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4;
}

template <int N, int NACC>
__global__ void __launch_bounds__(128) ts_probe(const float *A, const float *B, float *D,
                                                long long *cyc) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sB = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < N * 8; i += 128) *(float *)(sB + b_off(i / 8, i % 8)) = B[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    // A -> TMEM columns [0, 8): lane m = row m
    const int m = warp * 32 + lane;
    float v[8];
    for (int k = 0; k < 8; ++k) v[k] = A[m * 8 + k];
    long long s0 = clock64();
    const uint32_t lanebase = (uint32_t)(warp * 32) << 16;
    tmem_st8(tm + lanebase + 0, v);
    tmem_st8(tm + lanebase + 8, v);   // second copy (timing of a hi+lo pair)
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long s1 = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint64_t bd = make_desc(smem_u32(sB), 128, 256, 0);
    constexpr uint32_t idesc = make_idesc(128, N);
    if (warp == 0) {
        if (elect_one()) {
            mma_ts(tm + 64, tm + 0, bd, idesc, 0);
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t0 = clock64();
        if (NACC >= 100) {
            // conv-kernel pattern: 4 M tiles x (A_hi.B_hi, A_hi.B_lo, A_lo.B_hi), distinct
            // A columns per tile, two B tiles; 43 x 12 = 516 MMAs
            const uint64_t bd2 = make_desc(smem_u32(sB) + N * 32, 128, 256, 0);
            for (int r = 0; r < 43; ++r) {
                if (elect_one()) {
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) {
                        const uint32_t d = tm + 256 + mt * N;
                        const uint32_t ahi = tm + mt * 16, alo = ahi + 8;
                        mma_ts(d, ahi, bd, idesc, r > 0);
                        mma_ts(d, ahi, bd2, idesc, 1);
                        mma_ts(d, alo, bd, idesc, 1);
                    }
                }
                __syncwarp();
            }
        } else {
            for (int r = 0; r < 512 / NACC; ++r) {
#pragma unroll
                for (int q = 0; q < NACC; ++q)
                    if (elect_one()) mma_ts(tm + 256 + q * N, tm + (q & 1) * 8, bd, idesc, r > 0);
                __syncwarp();
            }
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 1);
        if (lane == 0) {
            cyc[0] = clock64() - t0;
            cyc[1] = s1 - s0;
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < N; c0 += 16) {
        float o[16];
        tmem_ld16(tm + lanebase + 64 + c0, o);
        for (int i = 0; i < 16; ++i) D[m * N + c0 + i] = o[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

static float trunc_tf32(float x) {
    uint32_t u = *(uint32_t *)&x;
    u &= 0xFFFFE000u;
    return *(float *)&u;
}

template <int N, int NACC>
static void run() {
    std::vector<float> A(128 * 8), B(N * 8), D(128 * N);
    srand(11 + N);
    for (auto &x : A) x = (float)rand() / RAND_MAX * 2 - 1;
    for (auto &x : B) x = (float)rand() / RAND_MAX * 2 - 1;
    float *dA, *dB, *dD;
    long long *dc;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 16));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    int smem = N * 64 + 2048;
    CK(cudaFuncSetAttribute(ts_probe<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ts_probe<N, NACC><<<1, 128, smem>>>(dA, dB, dD, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    long long c[2];
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost));
    double err = 0, scale = 0;
    for (int mm = 0; mm < 128; ++mm)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < 8; ++k) s += (double)trunc_tf32(A[mm * 8 + k]) * trunc_tf32(B[n * 8 + k]);
            err = fmax(err, fabs(s - D[mm * N + n]));
            scale = fmax(scale, fabs(s));
        }
    printf("TS N=%3d nacc=%d: maxerr vs trunc-tf32 %.3e (scale %.2f)  %.2f cycles/MMA; "
           "tcgen05.st 2x(32x32b.x8) + wait: %lld cycles\n", N, NACC, err, scale, c[0] / (NACC >= 100 ? 516.0 : 512.0),
           c[1]);
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
}

int main() {
    CK(cudaSetDevice(0));
    run<16, 1>(); run<32, 1>(); run<16, 100>(); run<32, 100>(); run<64, 100>();
    run<128, 1>(); run<256, 1>();
    return 0;
}
