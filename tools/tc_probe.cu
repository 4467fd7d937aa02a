// tcgen05 / TMA probe for the 3xTF32 dilated-conv design (sm_100a).
//
// Answers, on the real B200, the questions the tensor-core conv kernel is built on:
//  1. Does kind::tf32 with A MN-major SWIZZLE_128B (activations straight from a CHW
//     map) and B K-major no-swizzle (pre-arranged weights) give D = A.B?  Which
//     fp32->tf32 conversion does the datapath apply to raw fp32 bits (truncate or
//     round-to-nearest)?  -> decides how the "lo" residual of 3xTF32 is formed.
//  2. Cycles per tcgen05.mma (M=128, K=8) for N = 16..256, operands in SMEM:
//     the skinny-N operand-bandwidth question (hard part 1).
//  3. TMA tiled load of a box {32 W, 8 C, 4 H} from an NCHW tensor whose map
//     lists dims as (W, C, H, N) with permuted strides, SWIZZLE_128B, lands in
//     exactly the canonical MN-major SW128 layout the MMA reads.
//
// Build+run: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tools/tc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version 1 (sm100)
    d |= (uint64_t)(layout & 7) << 61;
    return d;
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, a_major, b_major, N, M
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) |
           ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc,
                                         uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                     "r"(smem_u32(b)) : "memory");
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

// SWIZZLE_128B: 16B-chunk index (bits 4..6) ^= row-in-atom (bits 7..9); SW32: bit 4 ^= bit 7
__host__ __device__ inline uint32_t sw128(uint32_t off) { return off ^ (((off >> 7) & 7) << 4); }
__host__ __device__ inline uint32_t sw32(uint32_t off) { return off ^ (((off >> 7) & 1) << 4); }

// A operand layouts (M=128 x K=8 tf32) -- mode:
//  0 MN-major SW128   : m = blk*32 + px; atom blk at blk*1024 (LBO), K-row k at k*128
//  1 K-major  SW32    : 8-row groups of 32B rows at 256B (SBO)
//  2 K-major  INTERL. : core 8 rows x 16B; K halves at LBO=128, row groups at SBO=256
//  3 MN-major INTERL. : core 4 MN x 8 K (16B rows); MN blocks at SBO=128
__device__ inline uint32_t a_off(int mode, int m, int k) {
    switch (mode) {
        case 0: return sw128((m >> 5) * 1024 + k * 128 + (m & 31) * 4);
        case 1: return sw32((m >> 3) * 256 + (m & 7) * 32 + k * 4);
        case 2: return (m >> 3) * 256 + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4;
        default: return (m >> 2) * 128 + k * 16 + (m & 3) * 4;
    }
}
__device__ inline uint64_t a_desc(int mode, uint32_t base) {
    switch (mode) {
        case 0: return make_desc(base, 1024, 8192, 2);
        case 1: return make_desc(base, 16, 256, 6);
        case 2: return make_desc(base, 128, 256, 0);
        default: return make_desc(base, 8192, 128, 0);
    }
}
__device__ inline uint32_t b_off(int n, int k) {
    return (n >> 3) * 256 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4;
}

struct ProbeArgs {
    const float *A;  // [128][8] row-major (m, k)
    const float *B;  // [N][8]
    float *D;        // [128][N]
    int N;
    int reps;
    long long *cycles;
    int mode;
    int nacc;
};

__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
    return pred;
}

template <int N, int NACC>
__global__ void __launch_bounds__(128) mma_probe(ProbeArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char *sA = smem;                      // 4 KB (8 KB reserved)
    unsigned char *sB = smem + 8192;               // N*32 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int tid = threadIdx.x, warp = tid >> 5;
    const int mode = a.mode;
    for (int i = tid; i < 128 * 8; i += 128) {
        int m = i / 8, k = i % 8;
        *(float *)(sA + a_off(mode, m, k)) = a.A[i];
    }
    for (int i = tid; i < N * 8; i += 128) {
        int n = i / 8, k = i % 8;
        *(float *)(sB + b_off(n, k)) = a.B[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = tbase;
    uint64_t ad = a_desc(mode, smem_u32(sA));
    uint64_t bd = make_desc(smem_u32(sB), 128, 256, 0);
    const uint32_t idesc = make_idesc(128, N, (mode == 0 || mode == 3) ? 1 : 0, 0);
    if (warp == 0) {
        if (elect_one()) {
            mma_tf32(tm, ad, bd, idesc, 0);
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t0 = clock64();
        for (int r = 0; r < 512 / NACC; ++r) {
#pragma unroll
            for (int q = 0; q < NACC; ++q)
                if (elect_one()) mma_tf32(tm + 256 + q * N, ad, bd, idesc, r > 0);
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 1);
        if (tid == 0) a.cycles[0] = clock64() - t0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + c0, v);
        int m = warp * 32 + (tid & 31);
        for (int i = 0; i < 16; ++i) a.D[m * N + c0 + i] = v[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

// TMA probe: load box {32,8,4} of a (W,C,H,N)-ordered map of an NCHW tensor into smem
__global__ void tma_probe(const __grid_constant__ CUtensorMap tmap, float *out, int c0, int x0,
                          int y0, int n0) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, 4096);
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
            "[%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem)),
            "l"((uint64_t)&tmap), "r"(smem_u32(&bar)), "r"(x0), "r"(c0), "r"(y0), "r"(n0)
            : "memory");
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = ((float *)smem)[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static float tf32_trunc(float x) {
    uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x;
}
static float tf32_rn(float x) {
    uint32_t u; memcpy(&u, &x, 4);
    uint32_t lsb = (u >> 13) & 1; u += 0xFFF + lsb; u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x;
}

template <int N, int NACC>
static void run_mma(const char *label, int mode) {
    const int nacc = NACC;
    std::vector<float> A(128 * 8), B(N * 8), D(128 * N);
    srand(7 + N);
    for (auto &v : A) v = (float)rand() / RAND_MAX * 2 - 1;
    for (auto &v : B) v = (float)rand() / RAND_MAX * 2 - 1;
    float *dA, *dB, *dD; long long *dc;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    ProbeArgs a{dA, dB, dD, N, 512, dc, mode, nacc};
    int smem = 8192 + N * 32 + 1024;
    CK(cudaFuncSetAttribute(mma_probe<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    mma_probe<N, NACC><<<1, 128, smem>>>(a);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    long long cyc;
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    double e_tr = 0, e_rn = 0, e_raw = 0, scale = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double s_tr = 0, s_rn = 0, s_raw = 0;
            for (int k = 0; k < 8; ++k) {
                s_tr += (double)tf32_trunc(A[m * 8 + k]) * tf32_trunc(B[n * 8 + k]);
                s_rn += (double)tf32_rn(A[m * 8 + k]) * tf32_rn(B[n * 8 + k]);
                s_raw += (double)A[m * 8 + k] * B[n * 8 + k];
            }
            double d = D[m * N + n];
            e_tr = fmax(e_tr, fabs(d - s_tr)); e_rn = fmax(e_rn, fabs(d - s_rn));
            e_raw = fmax(e_raw, fabs(d - s_raw)); scale = fmax(scale, fabs(s_raw));
        }
    printf("  D[0][0..2] = %g %g %g | fp32 ref %g %g %g\n", D[0], D[1], D[2],
           A[0]*B[0]+A[1]*B[1]+A[2]*B[2]+A[3]*B[3]+A[4]*B[4]+A[5]*B[5]+A[6]*B[6]+A[7]*B[7],
           A[0]*B[8]+A[1]*B[9]+A[2]*B[10]+A[3]*B[11]+A[4]*B[12]+A[5]*B[13]+A[6]*B[14]+A[7]*B[15],
           A[0]*B[16]+A[1]*B[17]+A[2]*B[18]+A[3]*B[19]+A[4]*B[20]+A[5]*B[21]+A[6]*B[22]+A[7]*B[23]);
    printf("%s nacc=%d mode=%d N=%3d: maxerr vs trunc-tf32 %.3e, vs rn-tf32 %.3e, vs fp32 %.3e (scale %.2f); "
           "%.2f cycles/MMA (512 back-to-back)\n", label, nacc, mode, N, e_tr, e_rn, e_raw, scale,
           cyc / 512.0);
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
}

int main() {
    int dev = 0; CK(cudaSetDevice(dev));
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
    printf("device %s, %d SMs, clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
    for (int mode = 1; mode < 3; ++mode) {
        run_mma<16, 1>("mma", mode); run_mma<16, 2>("mma", mode); run_mma<16, 4>("mma", mode);
        run_mma<16, 8>("mma", mode);
        run_mma<32, 1>("mma", mode); run_mma<32, 2>("mma", mode); run_mma<32, 4>("mma", mode);
        run_mma<32, 8>("mma", mode);
        run_mma<64, 1>("mma", mode); run_mma<64, 2>("mma", mode); run_mma<64, 4>("mma", mode);
        run_mma<128, 1>("mma", mode); run_mma<128, 2>("mma", mode);
        run_mma<256, 1>("mma", mode);
    }
    return 0;

    // ---- TMA probe
    EncodeFn encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q));
    const int Nn = 2, C = 11, H = 13, W = 72;
    std::vector<float> X((size_t)Nn * C * H * W);
    for (size_t i = 0; i < X.size(); ++i) X[i] = (float)i;
    float *dX, *dOut;
    CK(cudaMalloc(&dX, X.size() * 4)); CK(cudaMalloc(&dOut, 4096));
    CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)Nn};
    cuuint64_t strides[3] = {(cuuint64_t)H * W * 4, (cuuint64_t)W * 4, (cuuint64_t)C * H * W * 4};
    cuuint32_t box[4] = {32, 8, 4, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dX, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    int c0 = 5, x0 = -3, y0 = 10, n0 = 1;
    tma_probe<<<1, 128, 4096 + 1024>>>(tm, dOut, c0, x0, y0, n0);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    std::vector<float> out(1024);
    CK(cudaMemcpy(out.data(), dOut, 4096, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int h = 0; h < 4; ++h)
        for (int k = 0; k < 8; ++k)
            for (int px = 0; px < 32; ++px) {
                int c = c0 + k, y = y0 + h, x = x0 + px;
                float want = (c < C && y < H && x >= 0 && x < W)
                                 ? X[(((size_t)n0 * C + c) * H + y) * W + x] : 0.f;
                uint32_t off = sw128(h * 1024 + k * 128 + px * 4);
                if (out[off / 4] != want) ++bad;
            }
    printf("TMA box {32,8,4} permuted-dims SW128 layout: %s (%d mismatches)\n",
           bad ? "MISMATCH" : "OK", bad);
    return 0;
}
