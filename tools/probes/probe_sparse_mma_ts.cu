// Hardware probe: tcgen05.mma.sp kind::f16 with the compressed A operand in
// TMEM ("[a-tmem]" form, SASS UTCHMMA tmem[A]) instead of shared memory.
// M=128, N=64, K=64 (two K-steps), exact integer data; B MN-major in smem and
// metadata in TMEM as the stencil kernel uses them (probe_sparse_mma.cu).
// Tries candidate A layouts: lane = row, K-step s at column base + s*8, and
// compressed element j of the step at
//   L1: column j/2, half j%2      L3: column j%8, half j/8
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_fp16.h>
#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"

using namespace sst::ptx;

constexpr int M = 128, N = 64, K = 64, KS = K / 32;

__device__ __forceinline__ void mma_sp_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t e_tmem, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%3], %4, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(e_tmem), "r"(idesc), "r"(acc)
        : "memory");
}

struct Args {
    const uint32_t* a_words;  // [M][KS*8] TMEM words (two halves each)
    const __half* b_img;      // K x N smem image, MN-major
    const uint32_t* e_words;  // [KS][128]
    float* d;
    int a_step_cols;          // TMEM column advance per K step
};

__global__ void probe(Args args) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __half* sb = reinterpret_cast<__half*>(smem);
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < K * N; i += blockDim.x) sb[i] = args.b_img[i];
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&tmem_base, 256);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base;
    const uint32_t ecol = 128, acol = 160;
    const uint32_t lanebase = tb + ((uint32_t)(warp * 32) << 16);
    for (int s = 0; s < KS; ++s)
        tmem_st_32x32b_x1(lanebase + ecol + s, args.e_words[s * 128 + warp * 32 + lane_id()]);
    for (int c = 0; c < KS * 8; ++c)
        tmem_st_32x32b_x1(lanebase + acol + c, args.a_words[(warp * 32 + lane_id()) * (KS * 8) + c]);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint32_t idesc = make_idesc_f16(M, N, true, 0, 1);
        for (int s = 0; s < KS; ++s) {
            const uint64_t bd = make_smem_desc(smem_u32(sb) + s * 4 * 128, 128, (K / 8) * 128);
            const uint32_t ea = tb + ecol + s;
            mma_sp_f16_ts(tb, tb + acol + s * args.a_step_cols, bd, ea & ~1u, idesc | (ea & 1u), s > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c = 0; c < N; c += 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(lanebase + c, r);
        tmem_wait_ld();
        for (int j = 0; j < 16; ++j) args.d[(warp * 32 + lane_id()) * N + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 256);
}

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

static uint16_t h16(float f) {
    __half h = __float2half(f);
    return *reinterpret_cast<uint16_t*>(&h);
}

int main() {
    std::mt19937 rng(7);
    std::vector<float> A(M * K, 0.f), B(K * N);
    std::vector<uint8_t> meta(M * K / 4);
    std::vector<float> vals(M * K / 2);
    for (int m = 0; m < M; ++m)
        for (int g = 0; g < K / 4; ++g) {
            int p0 = rng() % 3, p1 = p0 + 1 + rng() % (3 - p0);
            float v0 = float(int(rng() % 7) - 3), v1 = float(int(rng() % 7) - 3);
            A[m * K + 4 * g + p0] = v0;
            A[m * K + 4 * g + p1] = v1;
            vals[m * (K / 2) + 2 * g] = v0;
            vals[m * (K / 2) + 2 * g + 1] = v1;
            meta[m * (K / 4) + g] = uint8_t(p0 | (p1 << 2));
        }
    for (auto& v : B) v = float(int(rng() % 9) - 4);
    std::vector<double> ref(M * N, 0.0);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double acc = 0;
            for (int k = 0; k < K; ++k) acc += double(A[m * K + k]) * B[k * N + n];
            ref[m * N + n] = acc;
        }
    std::vector<__half> bmn(K * N);
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) {
            size_t u_mn = (n / 8) * (K / 8) * 8 + (k / 8) * 8 + (k % 8);
            bmn[u_mn * 8 + n % 8] = __float2half(B[k * N + n]);
        }
    std::vector<uint32_t> e_words(KS * 128, 0);
    for (int s = 0; s < KS; ++s)
        for (int m = 0; m < M; ++m)
            for (int gl = 0; gl < 8; ++gl) {
                uint32_t nib = meta[m * (K / 4) + s * 8 + gl];
                int m0 = m % 8, m1 = (m / 8) % 2, m2 = m / 16;
                int lane = m0 + 8 * (gl / 4) + 16 * m2;
                e_words[s * 128 + lane] |= nib << (4 * ((gl % 4) + 4 * m1));
            }
    __half* db;
    uint32_t *de, *da;
    float* dd;
    CK(cudaMalloc(&db, K * N * 2));
    CK(cudaMalloc(&de, KS * 128 * 4));
    CK(cudaMalloc(&da, M * KS * 8 * 4));
    CK(cudaMalloc(&dd, M * N * 4));
    CK(cudaMemcpy(db, bmn.data(), K * N * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(de, e_words.data(), KS * 128 * 4, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
    for (int layout = 1; layout <= 3; layout += 2)
        for (int step_cols : {8, 16}) {
            std::vector<uint32_t> aw(M * KS * 8, 0);
            for (int m = 0; m < M; ++m)
                for (int jj = 0; jj < K / 2; ++jj) {
                    const int s = jj / 16, j = jj % 16;
                    const int col = layout == 1 ? j / 2 : j % 8, half = layout == 1 ? j % 2 : j / 8;
                    aw[m * (KS * 8) + s * 8 + col] |= uint32_t(h16(vals[m * (K / 2) + jj])) << (16 * half);
                }
            if (step_cols == 16) continue;  // the A words are packed at 8 columns per step
            CK(cudaMemcpy(da, aw.data(), aw.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemset(dd, 0, M * N * 4));
            Args a{da, db, de, dd, step_cols};
            probe<<<1, 128, 16384>>>(a);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            std::vector<float> out(M * N);
            CK(cudaMemcpy(out.data(), dd, M * N * 4, cudaMemcpyDeviceToHost));
            double maxerr = 0;
            int bad = 0;
            for (int i = 0; i < M * N; ++i) {
                double e = std::fabs(out[i] - ref[i]);
                maxerr = std::max(maxerr, e);
                bad += e > 0;
            }
            printf("A in TMEM layout L%d, %d cols/step: max_err=%g mismatches=%d/%d d[0..3]=%g %g %g %g ref=%g %g %g %g\n",
                   layout, step_cols, maxerr, bad, M * N, out[0], out[1], out[2], out[3], ref[0], ref[1],
                   ref[2], ref[3]);
        }
    return 0;
}
