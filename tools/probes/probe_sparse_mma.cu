// Hardware probe: pins down the tcgen05.mma.sp kind::f16 operand conventions
// the stencil kernel relies on (A K-major interleaved compressed operand,
// B MN-major or K-major interleaved, metadata written to TMEM with
// tcgen05.st). Runs one CTA, M=128, N=64, K=64 (two K-steps), exact integer
// data, and reports the max error of every (B layout, E layout) combination
// against a CPU product.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_fp16.h>
#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"

using namespace sst::ptx;

constexpr int M = 128, N = 64, K = 64, KS = K / 32;

struct Args {
    const __half* a_img;   // M x K/2 compressed, smem image (K-major interleave)
    const __half* b_img;   // K x N smem image
    const uint32_t* e_words;  // [KS][128]
    float* d;              // M x N
    int b_mn;              // 1: B MN-major image, 0: K-major
};

__global__ void probe(Args args) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __half* sa = reinterpret_cast<__half*>(smem);                 // 8 KB
    __half* sb = reinterpret_cast<__half*>(smem + 8192);          // 8 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < M * K / 2; i += blockDim.x) sa[i] = args.a_img[i];
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
    const uint32_t ecol = 128;
    for (int s = 0; s < KS; ++s) {
        uint32_t w = args.e_words[s * 128 + warp * 32 + lane_id()];
        tmem_st_32x32b_x1(tb + ((uint32_t)(warp * 32) << 16) + ecol + s, w);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint32_t idesc = make_idesc_f16(M, N, true, 0, args.b_mn);
        for (int s = 0; s < KS; ++s) {
            // A: per K-step block of 4096 B; LBO (K dir) 128 B, SBO (M dir) 256 B
            uint64_t ad = make_smem_desc(smem_u32(sa) + s * 4096, 128, 256);
            uint64_t bd;
            if (args.b_mn) {
                // B MN-major: unit(n,k) = (n/8)*SBO + (k/8)*LBO + k%8; LBO=128, SBO=(K/8)*128
                bd = make_smem_desc(smem_u32(sb) + s * 4 * 128, 128, (K / 8) * 128);
            } else {
                // B K-major: unit(n,k) = (n/8)*SBO + (k/8)*LBO + n%8; LBO=128, SBO=(K/8)*128
                bd = make_smem_desc(smem_u32(sb) + s * 4 * 128, 128, (K / 8) * 128);
            }
            // metadata address is 2-column granular: the low column bit goes to sparse_id2
            const uint32_t ea = tb + ecol + s;
            mma_sp_f16(tb, ad, bd, ea & ~1u, idesc | (ea & 1u), s > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c = 0; c < N; c += 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tb + ((uint32_t)(warp * 32) << 16) + c, r);
        tmem_wait_ld();
        for (int j = 0; j < 16; ++j)
            args.d[(warp * 32 + lane_id()) * N + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 256);
}

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

int main() {
    std::mt19937 rng(7);
    // logical A: M x K, 2:4 per 4-group, small ints
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
    // A image: s*2048 elems + (m/8)*128 + (j/8)*64 + (m%8)*8 + j%8  (in halves)
    std::vector<__half> aimg(M * K / 2);
    for (int m = 0; m < M; ++m)
        for (int jj = 0; jj < K / 2; ++jj) {
            int s = jj / 16, j = jj % 16;
            size_t off = s * 2048 + (m / 8) * 128 + (j / 8) * 64 + (m % 8) * 8 + j % 8;
            aimg[off] = __float2half(vals[m * (K / 2) + jj]);
        }
    std::vector<__half> bmn(K * N), bk(K * N);
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) {
            // MN-major: unit = (n/8)*(K/8) + (k/8)*8 ... in halves: unit*8 + n%8
            size_t u_mn = (n / 8) * (K / 8) * 8 + (k / 8) * 8 + (k % 8);
            bmn[u_mn * 8 + n % 8] = __float2half(B[k * N + n]);
            size_t u_k = (n / 8) * (K / 8) * 8 + (k / 8) * 8 + (n % 8);
            bk[u_k * 8 + k % 8] = __float2half(B[k * N + n]);
        }
    // E layouts
    std::vector<uint32_t> e_cutlass(KS * 128, 0), e_naive(KS * 128, 0);
    for (int s = 0; s < KS; ++s)
        for (int m = 0; m < M; ++m)
            for (int gl = 0; gl < 8; ++gl) {
                uint32_t nib = meta[m * (K / 4) + s * 8 + gl];
                // naive: lane = m, nibble gl
                e_naive[s * 128 + m] |= nib << (4 * gl);
                // cutlass-derived: m = m0 + 8 m1 + 16 m2 ; gl = g_local + 4 k1
                int m0 = m % 8, m1 = (m / 8) % 2, m2 = m / 16;
                int g_local = gl % 4, k1 = gl / 4;
                int lane = m0 + 8 * k1 + 16 * m2;
                int nibidx = g_local + 4 * m1;
                e_cutlass[s * 128 + lane] |= nib << (4 * nibidx);
            }
    __half *da, *db;
    uint32_t* de;
    float* dd;
    CK(cudaMalloc(&da, aimg.size() * 2));
    CK(cudaMalloc(&db, K * N * 2));
    CK(cudaMalloc(&de, KS * 128 * 4));
    CK(cudaMalloc(&dd, M * N * 4));
    CK(cudaMemcpy(da, aimg.data(), aimg.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    const char* bnames[2] = {"B K-major", "B MN-major"};
    const char* enames[2] = {"E cutlass-layout", "E naive lane=row"};
    for (int bmode = 0; bmode < 2; ++bmode)
        for (int emode = 0; emode < 2; ++emode) {
            CK(cudaMemcpy(db, bmode ? bmn.data() : bk.data(), K * N * 2, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(de, emode ? e_naive.data() : e_cutlass.data(), KS * 128 * 4,
                          cudaMemcpyHostToDevice));
            CK(cudaMemset(dd, 0, M * N * 4));
            Args a{da, db, de, dd, bmode};
            probe<<<1, 128, 32768>>>(a);
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
            printf("%s, %s: max_err=%g mismatches=%d/%d  d[0..3]=%g %g %g %g ref=%g %g %g %g\n",
                   bnames[bmode], enames[emode], maxerr, bad, M * N, out[0], out[1], out[2],
                   out[3], ref[0], ref[1], ref[2], ref[3]);
        }
    return 0;
}
