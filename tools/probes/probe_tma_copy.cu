// Hardware probe: the DRAM ceiling of the stencil kernels' ACCESS PATTERN alone.
// A persistent TMA copy over an 8192 x 8192 fp32 grid with the 2D kernel's boxes
// (load {136, 66} patches, store 4 x {32, 64} boxes per 128 x 64 batch, batches
// x-fastest, 148 CTAs, NP loads in flight) and, for comparison, contiguous 1D bulk
// copies of the same bytes. No compute: what the memory system gives this pattern.
// Usage: probe_tma_copy [np=3]
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int kN = 8192, kBW = 128, kBH = 64, kPW = 136, kPH = 66, kMaxNP = 4;
constexpr int kNbx = kN / kBW, kNby = (kN - 2) / kBH;

struct Smem {
    alignas(128) float patch[kMaxNP][(kPW * kPH + 31) / 32 * 32];  // TMA destinations: 128-byte aligned
    alignas(1024) float out[4][32 * kBH];
    uint64_t full[kMaxNP];
};

// mode 0: box pattern (patch loads + 4 store boxes); 1: loads only; 2: stores only
__global__ void __launch_bounds__(32, 1) box_copy(const __grid_constant__ CUtensorMap tin,
                                                  const __grid_constant__ CUtensorMap tout, int np, int mode) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw + ((1024u - (sst::ptx::smem_u32(raw) & 1023u)) & 1023u));
    if (threadIdx.x != 0) return;
    for (int s = 0; s < np; ++s) sst::ptx::mbar_init(&S.full[s], 1);
    sst::ptx::fence_mbar_init();
    const int nb = kNbx * kNby;
    int it = 0;
    for (int b = blockIdx.x; b < nb; b += gridDim.x, ++it) {
        const int X0 = (b % kNbx) * kBW, Y0 = (b / kNbx) * kBH;
        const int s = it % np;
        if (mode != 2) {
            if (it >= np) sst::ptx::mbar_wait(&S.full[s], ((it / np) - 1) & 1);
            sst::ptx::mbar_arrive_expect_tx(&S.full[s], kPW * kPH * 4);
            sst::ptx::tma_load_2d(S.patch[s], &tin, &S.full[s], X0 > 4 ? X0 - 4 : 0, Y0);
        }
        if (mode != 1) {
            for (int c = 0; c < 4; ++c) sst::ptx::tma_store_2d(&tout, S.out[c], X0 + 32 * c, Y0 + 1);
            sst::ptx::bulk_commit();
            sst::ptx::bulk_wait_read<4>();
        }
    }
    if (mode != 2)
        for (int j = (it > np ? it - np : 0); j < it; ++j) sst::ptx::mbar_wait(&S.full[j % np], (j / np) & 1);
    sst::ptx::bulk_wait<0>();
}

// box loads by TMA (warp 0, as above) + the 128 x 64 output of each batch written with
// coalesced 16-byte LSU stores by 4 warps (a warp writes 512 contiguous bytes per row);
// cs: st.global.cs (streaming) instead of st.global
template <bool CS>
__global__ void __launch_bounds__(160, 1) box_lsu(const __grid_constant__ CUtensorMap tin, float* out, int np,
                                                  int loads) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw + ((1024u - (sst::ptx::smem_u32(raw) & 1023u)) & 1023u));
    const int nb = kNbx * kNby;
    if (threadIdx.x < 32) {
        if (threadIdx.x != 0 || !loads) return;
        for (int s = 0; s < np; ++s) sst::ptx::mbar_init(&S.full[s], 1);
        sst::ptx::fence_mbar_init();
        int it = 0;
        for (int b = blockIdx.x; b < nb; b += gridDim.x, ++it) {
            const int X0 = (b % kNbx) * kBW, Y0 = (b / kNbx) * kBH;
            const int s = it % np;
            if (it >= np) sst::ptx::mbar_wait(&S.full[s], ((it / np) - 1) & 1);
            sst::ptx::mbar_arrive_expect_tx(&S.full[s], kPW * kPH * 4);
            sst::ptx::tma_load_2d(S.patch[s], &tin, &S.full[s], X0 > 4 ? X0 - 4 : 0, Y0);
        }
        for (int j = (it > np ? it - np : 0); j < it; ++j) sst::ptx::mbar_wait(&S.full[j % np], (j / np) & 1);
        return;
    }
    const int t = threadIdx.x - 32, w = t / 32, lane = t % 32;
    const float4* src = reinterpret_cast<const float4*>(S.out[0]);
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
        const int X0 = (b % kNbx) * kBW, Y0 = (b / kNbx) * kBH + 1;
        for (int row = w; row < kBH; row += 4) {
            const float4 v = src[(row * 32 + lane) & 2047];
            float4* dst = reinterpret_cast<float4*>(out + static_cast<size_t>(Y0 + row) * kN + X0) + lane;
            if (CS)
                asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                             "f"(v.w) : "memory");
            else
                *dst = v;
        }
    }
}

// contiguous: each CTA copies 32 KB chunks (same total bytes as one batch's load + store)
__global__ void __launch_bounds__(32, 1) linear_copy(const float* in, float* out, size_t chunks, int np) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw + ((1024u - (sst::ptx::smem_u32(raw) & 1023u)) & 1023u));
    if (threadIdx.x != 0) return;
    for (int s = 0; s < np; ++s) sst::ptx::mbar_init(&S.full[s], 1);
    sst::ptx::fence_mbar_init();
    constexpr uint32_t kChunk = 32768;
    int it = 0;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x, ++it) {
        const int s = it % np;
        if (it >= np) {
            sst::ptx::mbar_wait(&S.full[s], ((it / np) - 1) & 1);
        }
        sst::ptx::mbar_arrive_expect_tx(&S.full[s], kChunk);
        sst::ptx::bulk_copy_g2s(S.patch[s], reinterpret_cast<const uint8_t*>(in) + c * kChunk, kChunk, &S.full[s]);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         reinterpret_cast<uint8_t*>(out) + c * kChunk),
                     "r"(sst::ptx::smem_u32(S.out[0])), "r"(kChunk)
                     : "memory");
        sst::ptx::bulk_commit();
        sst::ptx::bulk_wait_read<4>();
    }
    for (int j = (it > np ? it - np : 0); j < it; ++j) sst::ptx::mbar_wait(&S.full[j % np], (j / np) & 1);
    sst::ptx::bulk_wait<0>();
}

int main(int argc, char** argv) {
    const int np = argc > 1 ? std::atoi(argv[1]) : 3;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<EncodeTiledFn>(fn);
    const size_t cells = static_cast<size_t>(kN) * kN;
    float *a, *b;
    cudaMalloc(&a, cells * 4);
    cudaMalloc(&b, cells * 4);
    cudaMemset(a, 0, cells * 4);
    cudaMemset(b, 0, cells * 4);
    CUtensorMap tin, tout;
    cuuint64_t dim[2] = {kN, kN}, stride[1] = {kN * 4};
    cuuint32_t pbox[2] = {kPW, kPH}, obox[2] = {32, kBH}, es[2] = {1, 1};
    encode(&tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dim, stride, pbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    encode(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b, dim, stride, obox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = static_cast<int>(sizeof(Smem)) + 1024;  // slack for the 1 KiB base alignment
    cudaFuncSetAttribute(box_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(linear_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double nbatch = static_cast<double>(kNbx) * kNby;
    const double alg = nbatch * kBW * kBH * 8.0;  // 8 B per output cell
    const char* names[3] = {"box pattern (load + store)", "box loads only", "box stores only"};
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            box_copy<<<sms, 32, smem>>>(tin, tout, np, mode);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        const double bytes = nbatch * ((mode != 2 ? kPW * kPH * 4.0 : 0) + (mode != 1 ? kBW * kBH * 4.0 : 0));
        printf("%-28s np %d: %8.1f us  moved %7.1f GB/s  algorithmic(8 B/cell) %7.1f GB/s\n", names[mode], np,
               best * 1e3, bytes / (best * 1e-3) / 1e9, mode == 0 ? alg / (best * 1e-3) / 1e9 : 0.0);
    }
    cudaFuncSetAttribute(box_lsu<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(box_lsu<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int variant = 0; variant < 4; ++variant) {
        const bool cs = variant & 1, loads = variant < 2;
        float bst = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (cs)
                box_lsu<true><<<sms, 160, smem>>>(tin, b, np, loads);
            else
                box_lsu<false><<<sms, 160, smem>>>(tin, b, np, loads);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            bst = std::min(bst, ms);
        }
        const double bytes = nbatch * ((loads ? kPW * kPH * 4.0 : 0) + kBW * kBH * 4.0);
        printf("%-28s np %d: %8.1f us  moved %7.1f GB/s  algorithmic(8 B/cell) %7.1f GB/s\n",
               loads ? (cs ? "TMA loads + LSU st.cs" : "TMA loads + LSU st") : (cs ? "LSU st.cs only" : "LSU st only"),
               np, bst * 1e3, bytes / (bst * 1e-3) / 1e9, loads ? alg / (bst * 1e-3) / 1e9 : 0.0);
    }
    float best = 1e30f;
    const size_t chunks = cells * 4 / 32768;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        linear_copy<<<sms, 32, smem>>>(a, b, chunks, np);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    printf("%-28s np %d: %8.1f us  moved %7.1f GB/s\n", "linear 32 KB bulk copies", np, best * 1e3,
           2.0 * cells * 4 / (best * 1e-3) / 1e9);
    printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
