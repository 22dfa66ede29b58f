// stencil_kernel.cuh — one time step of a compiled 2:4-sparse stencil operator
// on sm_100a. The reference's hot loop (proj/core/src/emulator.cpp:134-193,
// tiled_sparse_matmul with the b_entry provider, scattered through
// output_position, layout.cpp:190-209) becomes, per CTA batch of
// TXB x TYB output tiles (tile = 16 x 8 outputs, D row m = dx*8 + dy):
//
//   warp 0      TMA producer: grid patch (+halo, zero-filled outside) -> smem,
//               NP-deep ring so several patches are in flight per SM
//   warps 2-5   gather: B''[q, tile] = patch[tile_origin + koff[q]] (the
//               memory map of layout.cpp:162-188), fp32 -> fp16 (RNE, the
//               reference round16 rounding), into the UMMA MN-major operand
//   warp 1      MMA issuer: tcgen05.mma.sp.cta_group::1.kind::f16, A'' from
//               smem (compressed, K-major), metadata from TMEM, D in TMEM
//   warps 6-9   epilogue: tcgen05.ld -> stores of the interior outputs
//
// mbarrier handshakes between roles, double-buffered B operand and TMEM
// accumulator, persistent CTAs (one per SM) striding over batches.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "sm100_ptx.cuh"

namespace sst {

constexpr int kThreads = 320;
constexpr int kGatherWarp0 = 2, kGatherWarps = 4;
constexpr int kEpiWarp0 = 6, kEpiWarps = 4;
constexpr int kTileW = 16, kTileH = 8;  // r1, r2
constexpr uint32_t kTmemCols = 256;

struct StepParams {
    const uint4* a_img;        // A'' smem image (fp16), nks * 4096 bytes
    const uint32_t* e_words;   // [nks][128]
    const int32_t* koff;       // [k_pad]
    const uint8_t* korder;     // [k_pad / 8]
    float* out;                // output storage buffer
    int64_t row_pitch;         // elements
    int64_t plane_pitch;       // elements
    int32_t left_pad;
    int32_t gx, gy, gz;        // logical extents
    int32_t r;                 // radius
    int32_t slow_lo, slow_hi;  // window over the slowest axis (y in 2D, z in 3D), interior coords
    int32_t y_end;             // interior rows (gy - 2r)
    int32_t nbx, nby, nbz, nbatch;
    int32_t k_pad, nks;
    int32_t patch_w, patch_h, patch_planes;
};

struct SmemLayout {
    uint32_t a, b, b_stride, p, p_stride, koff, korder, bars, tmem_slot, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

template <int TXB, int TYB, int NP>
__host__ __device__ inline SmemLayout smem_layout(int nks, int k_pad, int patch_w, int patch_h,
                                                  int planes) {
    constexpr int N = TXB * TYB;
    SmemLayout L{};
    uint32_t o = 0;
    L.a = o;
    o += static_cast<uint32_t>(nks) * 4096u;
    L.b_stride = align_up(static_cast<uint32_t>(k_pad) * N * 2u, 1024);
    L.b = o = align_up(o, 1024);
    o += 2 * L.b_stride;
    L.p_stride = align_up(static_cast<uint32_t>(patch_w * patch_h * planes) * 4u, 128);
    L.p = o = align_up(o, 128);
    o += NP * L.p_stride;
    L.koff = o = align_up(o, 16);
    o += static_cast<uint32_t>(k_pad) * 4u;
    L.korder = o = align_up(o, 16);
    o += static_cast<uint32_t>(k_pad / 8);
    L.bars = o = align_up(o, 8);
    o += (2 * NP + 8) * 8;
    L.tmem_slot = o;
    o += 16;
    L.total = align_up(o, 128);
    return L;
}

template <int DIMS, int TXB, int TYB, int NP>
__global__ void __launch_bounds__(kThreads, 1)
    stencil_step_kernel(const __grid_constant__ CUtensorMap tmap_in, const StepParams p) {
    static_assert(TXB == 8, "gather assumes 8 x-tiles per MMA column group");
    static_assert(TYB % 4 == 0 || TYB < 4, "gather warps split the tile rows");
    constexpr int N = TXB * TYB;
    static_assert(N % 16 == 0 && N <= 128, "UMMA N for M=128");
    using namespace ptx;

    extern __shared__ __align__(1024) uint8_t smem[];
    const SmemLayout L = smem_layout<TXB, TYB, NP>(p.nks, p.k_pad, p.patch_w, p.patch_h, p.patch_planes);
    uint8_t* sA = smem + L.a;
    uint8_t* sB = smem + L.b;     // 2 stages of b_stride bytes
    uint8_t* sP = smem + L.p;     // NP stages of p_stride bytes
    int32_t* sKoff = reinterpret_cast<int32_t*>(smem + L.koff);
    uint8_t* sKorder = smem + L.korder;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* patch_full = bars;
    uint64_t* patch_empty = bars + NP;
    uint64_t* b_full = bars + 2 * NP;
    uint64_t* b_empty = b_full + 2;
    uint64_t* d_full = b_full + 4;
    uint64_t* d_empty = b_full + 6;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        for (int s = 0; s < NP; ++s) {
            mbar_init(&patch_full[s], 1);
            mbar_init(&patch_empty[s], kGatherWarps);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&b_full[s], kGatherWarps);
            mbar_init(&b_empty[s], 1);
            mbar_init(&d_full[s], 1);
            mbar_init(&d_empty[s], kEpiWarps);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmap_in);
    }
    if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
    {  // constant operands: A'' image, gather tables
        const int n16 = p.nks * 4096 / 16;
        uint4* dstA = reinterpret_cast<uint4*>(sA);
        for (int i = threadIdx.x; i < n16; i += kThreads) dstA[i] = p.a_img[i];
        for (int i = threadIdx.x; i < p.k_pad; i += kThreads) sKoff[i] = p.koff[i];
        for (int i = threadIdx.x; i < p.k_pad / 8; i += kThreads) sKorder[i] = p.korder[i];
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t e_col = 2 * N;  // metadata columns after the two accumulators

    if (warp >= kEpiWarp0) {  // sparse metadata -> TMEM (each warp its lane quarter)
        const uint32_t q = static_cast<uint32_t>(warp % 4);
        for (int ks = 0; ks < p.nks; ++ks)
            tmem_st_32x32b_x1(tmem + ((q * 32u) << 16) + e_col + ks,
                              p.e_words[ks * 128 + q * 32 + lane]);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const int nbx = p.nbx, nby = p.nby;
    auto batch_coords = [&](int b, int& X0, int& Y0, int& Z0) {
        X0 = (b % nbx) * (TXB * kTileW);
        Y0 = ((b / nbx) % nby) * (TYB * kTileH) + (DIMS == 2 ? p.slow_lo : 0);
        Z0 = b / (nbx * nby) + (DIMS == 3 ? p.slow_lo : 0);
    };

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint32_t pbytes = static_cast<uint32_t>(p.patch_w * p.patch_h * p.patch_planes) * 4u;
            int it = 0;
            for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
                const int s = it % NP;
                const uint32_t ph = (it / NP) & 1;
                int X0, Y0, Z0;
                batch_coords(b, X0, Y0, Z0);
                mbar_wait(&patch_empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&patch_full[s], pbytes);
                // storage column X0 is 16-byte aligned (TMA requirement); the
                // window origin sits left_pad cells into the patch (koff has it)
                void* dst = sP + s * L.p_stride;
                if (DIMS == 2)
                    tma_load_2d(dst, &tmap_in, &patch_full[s], X0, Y0);
                else
                    tma_load_3d(dst, &tmap_in, &patch_full[s], X0, Y0, Z0);
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        const uint32_t idesc = make_idesc_f16(128, N, true, 0, 1);
        const uint32_t b_sbo = static_cast<uint32_t>(p.k_pad) * 16u;
        const uint32_t a0 = smem_u32(sA);
        int it = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            mbar_wait(&b_full[s], ph);
            mbar_wait(&d_empty[s], ph ^ 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t b0 = smem_u32(sB + s * L.b_stride);
                for (int ks = 0; ks < p.nks; ++ks) {
                    const uint64_t ad = make_smem_desc(a0 + ks * 4096u, 128, 256);
                    const uint64_t bd = make_smem_desc(b0 + ks * 512u, 128, b_sbo);
                    const uint32_t ea = tmem + e_col + static_cast<uint32_t>(ks);
                    mma_sp_f16(tmem + static_cast<uint32_t>(s * N), ad, bd, ea & ~1u,
                               idesc | (ea & 1u), ks > 0 ? 1u : 0u);
                }
                mma_commit(&b_empty[s]);
                mma_commit(&d_full[s]);
            }
            __syncwarp();
        }
    } else if (warp < kGatherWarp0 + kGatherWarps) {
        // ------------------------------------------------------------ gather
        // warp gw handles tile rows g = gw, gw + 4, ... for every K sweep j;
        // lane -> one B'' row k of the sweep, 8 tiles along x per 16-B store
        const int gw = warp - kGatherWarp0;
        const uint32_t row_stride = static_cast<uint32_t>(kTileH * p.patch_w) * 4u;
        int it = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int ps = it % NP;
            const uint32_t pph = (it / NP) & 1;
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            mbar_wait(&patch_full[ps], pph);
            mbar_wait(&b_empty[s], ph ^ 1);
            const uint32_t pbase = smem_u32(sP + ps * L.p_stride);
            const uint32_t bbase = smem_u32(sB + s * L.b_stride);
#pragma unroll 1
            for (int j = 0; j < p.nks; ++j) {
                const int k = sKorder[4 * j + static_cast<int>(lane / 8)] * 8 + static_cast<int>(lane % 8);
                const uint32_t src0 = pbase + static_cast<uint32_t>(sKoff[k]) * 4u;
                const uint32_t dst0 = bbase + static_cast<uint32_t>(k) * 16u;
#pragma unroll
                for (int g = gw; g < TYB; g += kGatherWarps) {
                    const uint32_t src = src0 + static_cast<uint32_t>(g) * row_stride;
                    float v[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[t]) : "r"(src + t * kTileW * 4));
                    uint32_t h[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const __half2 hv = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
                        h[i] = *reinterpret_cast<const uint32_t*>(&hv);
                    }
                    const uint32_t dst = dst0 + static_cast<uint32_t>(g * p.k_pad) * 16u;
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(h[0]),
                                 "r"(h[1]), "r"(h[2]), "r"(h[3])
                                 : "memory");
                }
            }
            fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&b_full[s]);
                mbar_arrive(&patch_empty[ps]);
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        const uint32_t q = static_cast<uint32_t>(warp % 4);
        const int m = static_cast<int>(q * 32 + lane);
        const int dx = m / kTileH, dy = m % kTileH;
        const int x_end = p.gx - p.r, y_end = DIMS == 2 ? p.slow_hi : p.y_end;
        const int64_t tile_row = static_cast<int64_t>(kTileH) * p.row_pitch;
        int it = 0;
        for (int b = blockIdx.x; b < p.nbatch; b += gridDim.x, ++it) {
            const int s = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            int X0, Y0, Z0;
            batch_coords(b, X0, Y0, Z0);
            // output (x, y) of D row m, tile (0, 0) of the batch
            const int x0 = X0 + dx + p.r, y0 = Y0 + dy;  // y0: interior row
            float* o = p.out + (DIMS == 3 ? static_cast<int64_t>(Z0 + p.r) * p.plane_pitch : 0) +
                       static_cast<int64_t>(y0 + p.r) * p.row_pitch + p.left_pad + x0;
            const bool full = X0 + TXB * kTileW + p.r <= x_end && Y0 + TYB * kTileH <= y_end;
            mbar_wait(&d_full[s], ph);
            tc_fence_after();
#pragma unroll 1
            for (int c0 = 0; c0 < N; c0 += 16) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tmem + ((q * 32u) << 16) + static_cast<uint32_t>(s * N + c0), v);
                tmem_wait_ld();
                if (full) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int n = c0 + i;
                        o[(n / TXB) * tile_row + (n % TXB) * kTileW] = __uint_as_float(v[i]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int n = c0 + i;
                        const bool ok = x0 + (n % TXB) * kTileW < x_end && y0 + (n / TXB) * kTileH < y_end;
                        if (ok) o[(n / TXB) * tile_row + (n % TXB) * kTileW] = __uint_as_float(v[i]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d_empty[s]);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
    }
}

}  // namespace sst
