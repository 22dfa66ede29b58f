// stencil_common.cuh — pieces shared by the sm_100a stencil kernels:
// launch parameters, constant-operand staging, the B'' gather, and the
// TMEM -> swizzled smem -> TMA-store epilogue of one 32-wide output box.
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
constexpr int kTXB = 8;                 // tiles per batch along x (128 outputs)
constexpr int kBoxW = 32;               // output box width (128 B, SWIZZLE_128B)
constexpr uint32_t kEpiBarrier = 1;     // named barrier of the 4 epilogue warps
constexpr int kStageBufs = 1;           // batch staging buffers (TMA stores in flight)

// Load (patch) and store (interior) tensor maps of both ping-pong buffers.
struct MapSet {
    CUtensorMap in[2];
    CUtensorMap out[2];
    CUtensorMap ring[2];  // 3D stream kernel: {4, TYB*8, 1} boxes of the right-edge chunk (kEdgeRing)
};

// Slab decomposition with peer-to-peer halos: the neighbours' halo slices in their
// buffers (by output parity), addressed in this rank's interior coordinates. Kept in
// global memory (TMA reads tensor maps from .global too) rather than in the kernel
// parameters: a larger parameter block measurably slowed L2-cold launches.
struct PeerMaps {
    CUtensorMap up[2];
    CUtensorMap down[2];
};

// Grouped launches (sst_run_steps_batch over identical grids): one launch advances every
// grid of the group by one step; per grid its patch-load and store maps and its output
// buffer, in global memory (TMA reads tensor maps from .global)
struct GroupMaps {
    CUtensorMap in;
    CUtensorMap out;
    float* out_buf;
    uint64_t pad[15];  // 64-byte aligned entries
};

struct StepParams {
    const uint4* a_img;        // A'' smem image (fp16), nks * 4096 bytes
    const uint32_t* e_words;   // [nks][128]
    const int32_t* gsrc;       // [k_pad/32][32] packed: (patch byte offset of the lane's B'' row) / 2
                               //   | (that row's index in an 8-tile group) << 16
    const int32_t* gdst;       // [k_pad/32][32] the row's byte offset (unpacked; staged, not read)
    float* buf[2];             // ping-pong storage buffers (right-edge columns, see epilogue)
    int32_t src;               // buffer holding the input of the launch's first step
    int32_t nsteps;            // time steps (operator applications) in this launch
    uint32_t* flags;           // [nbatch] per-batch step counters (multi-step launches)
    uint32_t flag_base;        // counter value meaning "step 0 of this launch not yet done"
    int64_t row_pitch, plane_pitch;  // storage pitches (elements)
    int32_t left_pad;
    int32_t load_x0;           // storage column of the patch start relative to X0 (16B aligned)
    int32_t load_y0;           // patch row offset: 0, or -r for a 1D fold's view (no ring rows)
    int32_t gx, gy, gz;        // logical extents
    int32_t r;                 // radius
    int32_t slow_lo, slow_hi;  // window over the slowest axis (y in 2D, z in 3D), interior coords
    int32_t y_end;             // interior rows (gy - 2r)
    int32_t nbx, nby, nbz, nbatch;
    int32_t nby1, slow_lo2;    // 2D two-window launches (kModePeer): batch rows [nby1, nby) cover the
                               // second window, starting at row slow_lo2 (nby1 == nby: one window)
    int32_t k_pad;             // B'' rows per MMA pass (per z slice when streaming)
    int32_t nks;               // 32-wide K steps in the A'' image (all slices)
    int32_t patch_w, patch_h, patch_planes;
    int32_t debug_mode;        // ablation bits (profiling only): 1 no stores, 2 no gather, 4 no MMA,
                               // 8 no right-edge plain stores, 16 TMA loads only (3D),
                               // 32 stores only (zeros), 64 staging without TMA stores,
                               // 128 TMA stores without staging
    int32_t tmem_cols;         // TMEM allocation (power of two >= the kernel's column budget)
    int32_t zchunk;            // 3D stream kernel: output planes per (band, z-chunk) run; 0 = whole column
    int32_t lo_sweep0;         // first gather sweep writing B_lo rows (SST_PREC_F16X2); = k_pad/32 otherwise
    const PeerMaps* peer_maps; // slab P2P halos (device memory), or null
    int32_t peer_mask;         // slab P2P halos: 1 = upper neighbour (lower slices), 2 = lower neighbour
    int32_t peer_down0;        // first interior slice that is the lower neighbour's halo (n_int - r)
    int32_t peer_down_c0;      // slice coordinate origin of the lower neighbour's map (>= 0 coordinates)
    int64_t peer_up_shift;     // (2D plain edge stores) storage-row shift into the upper neighbour's buffer
    int64_t peer_down_shift;   // ... into the lower neighbour's buffer
    float* peer_up_buf[2];     // neighbours' buffers by parity (plain right-edge stores)
    float* peer_down_buf[2];
    uint32_t* sched;           // 2D single-step launches: global batch counter (dynamic scheduling), or null
    uint32_t sched_base;       // counter value at launch start
    int32_t multi_dyn;         // 2D: the multi-step launch with dynamic batch ownership (kModeMultiDyn)
    unsigned long long* trace; // profiling only (sst_plan_set_trace): per CTA {smid, t_start, t_main, t_end}
    const float* fold_ring;    // 1D fold: the r right-ring cells' input values (else null)
    int64_t fold_nint;         // 1D fold: interior cells n_int = N - 2r (ring at [n_int, n_int + r))
    int32_t fold_w;            // 1D fold: interior cells per view row
    const GroupMaps* group;    // grouped launch (kModeGroup): per grid maps, group_n grids of nbatch batches
    int32_t group_n;
    int32_t reverse;           // dynamic single-step launches: batches drawn in reverse order
};

// Ablation bits (tools/ablate.py) are compiled in only with SST_ABLATION=1 (build
// env): a branch in the epilogue costs store throughput even when never taken.
#ifndef SST_ABLATION
#define SST_ABLATION 0
#endif
__device__ __forceinline__ int dbg(const StepParams& p) { return SST_ABLATION ? p.debug_mode : 0; }

__device__ __forceinline__ float* buf_of(const StepParams& p, int i) {
    return (i & 1) ? p.buf[1] : p.buf[0];  // select, not a dynamic param-space index
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// TMEM column budget of a kernel: accumulators, then the nks metadata columns,
// then (A in TMEM) 8 columns per K step starting on a 32-column boundary.
struct TmemCols {
    uint32_t e_col, a_col, need;
};
__host__ __device__ constexpr TmemCols tmem_budget(uint32_t acc_cols, uint32_t nks, bool a_in_tmem) {
    const uint32_t e = acc_cols, a = (acc_cols + nks + 31u) / 32u * 32u;
    return TmemCols{e, a, a_in_tmem ? a + nks * 8u : acc_cols + nks};
}

// tile (column n of the MMA) -> (tx, ty) of the batch: output box c (32 x-cells,
// tiles tx = 2c, 2c+1) owns columns [c*2*TYB, (c+1)*2*TYB), n = c*2*TYB + 2*ty + (tx & 1)
template <int TYB>
__host__ __device__ inline void tile_of_column(int n, int& tx, int& ty) {
    const int c = n / (2 * TYB), m = n % (2 * TYB);
    ty = m / 2;
    tx = 2 * c + (m & 1);
}

// Prologue staging, global -> smem by 1D bulk copies (TMA engine, one thread;
// a thread-strided copy loop is load-latency bound: 4.3 us for the 81 KiB of the
// 3D constants): the A'' image (to its smem home, or to `scratch` when it goes to
// TMEM), the TMEM metadata words (to `scratch`) and the gather tables. `scratch`
// is the B'' / staging / patch region, idle until the main loop; the host checks it
// is large enough. Call from one thread after pbar's init; everyone then waits on
// pbar (phase 0) after a CTA barrier.
template <bool AT>
__device__ __forceinline__ void stage_constants_issue(const StepParams& p, uint8_t* sA, uint8_t* scratch,
                                                      int32_t* sGsrc, int32_t* sGdst, uint64_t* pbar) {
    const uint32_t a_bytes = static_cast<uint32_t>(p.nks) * 4096u;
    const uint32_t e_bytes = static_cast<uint32_t>(p.nks) * 512u;
    const uint32_t t_bytes = static_cast<uint32_t>(p.k_pad) * 4u;
    ptx::mbar_arrive_expect_tx(pbar, a_bytes + e_bytes + 2 * t_bytes);
    ptx::bulk_copy_g2s(AT ? scratch : sA, p.a_img, a_bytes, pbar);
    ptx::bulk_copy_g2s(scratch + (AT ? a_bytes : 0u), p.e_words, e_bytes, pbar);
    ptx::bulk_copy_g2s(sGsrc, p.gsrc, t_bytes, pbar);
    ptx::bulk_copy_g2s(sGdst, p.gdst, t_bytes, pbar);
}
__host__ __device__ inline uint32_t prologue_scratch_bytes(int nks, bool a_in_tmem) {
    return static_cast<uint32_t>(nks) * ((a_in_tmem ? 4096u : 0u) + 512u);
}

// 2:4 metadata -> TMEM columns [e_col, e_col + nks) (each epilogue warp its lane
// quarter), from the words staged in smem
template <bool AT>
__device__ __forceinline__ void store_metadata(const StepParams& p, const uint8_t* scratch, uint32_t tmem,
                                               uint32_t e_col, uint32_t q, uint32_t lane) {
    const uint32_t* sE = reinterpret_cast<const uint32_t*>(scratch + (AT ? p.nks * 4096 : 0));
    for (int ks = 0; ks < p.nks; ++ks)
        ptx::tmem_st_32x32b_x1(tmem + ((q * 32u) << 16) + e_col + ks, sE[ks * 128 + q * 32 + lane]);
    ptx::tmem_wait_st();
}

// Compressed A'' -> TMEM columns [a_col, a_col + 8 nks) (each epilogue warp its lane
// quarter): lane = A row m, K step s in 8 columns, kept values (2c, 2c+1) of the
// step packed in column c. The staged image is the UMMA K-major interleave
// (halves: s*2048 + (m/8)*128 + (j/8)*64 + (m%8)*8 + j%8), so each TMEM word is one
// aligned 32-bit smem load.
__device__ __forceinline__ void store_a_tmem(const StepParams& p, const uint8_t* scratch, uint32_t tmem,
                                             uint32_t a_col, uint32_t q, uint32_t lane) {
    const uint32_t m = q * 32u + lane;
    const uint32_t* a32 = reinterpret_cast<const uint32_t*>(scratch);
    for (int s = 0; s < p.nks; ++s) {
        uint32_t w[8];
#pragma unroll
        for (uint32_t c = 0; c < 8; ++c)
            w[c] = a32[static_cast<uint32_t>(s) * 1024u + (m / 8u) * 64u + (c / 4u) * 32u + (m % 8u) * 4u +
                       (c % 4u)];
        ptx::tmem_st_32x32b_x8(tmem + ((q * 32u) << 16) + a_col + static_cast<uint32_t>(s) * 8u, w);
    }
    ptx::tmem_wait_st();
}

// Patch byte offsets of the 8 tile origins of each 8-tile group a gather warp owns
// (ELEM: patch element bytes, 4 = fp32 storage, 2 = binary16 inter-step storage).
template <int TYB, int GPW, int ELEM = 4>
__device__ __forceinline__ void tile_offsets(int gw, int patch_w, int32_t (&toff)[GPW][8]) {
#pragma unroll
    for (int gi = 0; gi < GPW; ++gi)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            int tx, ty;
            tile_of_column<TYB>((gw + kGatherWarps * gi) * 8 + t, tx, ty);
            toff[gi][t] = (ty * kTileH * patch_w + tx * kTileW) * ELEM;
        }
}

// One batch of B'': B''[q, tile] = patch[tile_origin + koff[q]] as f16 (RNE), written
// into the UMMA MN-major operand (8 tiles per 16-byte core-matrix row). Sweeps are
// processed UNR at a time: all their shared loads are issued before the first
// conversion, so the loop is not bound by one LDS round trip per sweep.
// LO: the sweep writes the low term of the split operand, f16(v - f16(v)) (exact
// residual in f32; B_hi + B_lo carries ~22 significant bits of v).
// HIN: the patch holds binary16 storage (the previous step's outputs already rounded
// to binary16 RNE by its epilogue, i.e. exactly the value the f32 path's conversion
// here would produce): the gather copies the bits.
template <int GPW, int UNR, bool LO = false, bool HIN = false>
__device__ __forceinline__ void gather_sweeps(uint32_t pbase, uint32_t bbase, const int32_t* sGsrc,
                                              const int32_t* sGdst, int j0, int gw, uint32_t gstride,
                                              uint32_t lane, const int32_t (&toff)[GPW][8]) {
    uint32_t src[UNR], dst[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {  // packed table: one load per lane and sweep
        const uint32_t e = static_cast<uint32_t>(sGsrc[(j0 + u) * 32 + lane]);
        src[u] = pbase + ((e & 0xffffu) << 1);
        dst[u] = bbase + ((e >> 16) << 4);
    }
    (void)sGdst;
    if constexpr (HIN) {
        static_assert(!LO, "split operands need fp32 storage");
        uint32_t hv[UNR][GPW][8];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int gi = 0; gi < GPW; ++gi)
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(hv[u][gi][t]) : "r"(src[u] + toff[gi][t]));
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int gi = 0; gi < GPW; ++gi) {
                uint32_t h[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) h[i] = __byte_perm(hv[u][gi][2 * i], hv[u][gi][2 * i + 1], 0x5410);
                const uint32_t d = dst[u] + static_cast<uint32_t>(gw + kGatherWarps * gi) * gstride;
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(d), "r"(h[0]), "r"(h[1]), "r"(h[2]),
                             "r"(h[3])
                             : "memory");
            }
        return;
    }
    float v[UNR][GPW][8];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int gi = 0; gi < GPW; ++gi)
#pragma unroll
            for (int t = 0; t < 8; ++t)
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[u][gi][t]) : "r"(src[u] + toff[gi][t]));
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int gi = 0; gi < GPW; ++gi) {
            uint32_t h[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float a = v[u][gi][2 * i], b = v[u][gi][2 * i + 1];
                if constexpr (LO) {
                    a -= __half2float(__float2half_rn(a));
                    b -= __half2float(__float2half_rn(b));
                }
                const __half2 hv = __floats2half2_rn(a, b);
                h[i] = *reinterpret_cast<const uint32_t*>(&hv);
            }
            const uint32_t d = dst[u] + static_cast<uint32_t>(gw + kGatherWarps * gi) * gstride;
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(d), "r"(h[0]), "r"(h[1]), "r"(h[2]),
                         "r"(h[3])
                         : "memory");
        }
}

template <int GPW, bool LO, bool HIN = false>
__device__ __forceinline__ void gather_range(uint32_t pbase, uint32_t bbase, const int32_t* sGsrc,
                                             const int32_t* sGdst, int j, int j_end, int gw, uint32_t gstride,
                                             uint32_t lane, const int32_t (&toff)[GPW][8]) {
    constexpr int UNR = GPW >= 2 ? 2 : 3;  // 24-32 loads in flight per lane
#pragma unroll 1
    for (; j + UNR <= j_end; j += UNR)
        gather_sweeps<GPW, UNR, LO, HIN>(pbase, bbase, sGsrc, sGdst, j, gw, gstride, lane, toff);
#pragma unroll 1
    for (; j < j_end; ++j) gather_sweeps<GPW, 1, LO, HIN>(pbase, bbase, sGsrc, sGdst, j, gw, gstride, lane, toff);
}

// Sweeps [0, lo0) write B'' (or B_hi), sweeps [lo0, nsweeps) B_lo (SST_PREC_F16X2).
template <int GPW, bool HIN = false>
__device__ __forceinline__ void gather_batch(uint32_t pbase, uint32_t bbase, const int32_t* sGsrc,
                                             const int32_t* sGdst, int nsweeps, int gw,
                                             uint32_t gstride, uint32_t lane,
                                             const int32_t (&toff)[GPW][8], int lo0) {
    if constexpr (HIN) {  // binary16 storage: f16 operands only (no split)
        gather_range<GPW, false, true>(pbase, bbase, sGsrc, sGdst, 0, nsweeps, gw, gstride, lane, toff);
        return;
    }
    const int hi_end = min(nsweeps, lo0);
    gather_range<GPW, false>(pbase, bbase, sGsrc, sGdst, 0, hi_end, gw, gstride, lane, toff);
    if (hi_end < nsweeps)
        gather_range<GPW, true>(pbase, bbase, sGsrc, sGdst, hi_end, nsweeps, gw, gstride, lane, toff);
}

template <int CW>
__device__ __forceinline__ void tmem_load_box(uint32_t taddr, uint32_t (&v)[CW]) {
    if constexpr (CW == 16) {
        ptx::tmem_ld_32x32b_x16(taddr, v);
    } else if constexpr (CW == 8) {
        ptx::tmem_ld_32x32b_x8(taddr, v);
    } else {
        ptx::tmem_ld_32x32b_x4(taddr, v);
    }
    ptx::tmem_wait_ld();
}

// The whole accumulator of a batch (all NBOX output boxes) -> registers, then the
// TMEM slot is handed back before any store work starts.
template <int TYB>
__device__ __forceinline__ void tmem_load_batch(uint32_t taddr, uint32_t (&v)[kTXB / 2][2 * TYB]) {
#pragma unroll
    for (int c = 0; c < kTXB / 2; ++c) {
        if constexpr (TYB == 8) {
            ptx::tmem_ld_32x32b_x16(taddr + c * 16, v[c]);
        } else if constexpr (TYB == 4) {
            ptx::tmem_ld_32x32b_x8(taddr + c * 8, v[c]);
        } else {
            ptx::tmem_ld_32x32b_x4(taddr + c * 4, v[c]);
        }
    }
    ptx::tmem_wait_ld();
}

// Stage one batch of outputs (NBOX boxes of 32 x 8*TYB cells; this thread's values
// v) into a 128B-swizzled smem buffer and TMA-store it: one barrier pair per batch.
// TMA clips the innermost dimension at 16-byte granularity, so the store map ends at
// ox4 = ox & ~3 and the <= 3 interior columns [ox4, ox) are written with plain stores.
// Called by all 128 epilogue threads; `nb` (batch count) cycles NS buffers.
// Right-edge columns [ox4, ox) (<= 3) of a batch: plain stores (TMA clips stores
// in 16-byte units). A thread owns x = X0 + 32c + 16 par + dxl, so at most one
// (c, par) of the batch falls in [ox4, ox) for it; only that branch runs (TYB stores).
template <int DIMS, int TYB>
__device__ __forceinline__ void store_right_edge(const StepParams& p, float* dst,
                                                 const uint32_t (&v)[kTXB / 2][2 * TYB], int X0, int Y0,
                                                 int Z0, uint32_t q, uint32_t lane) {
    constexpr int NBOX = kTXB / 2;
    const int ox = p.gx - 2 * p.r, ox4 = ox & ~3;
    if (X0 + kTXB * kTileW <= ox4 || (dbg(p) & 8)) return;
    const int dxl = static_cast<int>(q) * 4 + static_cast<int>(lane / 8);
    const int y_lim = DIMS == 2 ? p.slow_hi : p.y_end;
    const int y0 = Y0 + static_cast<int>(lane % 8);
    float* rowp = dst + (DIMS == 3 ? static_cast<int64_t>(Z0 + p.r) * p.plane_pitch : 0) +
                  static_cast<int64_t>(y0 + p.r) * p.row_pitch + p.left_pad + p.r + X0 + dxl;
    const int64_t ystep = static_cast<int64_t>(kTileH) * p.row_pitch;
#pragma unroll
    for (int c = 0; c < NBOX; ++c)
#pragma unroll
        for (int par = 0; par < 2; ++par) {
            const int xo = c * kBoxW + par * kTileW;
            const int xr = X0 + xo + dxl;
            if (xr >= ox4 && xr < ox) {
#pragma unroll
                for (int ty = 0; ty < TYB; ++ty)
                    if (y0 + ty * kTileH < y_lim) rowp[xo + ty * ystep] = __uint_as_float(v[c][2 * ty + par]);
            }
        }
}

// Slab P2P halos, 2D: the <= 3 right-edge columns of the neighbours' halo rows
// (TMA stores clip them). Rare (right-edge batches of the boundary bands), so one
// warp copies them from the staged boxes after the staging barrier in a rolled loop
// (reading registers instead would unroll the whole edge case again per peer).
__device__ __forceinline__ void peer_right_edge(const StepParams& p, uint32_t stage, uint32_t s_stride, int X0,
                                                int Y0, int rows, float* up, float* down, uint32_t lane) {
    const int ox = p.gx - 2 * p.r, ox4 = ox & ~3;
    if (X0 + kTXB * kTileW <= ox4 || ox4 == ox) return;
    const int c = (ox4 - X0) / kBoxW;  // the box holding [ox4, ox4 + 4)
    const int w = ox - ox4;
    for (int e = static_cast<int>(lane); e < rows * w; e += 32) {
        const int yl = e / w, x = ox4 + e % w, y = Y0 + yl;
        const bool to_up = up != nullptr && y < p.r, to_down = down != nullptr && y >= p.peer_down0;
        if (!(to_up || to_down) || y >= p.slow_hi) continue;
        const int xl = x - X0 - c * kBoxW;
        float val;
        asm volatile("ld.shared.f32 %0, [%1];"
                     : "=f"(val)
                     : "r"(stage + static_cast<uint32_t>(c) * s_stride + static_cast<uint32_t>(yl) * 128u +
                           (static_cast<uint32_t>((xl / 4) ^ (yl % 8)) * 16u) + static_cast<uint32_t>(xl % 4) * 4u));
        const int64_t off = static_cast<int64_t>(y + p.r) * p.row_pitch + p.left_pad + p.r + x;
        if (to_up) up[off + p.peer_up_shift * p.row_pitch] = val;
        if (to_down) down[off + p.peer_down_shift * p.row_pitch] = val;
    }
}

// 1D fold: the last view row's store boxes also cover the r right-ring cells
// [n_int, n_int + r) of the 1D grid (TMA cannot clip inside a row of the view). They
// keep their input values: staged in place of the computed ones from the copy the
// plan saved before the run, so every step leaves the ring as it found it.
template <int TYB>
__device__ __forceinline__ void fold_keep_ring(const StepParams& p, uint32_t (&v)[kTXB / 2][2 * TYB], int X0,
                                               int Y0, uint32_t q, uint32_t lane) {
    const int yr = static_cast<int>(p.fold_nint / p.fold_w), xr = static_cast<int>(p.fold_nint % p.fold_w);
    if (yr < Y0 || yr >= Y0 + TYB * kTileH || xr + p.r <= X0 || xr >= X0 + kTXB * kTileW) return;
    const int dx = static_cast<int>(q) * 4 + static_cast<int>(lane / 8), dy = static_cast<int>(lane % 8);
#pragma unroll
    for (int c = 0; c < kTXB / 2; ++c)
#pragma unroll
        for (int i = 0; i < 2 * TYB; ++i) {
            const int x = X0 + c * kBoxW + (i & 1) * kTileW + dx, y = Y0 + (i / 2) * kTileH + dy;
            if (y == yr && x >= xr && x < xr + p.r && x < p.fold_w) v[c][i] = __float_as_uint(p.fold_ring[x - xr]);
        }
}

// Right-edge handling of store_batch:
//   kEdgePlain  the <= 3 columns [ox4, ox) as plain stores, before the staging
//               barriers (the 2D multi-step kernel's progress flags must cover them)
//   kEdgeRing   no plain stores: the store map runs to ox4 + 4 and the cells
//               [ox, ox4 + 4) of that last 16-byte chunk (boundary ring / row pad,
//               constant in time and equal in both buffers) are staged with their
//               current values, which the producer loaded (one small TMA box per
//               input plane) into `ring` (TYB*8 rows x 4 floats). Scattered 4-byte
//               stores on every plane of the right-edge CTAs cost the 3D kernel ~5 %
//               (and leave partially written 32-byte sectors behind).
enum EdgeMode { kEdgePlain = 0, kEdgeRing = 1 };

template <int DIMS, int TYB, int NS, int EDGE = kEdgePlain, bool PEER = true>
__device__ __forceinline__ void store_batch(const StepParams& p, const CUtensorMap* tmap_out, float* dst,
                                            uint32_t (&v)[kTXB / 2][2 * TYB], uint8_t* sS,
                                            uint32_t s_stride, int nb, int X0, int Y0, int Z0,
                                            uint32_t q, uint32_t lane, int etid, const float* ring = nullptr,
                                            const CUtensorMap* peer_up = nullptr,
                                            const CUtensorMap* peer_down = nullptr, float* peer_up_buf = nullptr,
                                            float* peer_down_buf = nullptr) {
    using namespace ptx;
    constexpr int CW = 2 * TYB, NBOX = kTXB / 2;
    const uint32_t dy = lane % 8, w4 = (lane / 8) * 4;
    const int ox = p.gx - 2 * p.r, ox4 = ox & ~3;
    // last column the store map covers (exclusive)
    const int oxs = (EDGE == kEdgeRing && ox4 != ox) ? ox4 + 4 : ox4;
    if constexpr (EDGE == kEdgePlain) {
        store_right_edge<DIMS, TYB>(p, dst, v, X0, Y0, Z0, q, lane);
    } else {
        if (ring != nullptr && X0 + kTXB * kTileW > ox) {
            const int dxl = static_cast<int>(q) * 4 + static_cast<int>(lane / 8);
#pragma unroll
            for (int c = 0; c < NBOX; ++c)
#pragma unroll
                for (int par = 0; par < 2; ++par) {
                    const int xr = X0 + c * kBoxW + par * kTileW + dxl;
                    if (xr >= ox && xr < oxs) {
#pragma unroll
                        for (int ty = 0; ty < TYB; ++ty)
                            v[c][2 * ty + par] =
                                __float_as_uint(ring[(ty * kTileH + static_cast<int>(dy)) * 4 + (xr - ox4)]);
                    }
                }
        }
    }
    const uint32_t buf = static_cast<uint32_t>(nb % NS) * NBOX * s_stride;
    const uint32_t stage = smem_u32(sS) + buf;
    if (etid == 0) bulk_wait_read<NS - 1>();  // this buffer's previous stores have read it
    named_bar_sync(kEpiBarrier, kEpiWarps * 32);
    if (!(dbg(p) & 128)) {  // (ablation 128: TMA stores without staging)
#pragma unroll
    for (int c = 0; c < NBOX; ++c)
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            // local output (x, y) of D row m = 32q + lane in tile (2c + (i&1), i/2); the
            // 16-byte chunk index is XOR-swizzled with (row % 8) as TMA SWIZZLE_128B expects
            const uint32_t y = static_cast<uint32_t>(i / 2) * kTileH + dy;
            const uint32_t chunk = (static_cast<uint32_t>(i & 1) * 4u + q) ^ dy;
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(stage + c * s_stride + y * 128u + chunk * 16u + w4),
                         "r"(v[c][i])
                         : "memory");
        }
    }
    // The named barrier drains every epilogue thread's staging stores (bar.sync has
    // CTA memory-ordering semantics); the issuing thread then orders them before its
    // async-proxy (TMA) reads with one proxy fence. A per-thread fence right after the
    // stores instead costs each thread a MEMBAR over its 32-64 stores in flight.
    named_bar_sync(kEpiBarrier, kEpiWarps * 32);
    if constexpr (DIMS == 2 && PEER)
        if (p.peer_mask != 0 && etid >= 32 && etid < 64 && (Y0 < p.r || Y0 + TYB * kTileH > p.peer_down0))
            peer_right_edge(p, stage, s_stride, X0, Y0, TYB * kTileH, peer_up_buf, peer_down_buf, lane);
    if (etid == 0 && !(dbg(p) & 64)) {  // (ablation 64: staging only, no TMA stores)
        fence_proxy_async_smem();
#pragma unroll
        for (int c = 0; c < NBOX; ++c) {
            const int bx0 = X0 + c * kBoxW;
            if (bx0 >= oxs) break;  // fully clipped
            if (DIMS == 2)
                tma_store_2d(tmap_out, sS + buf + c * s_stride, bx0, Y0 - p.slow_lo);  // map starts at the window
            else
                tma_store_3d(tmap_out, sS + buf + c * s_stride, bx0, Y0, Z0);
        }
        // slab decomposition with peer-to-peer halos: boundary slices also go straight
        // into the neighbours' halo slices (NVLink stores of the same staged boxes;
        // the peer maps span only the r halo slices, TMA clips everything else)
        const int slice0 = DIMS == 2 ? Y0 : Z0, nslice = DIMS == 2 ? TYB * kTileH : 1;
        if (PEER && peer_up != nullptr && slice0 < p.r) {
#pragma unroll 1
            for (int c = 0; c < NBOX; ++c) {
                const int bx0 = X0 + c * kBoxW;
                if (bx0 >= oxs) break;
                if (DIMS == 2)
                    tma_store_2d(peer_up, sS + buf + c * s_stride, bx0, Y0);
                else
                    tma_store_3d(peer_up, sS + buf + c * s_stride, bx0, Y0, Z0);
            }
        }
        if (PEER && peer_down != nullptr && slice0 + nslice > p.peer_down0) {
#pragma unroll 1
            for (int c = 0; c < NBOX; ++c) {
                const int bx0 = X0 + c * kBoxW;
                if (bx0 >= oxs) break;
                if (DIMS == 2)
                    tma_store_2d(peer_down, sS + buf + c * s_stride, bx0, Y0 - p.peer_down_c0);
                else
                    tma_store_3d(peer_down, sS + buf + c * s_stride, bx0, Y0, Z0 - p.peer_down_c0);
            }
        }
        bulk_commit();
    }
}

// ---------------------------------------------------------------------------
// binary16 inter-step storage (SST_PREC_F16, steps 1 .. T-1 of a run): the epilogue
// rounds the f32 accumulator to binary16 RNE — the value every consumer (the next
// step's gather) would compute from the f32 store — and stores 2 B per update.
// A batch (128 x 8*TYB outputs) stages as two 64-half (128 B) SWIZZLE_128B boxes.
// TMA clips stores in 16-byte units (8 halves): the store map ends at ox8 = ox & ~7
// and the <= 7 columns [ox8, ox) are plain 2-byte stores.
template <int DIMS, int TYB>
__device__ __forceinline__ void store_right_edge_h(const StepParams& p, __half* dst,
                                                   const uint32_t (&v)[kTXB / 2][2 * TYB], int X0, int Y0,
                                                   int Z0, uint32_t q, uint32_t lane) {
    constexpr int NBOX = kTXB / 2;
    const int ox = p.gx - 2 * p.r, ox8 = ox & ~7;
    if (X0 + kTXB * kTileW <= ox8 || (dbg(p) & 8)) return;
    const int dxl = static_cast<int>(q) * 4 + static_cast<int>(lane / 8);
    const int y_lim = DIMS == 2 ? p.slow_hi : p.y_end;
    const int y0 = Y0 + static_cast<int>(lane % 8);
    __half* rowp = dst + (DIMS == 3 ? static_cast<int64_t>(Z0 + p.r) * p.plane_pitch : 0) +
                   static_cast<int64_t>(y0 + p.r) * p.row_pitch + p.left_pad + p.r + X0 + dxl;
    const int64_t ystep = static_cast<int64_t>(kTileH) * p.row_pitch;
#pragma unroll
    for (int c = 0; c < NBOX; ++c)
#pragma unroll
        for (int par = 0; par < 2; ++par) {
            const int xo = c * kBoxW + par * kTileW;
            const int xr = X0 + xo + dxl;
            if (xr >= ox8 && xr < ox) {
#pragma unroll
                for (int ty = 0; ty < TYB; ++ty)
                    if (y0 + ty * kTileH < y_lim)
                        rowp[xo + ty * ystep] = __float2half_rn(__uint_as_float(v[c][2 * ty + par]));
            }
        }
}

// EDGE = kEdgeRing (3D stream kernel): as in store_batch, no plain stores; the store
// map runs to ox8 + 8 and the cells [ox, ox8 + 8) of that last 16-byte chunk are
// staged with the output storage's own (constant) binary16 values from `ring`
// (TYB*8 rows x 8 halves).
// Slab P2P halos, 2D binary16: the <= 7 right-edge columns [ox8, ox) of the
// neighbours' halo rows (TMA clips them), copied from the staged binary16 boxes.
__device__ __forceinline__ void peer_right_edge_h(const StepParams& p, uint32_t stage, uint32_t s_stride, int X0,
                                                  int Y0, int rows, __half* up, __half* down, uint32_t lane) {
    const int ox = p.gx - 2 * p.r, ox8 = ox & ~7;
    if (X0 + kTXB * kTileW <= ox8 || ox8 == ox) return;
    const int w = ox - ox8;
    for (int e = static_cast<int>(lane); e < rows * w; e += 32) {
        const int yl = e / w, x = ox8 + e % w, y = Y0 + yl;
        const bool to_up = up != nullptr && y < p.r, to_down = down != nullptr && y >= p.peer_down0;
        if (!(to_up || to_down) || y >= p.slow_hi) continue;
        const int xl = x - X0;  // box xl / 64, 16-byte chunk (xl % 64) / 8 swizzled with the row
        unsigned short bits;
        asm volatile("ld.shared.u16 %0, [%1];"
                     : "=h"(bits)
                     : "r"(stage + static_cast<uint32_t>(xl / 64) * s_stride + static_cast<uint32_t>(yl) * 128u +
                           (static_cast<uint32_t>(((xl % 64) / 8) ^ (yl % 8)) * 16u) +
                           static_cast<uint32_t>(xl % 8) * 2u));
        const __half val = *reinterpret_cast<const __half*>(&bits);
        const int64_t off = static_cast<int64_t>(y + p.r) * p.row_pitch + p.left_pad + p.r + x;
        if (to_up) up[off + p.peer_up_shift * p.row_pitch] = val;
        if (to_down) down[off + p.peer_down_shift * p.row_pitch] = val;
    }
}

// PEER (slabs with P2P halos; only the instantiations launched with peers carry the
// code): peer_up / peer_down are the neighbours' binary16 halo slices, stored from the
// same staged boxes as in store_batch; 2D also copies the <= 7 right-edge columns
// into peer_up_buf / peer_down_buf.
template <int DIMS, int TYB, int NS, int EDGE = kEdgePlain, bool PEER = false>
__device__ __forceinline__ void store_batch_h(const StepParams& p, const CUtensorMap* tmap_out, __half* dst,
                                              uint32_t (&v)[kTXB / 2][2 * TYB], uint8_t* sS,
                                              uint32_t s_stride, int nb, int X0, int Y0, int Z0, uint32_t q,
                                              uint32_t lane, int etid, const __half* ring = nullptr,
                                              const CUtensorMap* peer_up = nullptr,
                                              const CUtensorMap* peer_down = nullptr,
                                              __half* peer_up_buf = nullptr, __half* peer_down_buf = nullptr) {
    using namespace ptx;
    constexpr int CW = 2 * TYB, NBOX = kTXB / 2;
    constexpr int HBOX = 64;  // halves per 128-byte box row
    const uint32_t dy = lane % 8;
    const uint32_t inchunk = ((q & 1u) * 4u + lane / 8u) * 2u;  // byte of dx % 8 inside its 16 B chunk
    const int ox = p.gx - 2 * p.r, ox8 = ox & ~7;
    const int oxs = (EDGE == kEdgeRing && ox8 != ox) ? ox8 + 8 : ox8;  // store map end (exclusive)
    if constexpr (EDGE == kEdgePlain) {
        store_right_edge_h<DIMS, TYB>(p, dst, v, X0, Y0, Z0, q, lane);
    } else if (ring != nullptr && X0 + kTXB * kTileW > ox) {
        const int dxl = static_cast<int>(q) * 4 + static_cast<int>(lane / 8);
#pragma unroll
        for (int c = 0; c < NBOX; ++c)
#pragma unroll
            for (int par = 0; par < 2; ++par) {
                const int xr = X0 + c * kBoxW + par * kTileW + dxl;
                if (xr >= ox && xr < oxs) {
#pragma unroll
                    for (int ty = 0; ty < TYB; ++ty)  // exact: binary16 -> f32 -> binary16
                        v[c][2 * ty + par] =
                            __float_as_uint(__half2float(ring[(ty * kTileH + static_cast<int>(dy)) * 8 + (xr - ox8)]));
                }
            }
    }
    // a binary16 batch fills half an fp32 staging slot: 2 NS buffers, so the TMA
    // stores of batch n read one while batch n + 1 stages into the next
    constexpr int NSH = 2 * NS;
    const uint32_t buf = static_cast<uint32_t>(nb % NSH) * (NBOX / 2) * s_stride;
    const uint32_t stage = smem_u32(sS) + buf;
    if (etid == 0) bulk_wait_read<NSH - 1>();
    named_bar_sync(kEpiBarrier, kEpiWarps * 32);
#pragma unroll
    for (int c = 0; c < NBOX; ++c)
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            // x in the batch = 32c + 16 (i & 1) + dx, dx = 4q + lane / 8; box c / 2 holds
            // x in [64 (c / 2), 64 (c / 2) + 64): 16-byte chunk 4 (c & 1) + 2 (i & 1) + q / 2
            const uint32_t y = static_cast<uint32_t>(i / 2) * kTileH + dy;
            const uint32_t chunk = (static_cast<uint32_t>(c & 1) * 4u + static_cast<uint32_t>(i & 1) * 2u + q / 2u) ^ dy;
            const __half h = __float2half_rn(__uint_as_float(v[c][i]));
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(stage + static_cast<uint32_t>(c / 2) * s_stride + y * 128u +
                                                         chunk * 16u + inchunk),
                         "h"(*reinterpret_cast<const unsigned short*>(&h))
                         : "memory");
        }
    named_bar_sync(kEpiBarrier, kEpiWarps * 32);
    if constexpr (DIMS == 2 && PEER)
        if (p.peer_mask != 0 && etid >= 32 && etid < 64 && (Y0 < p.r || Y0 + TYB * kTileH > p.peer_down0))
            peer_right_edge_h(p, stage, s_stride, X0, Y0, TYB * kTileH, peer_up_buf, peer_down_buf, lane);
    if (etid == 0 && !(dbg(p) & 64)) {
        fence_proxy_async_smem();
#pragma unroll
        for (int cb = 0; cb < NBOX / 2; ++cb) {
            const int bx0 = X0 + cb * HBOX;
            if (bx0 >= oxs) break;  // fully clipped
            if (DIMS == 2)
                tma_store_2d(tmap_out, sS + buf + cb * s_stride, bx0, Y0 - p.slow_lo);
            else
                tma_store_3d(tmap_out, sS + buf + cb * s_stride, bx0, Y0, Z0);
        }
        if constexpr (PEER && DIMS == 2) {  // (the lower neighbour's map starts in its guard rows)
            if (peer_up != nullptr && Y0 < p.r) {
#pragma unroll 1
                for (int cb = 0; cb < NBOX / 2; ++cb) {
                    const int bx0 = X0 + cb * HBOX;
                    if (bx0 >= oxs) break;
                    tma_store_2d(peer_up, sS + buf + cb * s_stride, bx0, Y0);
                }
            }
            if (peer_down != nullptr && Y0 + TYB * kTileH > p.peer_down0) {
#pragma unroll 1
                for (int cb = 0; cb < NBOX / 2; ++cb) {
                    const int bx0 = X0 + cb * HBOX;
                    if (bx0 >= oxs) break;
                    tma_store_2d(peer_down, sS + buf + cb * s_stride, bx0, Y0 - p.peer_down_c0);
                }
            }
        }
        if constexpr (PEER && DIMS == 3) {
            if (peer_up != nullptr && Z0 < p.r) {
#pragma unroll 1
                for (int cb = 0; cb < NBOX / 2; ++cb) {
                    const int bx0 = X0 + cb * HBOX;
                    if (bx0 >= oxs) break;
                    tma_store_3d(peer_up, sS + buf + cb * s_stride, bx0, Y0, Z0);
                }
            }
            if (peer_down != nullptr && Z0 + 1 > p.peer_down0) {
#pragma unroll 1
                for (int cb = 0; cb < NBOX / 2; ++cb) {
                    const int bx0 = X0 + cb * HBOX;
                    if (bx0 >= oxs) break;
                    tma_store_3d(peer_down, sS + buf + cb * s_stride, bx0, Y0, Z0 - p.peer_down_c0);
                }
            }
        }
        bulk_commit();
    }
}

}  // namespace sst
