// stencil_kernel.cuh — one time step of a compiled 2:4-sparse stencil operator
// on sm_100a (2D, and the monolithic 3D variant). The reference's hot loop
// (proj/core/src/emulator.cpp:134-193, tiled_sparse_matmul with the b_entry
// provider, scattered through output_position, layout.cpp:190-209) becomes,
// per CTA batch of 8 x TYB output tiles (tile = 16 x 8 outputs, D row m = dx*8 + dy):
//
//   warp 0      TMA producer: grid patch (+halo, zero-filled outside) -> smem,
//               NP-deep ring so several patches are in flight per SM
//   warps 2-5   gather: B''[q, tile] = patch[tile_origin + koff[q]] (the
//               memory map of layout.cpp:162-188), fp32 -> fp16 (RNE, the
//               reference round16 rounding), into the UMMA MN-major operand
//   warp 1      MMA issuer: tcgen05.mma.sp.cta_group::1.kind::f16, compressed
//               A'' from TMEM (the default AT variants; K-major smem in the
//               AT = false ones), metadata from TMEM, D in TMEM
//   warps 6-9   epilogue: tcgen05.ld -> 128B-swizzled smem staging -> TMA
//               bulk store through a tensor map clipped to the interior
//
// mbarrier handshakes between roles, double-buffered B operand and TMEM
// accumulator, persistent CTAs (one per SM) striding over batches.
#pragma once

#include "stencil_common.cuh"

namespace sst {

struct SmemLayout {
    uint32_t a, b, b_stride, p, p_stride, s, s_stride, gsrc, gdst, bars, tmem_slot, total;
    uint32_t pbar;  // prologue mbarrier (constant staging by bulk copy)
    uint32_t ring;  // 3D stream kernel: right-edge ring-value cache (ring_slots() x TYB*8 x 4 floats)
};

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// Shared-memory carve-up; np / nbb / ns = patch, B'' and output-staging ring
// depths, nbars mbarriers.
template <int TYB>
__host__ __device__ inline SmemLayout smem_layout_generic(int nks, int k_pad, int patch_w, int patch_h,
                                                          int planes, int np, int nbb, int nbars,
                                                          int ns = kStageBufs, bool a_in_tmem = false,
                                                          int elem = 4) {
    constexpr int N = kTXB * TYB;
    SmemLayout L{};
    uint32_t o = 0;
    L.a = o;
    o += a_in_tmem ? 0u : static_cast<uint32_t>(nks) * 4096u;
    L.b_stride = align_up(static_cast<uint32_t>(k_pad) * N * 2u, 1024);
    L.b = o = align_up(o, 1024);
    o += nbb * L.b_stride;
    L.s_stride = align_up(static_cast<uint32_t>(kBoxW * kTileH * TYB) * 4u, 1024);
    L.s = o = align_up(o, 1024);
    o += ns * (kTXB / 2) * L.s_stride;
    L.p_stride = align_up(static_cast<uint32_t>(patch_w * patch_h * planes * elem), 128);
    L.p = o = align_up(o, 128);
    o += np * L.p_stride;
    // the prologue stages the A'' image / metadata words in [L.b, L.gsrc) before
    // moving them into TMEM: deep A'' (fused 3D, 40 K steps) needs more than the rings
    const uint32_t scratch = prologue_scratch_bytes(nks, a_in_tmem);
    if (o < L.b + scratch) o = L.b + scratch;
    L.gsrc = o = align_up(o, 16);
    o += static_cast<uint32_t>(k_pad) * 4u;
    L.gdst = o;
    o += static_cast<uint32_t>(k_pad) * 4u;
    L.bars = o = align_up(o, 8);
    o += nbars * 8;
    L.pbar = o;
    o += 8;
    L.tmem_slot = o;
    o += 16;
    L.total = align_up(o, 128);
    return L;
}

// Dynamic batch scheduling of single-step launches: the producer draws batch
// indices from a global counter and hands them to the other roles through a ring
// of kBidSlots (index, mbarrier) slots (reuse is safe: the producer cannot run
// kBidSlots iterations ahead of the epilogue through the patch / B'' / accumulator
// rings, 3 + 2 + 2 deep).
constexpr int kBidSlots = 16;
constexpr int kDrawAhead = 2;  // dynamic scheduling: counter draws in flight per CTA
constexpr int kDrawGroup = 2;  // consecutive batches (items) per counter draw
// dynamic multi-step mode: items committed but not yet published (publication every
// kPubEvery items, lagging kPubLag store groups)
constexpr int kPubEvery = 8, kPubLag = 2, kPubRing = 16;
static_assert(kPubRing >= kPubEvery + kPubLag + 1, "publication ring");

template <int TYB, int NP, bool AT, int NS = kStageBufs, int NBB = 2, int NACC = 2>
__host__ __device__ inline SmemLayout smem_layout(int nks, int k_pad, int patch_w, int patch_h,
                                                  int planes, int elem = 4) {
    static_assert(kBidSlots > NP + NBB + NACC, "batch-index ring vs pipeline depth");
    SmemLayout L = smem_layout_generic<TYB>(nks, k_pad, patch_w, patch_h, planes, NP, NBB,
                                            2 * NP + 2 * NBB + 2 * NACC + kBidSlots, NS, AT, elem);
    L.ring = align_up(L.total, 16);  // the batch-index ring (int32 x kBidSlots), then the
                                     // dynamic multi-step mode's unpublished items (kPubRing)
    L.total = align_up(L.ring + (kBidSlots + kPubRing) * 4, 128);
    return L;
}

// Multi-step dataflow. Every CTA walks the same number of iterations per step
// (nper = ceil(nbatch / grid); CTAs with one batch fewer run a no-op iteration) and
// publishes a progress counter: flags[cta] = flag_base + iterations whose stores
// are complete. Batch b of step t >= 1 reads outputs of step t - 1 of batches up
// to b + nbx + 1 (its 3 x 3 neighbourhood), each processed at step-(t-1) iteration
// <= (b + nbx + 1) / grid by its owner; so it may load once EVERY counter reached
// flag_base + (t - 1) nper + min(nper, (b + nbx + 1) / grid + 1). The producer warp
// keeps the minimum over all counters cached and refreshes it (one warp-wide
// sweep) only when a batch needs more: in steady state about once per step.
__device__ __forceinline__ uint32_t refresh_min(const StepParams& p, uint32_t need, uint32_t lane,
                                                uint32_t& polls) {
    for (;;) {
        int32_t worst = 0x7fffffff;
        for (int o = static_cast<int>(lane); o < static_cast<int>(gridDim.x); o += 32)
            worst = min(worst, static_cast<int32_t>(ptx::ld_relaxed_gpu(p.flags + o) - need));
        for (int sh = 16; sh > 0; sh >>= 1) worst = min(worst, __shfl_xor_sync(0xffffffffu, worst, sh));
        if (worst >= 0) {
            if (lane == 1) ptx::fence_acq_rel_gpu();  // acquire; lane 0 (TMA issuer) never fences
            __syncwarp();
            return need + static_cast<uint32_t>(worst);
        }
        ++polls;
        ptx::nanosleep(128);
    }
}

// AT: compressed A'' in TMEM (tcgen05.mma.sp [a-tmem] form) instead of smem.
//
// MODE (compile-time, so each launch runs only its own code path: the kernel's
// instruction footprint matters for L2-cold launches):
//   0 static batch striding, one time step;
//   1 dynamic batches (p.sched counter), one time step;
//   2 multi-step dataflow with static batch ownership: one launch runs p.nsteps steps
//     (persistent CTAs, 2D, full window), step t reads buffer (src + t) & 1; no grid
//     barrier between steps: each CTA publishes a progress counter flags[cta] and a
//     producer loads batch b of step t once every CTA has stored its step-(t-1)
//     batches up to b + nbx + 1 (refresh_min); that also orders the write-after-read
//     on the ping-pong buffer (a CTA publishes only after it loaded those patches);
//   3 dynamic batches with the slab P2P halo stores (the only 2D instantiation that
//     carries the peer code: it measurably slowed the store path of the others), also
//     the two-window launch of the NCCL slab mode (both boundary windows at once);
//   4 multi-step dataflow with DYNAMIC ownership: items g = t * nbatch + b are drawn
//     in order from p.sched; the producer loads item (t, b) once the 3 x 3 batch
//     neighbourhood has flags[n] >= flag_base + t (its step t-1 stored); the epilogue
//     publishes flags[b] = flag_base + t + 1 after the item's stores complete (every
//     kPubEvery items, and whenever it idled 2 us, so no circular wait). Items of
//     step t depend only on items drawn earlier, and a CTA holds only items it drew,
//     so the schedule needs no co-residency.
//   5 grouped: dynamic batches over p.group_n identical grids (sst_run_steps_batch), item
//     g = grid * nbatch + batch, the grid's maps and output buffer from p.group
enum StepMode { kModeStatic = 0, kModeDynamic = 1, kModeMulti = 2, kModePeer = 3, kModeMultiDyn = 4, kModeGroup = 5 };

// NS: output staging buffers (TMA stores of batch n read one while batch n + 1 stages
// into the next; 1 = the epilogue waits for each batch's stores to leave smem)
// CPS: CTAs per SM the variant is built for (2: small-smem variants whose two co-resident
// CTAs overlap one another's pipeline bubbles; registers capped accordingly)
// HIN / HOUT: the input / output grid is binary16 storage (SST_PREC_F16 runs keep
// steps 1 .. T-1 in binary16: bitwise the same result, half the bytes per update);
// the out map and p's pitches / left pad then describe the f16 buffer, the in map,
// gather tables and patch width the input's storage.
// NBB / NACC: B'' operand stages in smem / accumulator stages in TMEM.
template <int DIMS, int TYB, int NP, bool AT, int MODE = kModeStatic, int NS = kStageBufs, int CPS = 1,
          bool HIN = false, bool HOUT = false, int NBB = 2, int NACC = 2>
__global__ void __launch_bounds__(kThreads, CPS)
    stencil_step_kernel(const __grid_constant__ MapSet maps, const StepParams p) {
    constexpr int N = kTXB * TYB;
    constexpr int CW = 2 * TYB;          // MMA columns per output box
    constexpr int NBOX = kTXB / 2;       // output boxes per batch
    constexpr int NGROUP = N / 8;        // 8-tile B'' groups
    constexpr int GPW = NGROUP >= kGatherWarps ? NGROUP / kGatherWarps : 1;
    constexpr int PUB_LAG = 2;           // newest store groups not waited for when publishing
    static_assert(N % 16 == 0 && N <= 128, "UMMA N for M=128");
    static_assert(NGROUP % kGatherWarps == 0 || NGROUP < kGatherWarps, "group split");
    using namespace ptx;

    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int ELEM = HIN ? 2 : 4;  // patch element bytes
    const SmemLayout L =
        smem_layout<TYB, NP, AT, NS, NBB, NACC>(p.nks, p.k_pad, p.patch_w, p.patch_h, p.patch_planes, ELEM);
    uint8_t* sA = smem + L.a;
    uint8_t* sB = smem + L.b;  // 2 stages
    uint8_t* sS = smem + L.s;  // output staging
    uint8_t* sP = smem + L.p;  // NP stages
    int32_t* sGsrc = reinterpret_cast<int32_t*>(smem + L.gsrc);
    int32_t* sGdst = reinterpret_cast<int32_t*>(smem + L.gdst);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* patch_full = bars;
    uint64_t* patch_empty = bars + NP;
    uint64_t* b_full = bars + 2 * NP;
    uint64_t* b_empty = b_full + NBB;
    uint64_t* d_full = b_empty + NBB;
    uint64_t* d_empty = d_full + NACC;
    uint64_t* bid_full = d_empty + NACC;  // [kBidSlots]
    int32_t* sBid = reinterpret_cast<int32_t*>(smem + L.ring);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem_slot);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = lane_id();
    const unsigned long long t_start = p.trace ? global_ns() : 0ull;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NP; ++s) {
            mbar_init(&patch_full[s], 1);
            mbar_init(&patch_empty[s], kGatherWarps);
        }
        for (int s = 0; s < NBB; ++s) {
            mbar_init(&b_full[s], kGatherWarps);
            mbar_init(&b_empty[s], 1);
        }
        for (int s = 0; s < NACC; ++s) {
            mbar_init(&d_full[s], 1);
            mbar_init(&d_empty[s], kEpiWarps);
        }
        for (int s = 0; s < kBidSlots; ++s) mbar_init(&bid_full[s], 1);
        fence_mbar_init();
        for (int i = 0; i < 2; ++i) {
            tma_prefetch_desc(&maps.in[i]);
            tma_prefetch_desc(&maps.out[i]);
        }
    }
    if (warp == 1) tmem_alloc(tmem_slot, static_cast<uint32_t>(p.tmem_cols));
    uint64_t* pbar = reinterpret_cast<uint64_t*>(smem + L.pbar);
    if (threadIdx.x == 0) {
        mbar_init(pbar, 1);
        fence_mbar_init();
        stage_constants_issue<AT>(p, sA, sB, sGsrc, sGdst, pbar);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    mbar_wait(pbar, 0);  // constants in smem
    const uint32_t tmem = *tmem_slot;
    // TMEM: two accumulators, the metadata columns, then (AT) the A'' operand
    const TmemCols tc = tmem_budget(NACC * N, static_cast<uint32_t>(p.nks), AT);
    const uint32_t e_col = tc.e_col;
    if (warp >= kEpiWarp0) {
        store_metadata<AT>(p, sB, tmem, e_col, static_cast<uint32_t>(warp % 4), lane);
        if constexpr (AT) store_a_tmem(p, sB, tmem, tc.a_col, static_cast<uint32_t>(warp % 4), lane);
    }
    fence_proxy_async_smem();  // scratch (generic writes / reads) is reused by TMA below
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // everything above touches only the plan's constants: it overlaps the previous
    // launch's tail under PDL. The grid buffers are read / written only below.
    grid_dep_wait();
    grid_dep_launch();
    const unsigned long long t_main = p.trace ? global_ns() : 0ull;

    const int nbx = p.nbx, nby = p.nby;
    const int G = static_cast<int>(gridDim.x);
    // iteration j = (step t, k): batch blockIdx.x + k * G, the same batches every step;
    // k beyond this CTA's batches is a no-op iteration (uniform nper for the counters)
    const int nper = (p.nbatch + G - 1) / G;
    const int total = nper * p.nsteps;
    auto batch_of = [&](int j, int& t, int& b) {
        t = j / nper;
        b = static_cast<int>(blockIdx.x) + (j - t * nper) * G;
    };
    auto batch_coords = [&](int b, int& X0, int& Y0, int& Z0) {
        if constexpr (MODE == kModeDynamic)  // reverse traversal: start where the previous step ended
            if (p.reverse) b = p.nbatch - 1 - b;
        X0 = (b % nbx) * (kTXB * kTileW);
        Y0 = ((b / nbx) % nby) * (TYB * kTileH) + (DIMS == 2 ? p.slow_lo : 0);
        Z0 = b / (nbx * nby) + (DIMS == 3 ? p.slow_lo : 0);
        if constexpr (DIMS == 2 && MODE == kModePeer) {  // two-window launch: second window
            const int by = (b / nbx) % nby;
            if (by >= p.nby1) Y0 = (by - p.nby1) * (TYB * kTileH) + p.slow_lo2;
        }
    };
    constexpr bool multi = MODE == kModeMulti;
    constexpr bool mdyn = MODE == kModeMultiDyn;
    // launches with a scheduler counter draw batches (mdyn: items) dynamically
    constexpr bool grp = MODE == kModeGroup;
    constexpr bool dyn = MODE == kModeDynamic || MODE == kModePeer || mdyn || grp;
    const int nitems = mdyn ? p.nbatch * p.nsteps : grp ? p.nbatch * p.group_n : p.nbatch;
    int32_t* sPub = sBid + kBidSlots;  // mdyn: committed, unpublished items (epilogue etid 0)
    constexpr bool peer = MODE == kModePeer || DIMS == 3;  // (3D whole-window: one instantiation)
    auto next_bid = [&](int r) {  // consumers: batch index of real iteration r (-1: done)
        mbar_wait(&bid_full[r % kBidSlots], (r / kBidSlots) & 1);
        return sBid[r % kBidSlots];
    };

    if ((dbg(p) & 32) && warp < kEpiWarp0) {
        // store-only ablation: only the epilogue runs (writes zeros)
    } else if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        // (the whole warp walks the loop: lane 0 issues, all lanes refresh counters)
        const uint32_t pbytes = static_cast<uint32_t>(p.patch_w * p.patch_h * p.patch_planes * ELEM);
        uint32_t polls = 0, known = p.flag_base;  // min over all progress counters seen
        int r = 0;                                // real (non no-op) iterations
        if constexpr (dyn) {
            // a CTA's first batch is blockIdx.x, later ones G + counter draws. Draws
            // run kDrawAhead batches ahead in a FIFO of registers (two slots, the loop
            // unrolled over them): the atomic's round trip (~0.7 us under load) would
            // otherwise bound the producer to one batch per round trip (binary16
            // patches: loads-only ablation 3.3 TB/s). Consuming slots in draw order
            // keeps the counter exact: each consumed batch triggers one draw, so a
            // launch advances it by nitems + G * (kDrawAhead - 1), and the first
            // invalid slot a CTA meets is followed only by invalid ones. With groups of
            // kDrawGroup batches per draw the count is in groups: ceil(nitems / kDrawGroup).
            uint32_t q0 = blockIdx.x, q1 = 0;
            if (lane == 0) q1 = static_cast<uint32_t>(G) + atomicAdd(p.sched, 1u) - p.sched_base;
            // one draw covers kDrawGroup consecutive batches (fewer same-address atomics)
            auto item = [&](uint32_t& slot) -> bool {
                uint32_t dgrp = 0;  // draw group (kDrawGroup consecutive items)
                if (lane == 0) {
                    dgrp = slot;
                    if (dgrp * static_cast<uint32_t>(kDrawGroup) < static_cast<uint32_t>(nitems))
                        slot = static_cast<uint32_t>(G) + atomicAdd(p.sched, 1u) - p.sched_base;
                }
                for (int e = 0; e < kDrawGroup; ++e) {
                int g = -1;
                if (lane == 0) {
                    const uint32_t gi = dgrp * static_cast<uint32_t>(kDrawGroup) + static_cast<uint32_t>(e);
                    g = gi < static_cast<uint32_t>(nitems) ? static_cast<int>(gi) : -1;
                    sBid[r % kBidSlots] = g;
                    mbar_arrive(&bid_full[r % kBidSlots]);
                }
                g = __shfl_sync(0xffffffffu, g, 0);
                if (g < 0) return false;
                if constexpr (MODE == kModeGroup)  // reverse traversal of the whole group
                    if (p.reverse) g = nitems - 1 - g;
                constexpr bool group_mode = MODE == kModeGroup;
                const int t = mdyn ? g / p.nbatch : 0, gj = group_mode ? g / p.nbatch : 0;
                const int b = mdyn ? g - t * p.nbatch : group_mode ? g - gj * p.nbatch : g;
                int X0, Y0, Z0;
                batch_coords(b, X0, Y0, Z0);
                if constexpr (mdyn) {
                    if (t > 0) {  // lanes 0..8: the 3 x 3 neighbourhood has stored step t - 1
                        const int by = b / nbx, bx = b - by * nbx;
                        const int ny = by + static_cast<int>(lane) / 3 - 1, nx = bx + static_cast<int>(lane) % 3 - 1;
                        const bool mine = lane < 9 && ny >= 0 && ny < nby && nx >= 0 && nx < nbx;
                        const uint32_t need = p.flag_base + static_cast<uint32_t>(t);
                        for (;;) {  // acquire loads: no separate fence on the issue path
                            const bool ok = !mine ||
                                static_cast<int32_t>(ld_acquire_gpu(p.flags + ny * nbx + nx) - need) >= 0;
                            if (__all_sync(0xffffffffu, ok)) break;
                            ++polls;
                            nanosleep(64);
                        }
                        if (lane == 0) fence_proxy_async_global();  // acquired data -> TMA reads
                    }
                }
                if (lane == 0) {
                    const int s = r % NP;
                    mbar_wait(&patch_empty[s], ((r / NP) & 1) ^ 1);
                    mbar_arrive_expect_tx(&patch_full[s], pbytes);
                    void* dst = sP + s * L.p_stride;
                    // (kernel-parameter maps and global maps in separate instantiations: a pointer
                    // that may be either is generic, and TMA faults on a generic param address)
                    if constexpr (MODE == kModeGroup) {
                        tma_load_2d(dst, &p.group[gj].in, &patch_full[s], X0 + p.load_x0, Y0 + p.load_y0);
                    } else {
                        const CUtensorMap* tin = &maps.in[(p.src + t) & 1];
                        if (DIMS == 2)
                            tma_load_2d(dst, tin, &patch_full[s], X0 + p.load_x0, Y0 + p.load_y0);
                        else
                            tma_load_3d(dst, tin, &patch_full[s], X0 + p.load_x0, Y0, Z0);
                    }
                }
                __syncwarp();
                ++r;
                }
                return true;
            };
            while (item(q0) && item(q1)) {
            }
        }
        for (int j = 0; j < (dyn ? 0 : total); ++j) {
            int t, b, X0, Y0, Z0;
            batch_of(j, t, b);
            if (b >= p.nbatch) continue;
            batch_coords(b, X0, Y0, Z0);
            bool refreshed = false;
            if (t > 0) {
                const int kneed = min(nper, (min(b + nbx + 1, p.nbatch - 1)) / G + 1);
                const uint32_t need = p.flag_base + static_cast<uint32_t>((t - 1) * nper + kneed);
                if (static_cast<int32_t>(known - need) < 0) {
                    known = refresh_min(p, need, lane, polls);
                    refreshed = true;
                }
            }
            if (lane == 0) {
                const int s = r % NP;
                const uint32_t ph = (r / NP) & 1;
                mbar_wait(&patch_empty[s], ph ^ 1);
                if (refreshed) fence_proxy_async_global();  // acquired data -> TMA reads
                mbar_arrive_expect_tx(&patch_full[s], pbytes);
                // storage column X0 is 16-byte aligned (TMA requirement); the
                // window origin sits left_pad cells into the patch (gsrc has it)
                void* dst = sP + s * L.p_stride;
                const CUtensorMap* tin = &maps.in[(p.src + t) & 1];
                if (DIMS == 2)
                    tma_load_2d(dst, tin, &patch_full[s], X0 + p.load_x0, Y0 + p.load_y0);
                else
                    tma_load_3d(dst, tin, &patch_full[s], X0 + p.load_x0, Y0, Z0);
            }
            __syncwarp();
            ++r;
        }
        if (lane == 0) tmem_slot[1] = polls;  // profiling (trace): counter sweeps that found a CTA behind
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        const uint32_t idesc = make_idesc_f16(128, N, true, 0, 1);
        const uint32_t b_sbo = static_cast<uint32_t>(p.k_pad) * 16u;
        const uint32_t a0 = smem_u32(sA);
        int r = 0;
        for (int j = 0; dyn || j < total; ++j, ++r) {
            int t, b;
            if constexpr (dyn) {
                if (next_bid(r) < 0) break;
            } else {
                batch_of(j, t, b);
                if (b >= p.nbatch) {
                    --r;
                    continue;
                }
            }
            const int s = r % NBB, sa = r % NACC;
            mbar_wait(&b_full[s], (r / NBB) & 1);
            mbar_wait(&d_empty[sa], ((r / NACC) & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t b0 = smem_u32(sB + s * L.b_stride);
                const int nks = (dbg(p) & 4) ? 1 : p.nks;
                for (int ks = 0; ks < nks; ++ks) {
                    const uint64_t bd = make_smem_desc(b0 + ks * 512u, 128, b_sbo);
                    const uint32_t ea = tmem + e_col + static_cast<uint32_t>(ks);
                    if constexpr (AT) {
                        mma_sp_f16_ts(tmem + static_cast<uint32_t>(sa * N), tmem + tc.a_col + ks * 8u, bd,
                                      ea & ~1u, idesc | (ea & 1u), ks > 0 ? 1u : 0u);
                    } else {
                        const uint64_t ad = make_smem_desc(a0 + ks * 4096u, 128, 256);
                        mma_sp_f16(tmem + static_cast<uint32_t>(sa * N), ad, bd, ea & ~1u,
                                   idesc | (ea & 1u), ks > 0 ? 1u : 0u);
                    }
                }
                mma_commit(&b_empty[s]);
                mma_commit(&d_full[sa]);
            }
            __syncwarp();
        }
    } else if (warp < kGatherWarp0 + kGatherWarps) {
        // ------------------------------------------------------------ gather
        const int gw = warp - kGatherWarp0;
        const bool active = gw < NGROUP;
        int32_t toff[GPW][8];
        tile_offsets<TYB, GPW, ELEM>(gw, p.patch_w, toff);
        const uint32_t gstride = static_cast<uint32_t>(p.k_pad) * 16u;  // bytes per 8-tile group
        const int nsweeps = (active && !(dbg(p) & 2)) ? p.k_pad / 32 : 0;
        int r = 0;
        for (int j = 0; dyn || j < total; ++j, ++r) {
            int t, b;
            if constexpr (dyn) {
                if (next_bid(r) < 0) break;
            } else {
                batch_of(j, t, b);
                if (b >= p.nbatch) {
                    --r;
                    continue;
                }
            }
            const int ps = r % NP;
            const uint32_t pph = (r / NP) & 1;
            const int s = r % NBB;
            mbar_wait(&patch_full[ps], pph);
            mbar_wait(&b_empty[s], ((r / NBB) & 1) ^ 1);
            gather_batch<GPW, HIN>(smem_u32(sP + ps * L.p_stride), smem_u32(sB + s * L.b_stride), sGsrc,
                              sGdst, nsweeps, gw, gstride, lane, toff, p.lo_sweep0);
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
        const int etid = threadIdx.x - kEpiWarp0 * 32;  // 0..127
        // progress publication (thread etid 0, which commits the TMA store groups):
        // iterations [0, committed) have committed stores, [0, published) are
        // published. Publishing needs the stores complete (bulk wait) and a
        // gpu-scope release, which also waits for this thread's newer stores, so it
        // is batched: every PUB_EVERY iterations (lagging PUB_LAG), and whenever the
        // epilogue has waited 2 us for an accumulator (so a stalled CTA never holds
        // back progress it has made: no circular wait between CTAs).
        constexpr int PUB_EVERY = 32;
        int committed = 0, published = 0, r = 0;
        auto publish = [&](int upto) {
            fence_proxy_async_global();
            fence_acq_rel_gpu();
            st_relaxed_gpu(p.flags + blockIdx.x, p.flag_base + static_cast<uint32_t>(upto));
            published = upto;
        };
        // mdyn: flags[b] per batch; items [published, committed) wait in sPub
        auto publish_items = [&](int upto) {
            fence_proxy_async_global();
            fence_acq_rel_gpu();
            for (int i = published; i < upto; ++i) {
                const int g = sPub[i % kPubRing], tt = g / p.nbatch;
                st_relaxed_gpu(p.flags + (g - tt * p.nbatch), p.flag_base + static_cast<uint32_t>(tt + 1));
            }
            published = upto;
        };
        for (int j = 0; dyn || j < total; ++j) {
            int t = 0, b, X0, Y0, Z0, gj = 0;
            if constexpr (dyn) {
                b = next_bid(r);
                if (b < 0) break;
                if constexpr (mdyn) {
                    if (etid == 0) sPub[j % kPubRing] = b;
                    t = b / p.nbatch;
                    b -= t * p.nbatch;
                }
                if constexpr (grp) {
                    if (p.reverse) b = nitems - 1 - b;
                    gj = b / p.nbatch;
                    b -= gj * p.nbatch;
                }
            } else {
                batch_of(j, t, b);
                if (b >= p.nbatch) {  // no-op iteration: nothing to store
                    committed = j + 1;
                    continue;
                }
            }
            batch_coords(b, X0, Y0, Z0);
            const int s = r % NACC;
            const uint32_t ph = (r / NACC) & 1;
            ++r;
            uint32_t v[NBOX][CW];
            if (dbg(p) & 32) {  // store-only ablation
#pragma unroll
                for (int c = 0; c < NBOX; ++c)
#pragma unroll
                    for (int i = 0; i < CW; ++i) v[c][i] = 0u;
            } else {
                if ((multi || mdyn) && etid == 0) {  // (constexpr: folded away otherwise)
                    const unsigned long long t0 = global_ns();
                    while (!mbar_try_wait(&d_full[s], ph)) {
                        if (published < committed && global_ns() - t0 > 2000ull) {
                            bulk_wait<0>();
                            if constexpr (mdyn)
                                publish_items(committed);
                            else
                                publish(committed);
                        }
                    }
                } else {
                    mbar_wait(&d_full[s], ph);
                }
                tc_fence_after();
                tmem_load_batch<TYB>(tmem + ((q * 32u) << 16) + static_cast<uint32_t>(s * N), v);
                tc_fence_before();  // accumulator read: hand it back to the MMA warp
                __syncwarp();
                if (lane == 0) mbar_arrive(&d_empty[s]);
            }
            if constexpr (DIMS == 2 && !HOUT)
                if (p.fold_ring != nullptr) fold_keep_ring<TYB>(p, v, X0, Y0, q, lane);
            if constexpr (grp) {  // grouped launch: the grid's map and buffer (global memory)
                if constexpr (HOUT) {
                    if (!(dbg(p) & 1))
                        store_batch_h<DIMS, TYB, NS>(p, &p.group[gj].out, reinterpret_cast<__half*>(p.group[gj].out_buf),
                                                     v, sS, L.s_stride, r - 1, X0, Y0, Z0, q, lane, etid);
                } else if (!(dbg(p) & 1)) {
                    store_batch<DIMS, TYB, NS, kEdgePlain, false>(p, &p.group[gj].out, p.group[gj].out_buf, v, sS,
                                                                   L.s_stride, r - 1, X0, Y0, Z0, q, lane, etid);
                }
            } else if constexpr (HOUT) {
                const int par = (p.src + t + 1) & 1;
                if (!(dbg(p) & 1))
                    store_batch_h<DIMS, TYB, NS, kEdgePlain, MODE == kModePeer>(
                        p, &maps.out[par], reinterpret_cast<__half*>(buf_of(p, par)), v, sS, L.s_stride, r - 1, X0,
                        Y0, Z0, q, lane, etid, nullptr, (p.peer_mask & 1) ? &p.peer_maps->up[par] : nullptr,
                        (p.peer_mask & 2) ? &p.peer_maps->down[par] : nullptr,
                        reinterpret_cast<__half*>(par ? p.peer_up_buf[1] : p.peer_up_buf[0]),
                        reinterpret_cast<__half*>(par ? p.peer_down_buf[1] : p.peer_down_buf[0]));
            } else if (!(dbg(p) & 1))
            {
                const int par = (p.src + t + 1) & 1;
                store_batch<DIMS, TYB, NS, kEdgePlain, peer>(
                    p, &maps.out[par], buf_of(p, par), v, sS, L.s_stride, r - 1, X0, Y0, Z0, q, lane, etid,
                    nullptr, (p.peer_mask & 1) ? &p.peer_maps->up[par] : nullptr,
                    (p.peer_mask & 2) ? &p.peer_maps->down[par] : nullptr, par ? p.peer_up_buf[1] : p.peer_up_buf[0],
                    par ? p.peer_down_buf[1] : p.peer_down_buf[0]);
            }
            committed = j + 1;
            if (multi && etid == 0 && committed - published >= PUB_EVERY + PUB_LAG) {
                bulk_wait<PUB_LAG>();
                publish(committed - PUB_LAG);
            }
            if (mdyn && etid == 0 && committed - published >= kPubEvery + kPubLag) {
                bulk_wait<kPubLag>();
                publish_items(committed - kPubLag);
            }
        }
        if (etid == 0) {
            bulk_wait<0>();  // stores globally complete before the CTA retires
            if (multi) publish(committed);
            if (mdyn) publish_items(committed);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (p.trace && threadIdx.x == 0) {
        unsigned long long* t = p.trace + 4 * blockIdx.x;
        t[0] = smid() | (static_cast<unsigned long long>(tmem_slot[1]) << 32);
        t[1] = t_start;
        t[2] = t_main;
        t[3] = global_ns();
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, static_cast<uint32_t>(p.tmem_cols));
    }
}

}  // namespace sst
