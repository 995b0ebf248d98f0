// mlp_tc.cuh — the predictor on the 5th-generation tensor cores (tcgen05),
// fused with the feature stage and the grid sweep.  Included by mlp.cu inside
// its anonymous namespace (shares Job, Stats, the sweep and output helpers).
//
// Precision: layers 1-2 are 3xTF32 products, D = Ah.Bh + Ah.Bl + Al.Bh with
// Xh = rna_tf32(X), Xl = X - Xh for activations and weights alike (~22
// mantissa bits per product, FP32 accumulation in TMEM); layers 3-4 run in
// FP32 on the FMA pipe.  Inside the 1e-5 relative contract on the predicted
// parameters (tests/test_gpu_tc.py, and test_gpu_mlp.py /
// test_gpu_pipeline.py run on both engines).
//
// Execution model — one persistent CTA per SM, 13 working warps (16 launched:
// setmaxnreg moves the idle warps' registers to the producers and epilogues),
// tiles of 128 kernels (the MMA M: TMEM lane m = kernel m of the tile), two
// tiles in flight:
//   * warps 0..3, PRODUCERS (thread = kernel): the feature stage of each tile
//     (CSR entries -> exact per-category fractions in a per-kernel list in
//     layer-1 K order; dense counts or fused input loaded a few chunks ahead),
//     split hi/lo and written 8 columns at a time into a 2-deep ring of
//     shared-memory chunks in the UMMA core-matrix layout — the L1 A operand.
//     CSR tiles skip the 8-column chunks no kernel of the tile touches (their
//     products are exact zeros); the K axis puts the 24 common PTX categories
//     first (tc_pos) so typical kernels touch 4 of 17 chunks;
//   * warp 12, lane 0: the MMA ISSUER.  L1 (N 112 x K 136) reads A from the
//     ring (SS), L2 (64 x 104) reads A from TMEM (TS); each k-step is three
//     kind::tf32 MMAs issued as soon as its 8-column chunk is ready (an event
//     loop over non-blocking mbarrier tests: L1 of the next tile interleaved
//     with L2 of the current one); tcgen05.commit frees ring buffers and
//     signals finished layers;
//   * warps 4..7 / 8..11, two EPILOGUE GROUPS taking alternate tiles, each
//     with its own TMEM slot: tcgen05.ld -> bias + sigmoid -> split ->
//     tcgen05.st of A2 in place over the consumed D1; then D2 -> sigmoid into
//     registers, layers 3-4 on the FMA pipe, clamp, the grid sweep of the tile
//     (thread = kernel) and the outputs — one group's tail overlaps the other
//     group's tile on the tensor core.
// TMEM (512 columns): slot g at 216 g: [0,112) D1 -> A2 hi (in place),
// [112,216) A2 lo; [432,496) D2 (shared, guarded by D2FREE); [496 + 8 g, +8)
// predictions computed on the FMA pipe.
//
// Non-finite inputs (a DCGM value, or any predict-mode feature): the producer
// computes that kernel's prediction on the FMA pipe (tc_forward_x, IEEE
// semantics like the reference) into the slot's spare TMEM columns and flags
// the row; a split inf - inf would otherwise turn inf * W into NaN.
// Non-finite weights never reach this engine (the host or a device flag routes
// such models to the FFMA engine, ws_kernel).

namespace tce {

constexpr int TT = 128;                            // kernels per tile
constexpr int kGroupT = 128;                       // threads of a role group (4 warps)
constexpr int kThreadsTC = 4 * kGroupT;  // producers, 2 epilogue groups, MMA warp (+3 idle)
// Role warpgroups.  The SMSP arbiter favours the highest warp id, so the latency-
// critical producers take the top warpgroup; the MMA issuer (mostly blocked in
// mbarrier waits) the lowest; its other three warps are idle.
constexpr int MMA_WG = 0, EPI_WG0 = 1, PROD_WG = 3;
constexpr int MMA_WARP = 4 * MMA_WG;
#ifndef DSO_MMA_SLEEP_NS
#define DSO_MMA_SLEEP_NS 256
#endif
constexpr unsigned kMmaSleepNs = DSO_MMA_SLEEP_NS;  // MMA issuer: barrier sleep while two event streams are open
#ifndef DSO_L3_UNROLL
#define DSO_L3_UNROLL 50
#endif
constexpr int kL3Unroll = DSO_L3_UNROLL;  // layer-3 input neurons per unrolled step
#ifndef DSO_TC_SWEEP_UNR
#define DSO_TC_SWEEP_UNR 4  // independent sweep groups per step in the epilogue
#endif
#ifndef DSO_EPI1_BATCH
#define DSO_EPI1_BATCH 4
#endif
constexpr int kEpi1Batch = DSO_EPI1_BATCH;
#ifndef DSO_EPI1_UNROLL
#define DSO_EPI1_UNROLL 1
#endif
constexpr int kEpi1Unroll = DSO_EPI1_UNROLL;  // layer-1 epilogue batches per unrolled step  // layer-1 epilogue chunks per TMEM load/store wait
// Registers (setmaxnreg): launched at 128 per thread; the MMA warpgroup (the MMA
// warp and three idle warps) releases down to 56, producers grow to 168 and the
// epilogue groups to 144 (128*168 + 256*144 + 128*56 = 64K).
constexpr int kRegLaunch = 128;  // ptxas allocation at launch (checked by launch_tc)
#ifndef DSO_REG_PROD
#define DSO_REG_PROD 168
#endif
#ifndef DSO_REG_EPI
#define DSO_REG_EPI 144
#endif
constexpr int kRegProd = DSO_REG_PROD, kRegEpi = DSO_REG_EPI, kRegMma = 56;
static_assert(128 * (kRegLaunch - kRegMma) >= 128 * (kRegProd - kRegLaunch) + 256 * (kRegEpi - kRegLaunch),
              "setmaxnreg: increases must be covered by releases");
constexpr int N1 = 112, K1 = 136, N2 = 64, K2 = 104;
constexpr int H1 = 100, H2 = 50, H3 = 25, H4 = 7;
// packed model (floats): L1/L2 weights hi/lo in the SWIZZLE_NONE K-major
// core-matrix layout (tc.cuh); L3/L4 (1,425 weights) stay FP32 for the FMA
// pipe, transposed [k][n] with n padded to 28 / 8 (FFMA2 neuron pairs);
// -b*log2(e) for the hidden layers, b4, the non-finite count
constexpr int W1H = 0, W1L = W1H + N1 * K1, W2H = W1L + N1 * K1, W2L = W2H + N2 * K2;
constexpr int W3T = W2L + N2 * K2, W4T = W3T + H2 * 28;
constexpr int NB1 = W4T + H3 * 8, NB2 = NB1 + N1, NB3 = NB2 + N2, B4 = NB3 + 32;
constexpr int FLAG = B4 + 16;
constexpr int kModel = FLAG + 4;
__host__ __device__ __forceinline__ int cm(int n, int k, int K) {
    return ((n >> 3) * (K >> 2) + (k >> 2)) * 32 + (n & 7) * 4 + (k & 3);
}
// Layer-1 K order of the count slots: the 24 categories every PTX kernel tends to
// list first (the set the reference's own synthetic kernels fill,
// ptx_features.cpp:18-49 / sim_harness.cpp:70-95: add mul fma setp mov ld st cvt
// bra ret bar | s32 u32 u64 f32 f64 b32 b64 | reg const global local param
// shared), then the other 102 in slot order.  A fixed relabelling of the K axis
// (weights packed to match), so the 8-column chunks of layer 1 that a tile leaves
// all-zero — skipped exactly — are as many as possible: 3 count chunks instead of
// up to 16 for such kernels.
__host__ __device__ __forceinline__ int common_slot(int i) {
    constexpr int kCommon[24] = {0,   4,   37,  39,  51,  54,  56,  61,  71,  74,  76,  103,
                                 107, 108, 111, 112, 115, 116, 118, 120, 121, 122, 123, 124};
    return kCommon[i];
}
__host__ __device__ inline int tc_pos(int slot) {  // slot -> position on the K axis (- 8)
    int below = 0;
    for (int i = 0; i < 24; ++i) {
        if (common_slot(i) == slot) return i;
        below += common_slot(i) < slot ? 1 : 0;
    }
    return 24 + slot - below;
}
// shared memory (floats)
#ifndef DSO_TC_RING
#define DSO_TC_RING 2
#endif
constexpr int kRing = DSO_TC_RING;           // X chunk buffers
static_assert(kRing <= 3, "ring barriers: MB_XFULL / MB_XEMPTY hold 3 each");
constexpr int kChunkF = 2 * TT * 8;          // hi [128][8] + lo [128][8] (core-matrix layout)
constexpr int S_STATS = kModel;              // mean[8] std[8]
constexpr int S_RING = S_STATS + 16;
constexpr int S_MISC = S_RING + kRing * kChunkF;  // u32: [0..1] chunk masks, [2..9] slow rows, [10..17] partial masks
constexpr int S_PERM = S_MISC + 24;  // u8 pos_of[128] (slot -> K position), slot_at[128]
// CSR per-slot tables: u64 chunk_one[128] (1 << 4 (chunk - 1): a row's live entries
// per chunk, 4 bits each, by one 64-bit add; 0 for slots >= 126) and u8 offl[128]
// (the slot's float offset inside a chunk row of the core-matrix layout)
constexpr int S_SLOTLUT = S_PERM + 64;
constexpr int S_OFFL = S_SLOTLUT + 256;
// CSR: the entries of tiles t and t+1, each bulk-copied a tile ahead into its own
// buffer (the tile's entry range widened to 16-byte boundaries).  Per buffer meta: [0,1] first staged entry index, [2]
// staged flag.  A tile whose range does not fit reads its entries from global.
// (26.9 entries per kernel on average fit.)
constexpr int kStageEnt = 3440;
constexpr int S_ESTAGE = S_OFFL + 32;
constexpr int S_EMETA = S_ESTAGE + 2 * kStageEnt;
constexpr int S_MBAR = S_EMETA + 8;
enum {
    MB_XFULL = 0, MB_XEMPTY = 3, MB_D1F = 6, MB_A2R = 8, MB_D2F = 34, MB_D2FREE = 36,
    MB_SLOWFREE = 37, MB_ESTAGE = 39, kMbars = 41
};
static_assert(S_ESTAGE % 4 == 0 && kStageEnt % 4 == 0, "bulk-copy destinations are 16-byte aligned");
constexpr int S_TSLOT = S_MBAR + 2 * kMbars;
constexpr int S_TABLES = (S_TSLOT + 4 + 3) & ~3;  // core4[nc], mem2[nm], level pairs
static_assert(kModel % 4 == 0 && S_RING % 4 == 0 && S_MBAR % 2 == 0, "tc smem alignment");
__host__ __device__ __forceinline__ int tc_pairs_offset(int nc, int nm) {
    return (S_TABLES + 4 * nc + 2 * nm + 3) & ~3;
}
// TMEM columns
constexpr int SLOT_COLS = 216, TD2 = 432, TSLOW = 496;
constexpr int A2LO = 112;
constexpr float kNL2E = -1.4426950408889634f;

// phase accounting (debug library only): producer 0, epilogue thread 128, MMA thread
#ifdef DSO_PHASE_TIMING
#define TPT_BEGIN(v) long long v = clock64()
#define TPT_END(ph, v)                                                              \
    do {                                                                            \
        if (threadIdx.x == 0 || threadIdx.x == kGroupT || threadIdx.x == 3 * kGroupT) \
            atomicAdd(&g_phase_cycles[ph], clock64() - (v));                        \
    } while (0)
#else
#define TPT_BEGIN(v) (void)0
#define TPT_END(ph, v) (void)0
#endif

// event timeline of CTA 0 (debug builds with -DDSO_TC_TRACE; dso_debug_trace)
#ifdef DSO_TC_TRACE
#define TRACE(ev, t)                                                   \
    do {                                                               \
        if (blockIdx.x == 0 && (t) < 64) g_trace[(ev) * 64 + (t)] = clock64(); \
    } while (0)
#else
#define TRACE(ev, t) (void)0
#endif

__device__ __forceinline__ void mb_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// The warp's tcgen05 traffic is complete and ordered before one arrival on b.
__device__ __forceinline__ void warp_signal(uint64_t* b) {
    tc::wait_st();
    tc::fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mb_arrive(b);
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Blocking test: suspends the thread (no issue slots used) until the phase with
// the given parity completes or about `ns` nanoseconds pass; true if completed.
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity, uint32_t ns) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity), "r"(ns)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void wait_acq(uint64_t* b, uint32_t ph) {
    mbar_wait(b, ph);
    tc::fence_after();
}

// hi/lo split of 8 values into two TMEM chunks
__device__ __forceinline__ void store_split(uint32_t a_hi, uint32_t a_lo, const float (&v)[8]) {
    float h[8], l[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        h[j] = tc::tf32_hi_finite(v[j]);  // sigmoid outputs: finite
        l[j] = v[j] - h[j];
    }
    tc::st8(a_hi, h);
    tc::st8(a_lo, l);
}

// Activation of one loaded 8-neuron chunk: sigmoid(acc + b) (neurons >= NREAL are
// padding: 0), split, stored as the next layer's A operand (not yet waited on).
template <int NREAL>
__device__ __forceinline__ void epi_act_store(const float (&v)[8], int c,
                                              const float* __restrict__ nb, uint32_t dst_hi,
                                              uint32_t dst_lo) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
        const float2 z = ffma2(make_float2(v[j], v[j + 1]), make_float2(kNL2E, kNL2E),
                               make_float2(nb[8 * c + j], nb[8 * c + j + 1]));
        float e0, e1, r0, r1;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(z.x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(z.y));
        const float2 d = fadd2(make_float2(1.f, 1.f), make_float2(e0, e1));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
        a[j] = 8 * c + j < NREAL ? r0 : 0.f;
        a[j + 1] = 8 * c + j + 1 < NREAL ? r1 : 0.f;
    }
    store_split(dst_hi, dst_lo, a);
}

// Hidden-layer epilogue of one 8-neuron chunk: sigmoid(acc + b) (neurons >=
// NREAL are padding: 0), split, stored as the next layer's A operand.
template <int NREAL>
__device__ __forceinline__ void epi_chunk(uint32_t src, uint32_t dst_hi, uint32_t dst_lo, int c,
                                          const float* __restrict__ nb, uint64_t* ready) {
    float v[8];
    tc::ld8(src, v);
    tc::wait_ld();
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
        const float2 z = ffma2(make_float2(v[j], v[j + 1]), make_float2(kNL2E, kNL2E),
                               make_float2(nb[8 * c + j], nb[8 * c + j + 1]));
        float e0, e1, r0, r1;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(z.x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(z.y));
        const float2 d = fadd2(make_float2(1.f, 1.f), make_float2(e0, e1));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
        a[j] = 8 * c + j < NREAL ? r0 : 0.f;
        a[j + 1] = 8 * c + j + 1 < NREAL ? r1 : 0.f;
    }
    store_split(dst_hi, dst_lo, a);
    warp_signal(ready);
}

// FP32 forward of one kernel's features on the FMA pipe: W = Wh + Wl exactly,
// sequential sums, the same sigmoid as the epilogues.
__device__ __noinline__ void tc_forward_x(const float* sm, const float* x, float* raw) {
    float h1[H1], h2[H2], h3[H3];
    const uint8_t* pos_of = reinterpret_cast<const uint8_t*>(sm + S_PERM);
    auto w = [&](int hi, int lo, int n, int kk, int K) {
        return sm[hi + cm(n, kk, K)] + sm[lo + cm(n, kk, K)];
    };
    auto sig = [&](float acc, float nbv) {
        float e, r;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(acc, kNL2E, nbv)));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
        return r;
    };
    for (int n = 0; n < H1; ++n) {
        float z = 0.f;
        for (int c = 0; c < DSO_FUSED_ROWS; ++c)
            z = fmaf(w(W1H, W1L, n, c < 8 ? c : 8 + pos_of[c - 8], K1), x[c], z);
        h1[n] = sig(z, sm[NB1 + n]);
    }
    for (int n = 0; n < H2; ++n) {
        float z = 0.f;
        for (int c = 0; c < H1; ++c) z = fmaf(w(W2H, W2L, n, c, K2), h1[c], z);
        h2[n] = sig(z, sm[NB2 + n]);
    }
    for (int n = 0; n < H3; ++n) {
        float z = 0.f;
        for (int c = 0; c < H2; ++c) z = fmaf(sm[W3T + c * 28 + n], h2[c], z);
        h3[n] = sig(z, sm[NB3 + n]);
    }
    for (int n = 0; n < H4; ++n) {
        float z = 0.f;
        for (int c = 0; c < H3; ++c) z = fmaf(sm[W4T + c * 8 + n], h3[c], z);
        raw[n] = fmaf(z + sm[B4 + n], sm[S_STATS + 8 + n], sm[S_STATS + n]);
    }
}

// CSR row of one kernel (thread = kernel): extent and DCGM prefetched a tile
// ahead in registers; the entries themselves are read from the tile's staged copy
// in shared memory (or from global when the tile was not staged).
struct Entries {
    uint64_t first;
    int cnt;
    float dg[8];
};
// The next tile's row extent and DCGM as raw loads: nothing consumes them until
// the tile changes (tc_csr_take), so their HBM latency hides behind this tile
// (deriving first / cnt at load time stalled the producer on every tile).
struct EntriesRaw {
    uint64_t a, b;
    float dg[8];
};

__device__ __forceinline__ void tc_csr_prefetch(const Job& J, int64_t k, EntriesRaw& R) {
    const int64_t kk = k < J.n ? k : J.n - 1;  // in bounds; tail rows are zeroed on take
    R.a = __ldg(J.row_ptr + kk);
    R.b = __ldg(J.row_ptr + kk + 1);
#pragma unroll
    for (int j = 0; j < 8; ++j) R.dg[j] = __ldg(J.dcgm + (int64_t)j * J.ld + kk);
}
__device__ __forceinline__ void tc_csr_take(const Job& J, int64_t k, const EntriesRaw& R,
                                            Entries& E) {
    const bool in = k < J.n;
    E.first = in ? R.a - J.ent_base : 0;
    E.cnt = in ? (int)(R.b - R.a) : 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) E.dg[j] = in ? R.dg[j] : 0.f;
}

// exact per-category totals -> (tf, rr) for normalize_count (see csr_features)
__device__ __forceinline__ void cat_scales(const uint64_t (&tot)[3], float (&tf)[3], float (&rr)[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        tf[c] = 0.f;
        rr[c] = 0.f;
        if (tot[c] != 0 && tot[c] < (1u << 24)) {
            tf[c] = __uint2float_rn((uint32_t)tot[c]);
            rr[c] = __frcp_rn(tf[c]);
        } else if (tot[c] != 0) {
            tf[c] = -(float)(tot[c] >> 24);
            rr[c] = (float)(tot[c] & 0xFFFFFFu);
        }
    }
}
// normalize_count without the wide-total branch: valid for tf >= 0 (a zero
// total has only zero counts: 0 * 0 -> 0); kernels with a total >= 2^24 take
// the general path
__device__ __forceinline__ float norm_fast(uint32_t c, int slot, const float (&tf)[3],
                                           const float (&rr)[3]) {
    const int cat = cat_of_row(slot);
    const float t = cat == 0 ? tf[0] : (cat == 1 ? tf[1] : tf[2]);
    const float r = cat == 0 ? rr[0] : (cat == 1 ? rr[1] : rr[2]);
    const float cf = (__int_as_float(0x4B000000u | (c & 0x7FFFFFu)) - 8388608.f) +
                     ((c & 0x800000u) ? 8388608.f : 0.f);
    const float qq = __fmul_rn(cf, r);
    return fmaf(fmaf(-qq, t, cf), r, qq);
}
__device__ __forceinline__ float norm_slot(uint32_t cnt, int slot, const float (&tf)[3],
                                           const float (&rr)[3]) {
    const int cat = cat_of_row(slot);
    return normalize_count(cnt, cat == 0 ? tf[0] : (cat == 1 ? tf[1] : tf[2]),
                           cat == 0 ? rr[0] : (cat == 1 ? rr[1] : rr[2]));
}

// st.shared.f32 under a predicate (no branch around the store)
__device__ __forceinline__ void sts_pred(uint32_t a, float v, bool p) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.f32 [%0], %1; }" ::"r"(a), "f"(v),
                 "r"((uint32_t)p)
                 : "memory");
}

// One 8-column chunk of one kernel into a ring buffer (core-matrix layout).
__device__ __forceinline__ void put_chunk(float* buf, int row, const float (&v)[8]) {
    float h[8], l[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        h[j] = tc::tf32_hi(v[j]);
        l[j] = v[j] - h[j];
    }
    const int o = (row >> 3) * 64 + (row & 7) * 4;
    *reinterpret_cast<float4*>(buf + o) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(buf + o + 32) = make_float4(h[4], h[5], h[6], h[7]);
    *reinterpret_cast<float4*>(buf + TT * 8 + o) = make_float4(l[0], l[1], l[2], l[3]);
    *reinterpret_cast<float4*>(buf + TT * 8 + o + 32) = make_float4(l[4], l[5], l[6], l[7]);
}

// The tensor-core pipeline kernel.  MODE_PRED: fused [134][ld] input, outputs
// raw/params/clamped; MODE_DENSE: [126][ld] counts + DCGM; MODE_CSR: CSR
// counts + DCGM; the pipeline modes run the fused sweep.
template <int MODE>
__global__ void __launch_bounds__(kThreadsTC, 1)
    tc_kernel(const float* __restrict__ model, Stats stats, Job J) {
    constexpr bool PIPE = MODE != MODE_PRED;
    extern __shared__ __align__(16) float sm[];
    if (reinterpret_cast<const int*>(model)[FLAG] != 0) return;  // non-finite weights: FFMA engine
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint64_t* mb = reinterpret_cast<uint64_t*>(sm + S_MBAR);
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + S_MISC);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + S_TSLOT);
    {
        const float4* src = reinterpret_cast<const float4*>(model);
        float4* dst = reinterpret_cast<float4*>(sm);
        for (int i = tid; i < kModel / 4; i += kThreadsTC) dst[i] = __ldg(src + i);
        if (tid < 8) {
            sm[S_STATS + tid] = stats.mean[tid];
            sm[S_STATS + 8 + tid] = stats.std_[tid];
        }
        if (tid < 24) misc[tid] = 0u;
        if (tid < DSO_COUNT_ROWS) {
            uint8_t* pm = reinterpret_cast<uint8_t*>(sm + S_PERM);
            const int ps = tc_pos(tid);
            pm[tid] = (uint8_t)ps;
            pm[128 + ps] = (uint8_t)tid;
        }
        if (tid < 128) {
            const int ps = tid < DSO_COUNT_ROWS ? tc_pos(tid) : 0;
            reinterpret_cast<uint64_t*>(sm + S_SLOTLUT)[tid] =
                tid < DSO_COUNT_ROWS ? 1ull << (4 * ((ps + 8) >> 3) - 4) : 0ull;
            reinterpret_cast<uint8_t*>(sm + S_OFFL)[tid] = (uint8_t)(((ps & 7) >> 2) * 32 + (ps & 3));
        }
        if (PIPE) {
            float4* sc = reinterpret_cast<float4*>(sm + S_TABLES);
            float2* smm = reinterpret_cast<float2*>(sm + S_TABLES + 4 * J.nc);
            for (int i = tid; i < J.nc; i += kThreadsTC) sc[i] = J.core4[i];
            for (int j = tid; j < J.nm; j += kThreadsTC) smm[j] = J.mem2[j];
            if (J.pairs)
                build_pairs(reinterpret_cast<float4*>(sm + tc_pairs_offset(J.nc, J.nm)), J.core4,
                            J.nc);
        }
        if (tid == 0) {
            for (int b = 0; b < kRing; ++b) {
                mb_init(mb + MB_XFULL + b, 4);
                mb_init(mb + MB_XEMPTY + b, 1);
            }
            for (int g = 0; g < 2; ++g) {
                mb_init(mb + MB_D1F + g, 1);
                mb_init(mb + MB_D2F + g, 1);
                mb_init(mb + MB_SLOWFREE + g, 4);
                for (int c = 0; c < 13; ++c) mb_init(mb + MB_A2R + 13 * g + c, 4);
            }
            mb_init(mb + MB_D2FREE, 4);
            mb_init(mb + MB_ESTAGE, 1);
            mb_init(mb + MB_ESTAGE + 1, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        if (warp == MMA_WARP) tc::tmem_alloc<512>(tslot);
        // weights written through the generic proxy are read by the tensor core
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tslot;
    const int64_t tiles = (J.n + TT - 1) / TT;
    const int64_t my_tiles =
        (int64_t)blockIdx.x < tiles ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto t0_of = [&](int64_t i) { return (blockIdx.x + i * gridDim.x) * (int64_t)TT; };

    if ((warp >> 2) == MMA_WG) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegMma));
    }
    if (warp == MMA_WARP || warp == MMA_WARP + 1) {
        // ============================== MMA issuers ===============================
        // Two threads in two warps (two SMSPs), each sleeping in the mbarrier of its
        // own next event, no polling: warp MMA_WARP issues layer 1 (chunk by chunk
        // as the producers hand them over), warp MMA_WARP + 1 layer 2 (chunk by
        // chunk as the epilogue group stores A2).  Tile t's layer 1 reuses the TMEM
        // slot of tile t-2, so it starts once layer 2 of tile t-2 has completed
        // (its commit barrier MB_D2F): no ordering between the two issuers' MMAs
        // is assumed.
        if (lane == 0) {
            const uint32_t id1 = tc::idesc_tf32(128, N1), id2 = tc::idesc_tf32(128, N2);
            const uint32_t s0 = smem_u32(sm);
            auto bd = [&](int off, int kk, int K) {
                return tc::sdesc(s0 + off * 4 + kk * 256, 128, (uint32_t)(K >> 2) * 128);
            };
            unsigned long long n_k = 0;  // k-steps issued (evidence counters)
            if (warp == MMA_WARP) {
                uint32_t g = 0;  // ring chunks consumed
                for (int64_t t = 0; t < my_tiles; ++t) {
                    const int sl = (int)(t & 1);
                    if (t >= 2) mbar_wait(mb + MB_D2F + sl, (uint32_t)(((t >> 1) - 1) & 1));
                    const uint32_t D = tbase + (uint32_t)(sl * SLOT_COLS);
                    uint32_t mask = 0u;
                    for (int c = 0; c < 17; ++c) {
                        const int b = (int)(g % kRing);
                        if (c > 0 && !((mask >> c) & 1u)) continue;
                        mbar_wait(mb + MB_XFULL + b, (g / kRing) & 1u);
                        tc::fence_after();
                        if (c == 0) {
                            mask = misc[sl];  // published before the tile's first chunk
                            TRACE(0, t);
                        }
                        const uint32_t xa = s0 + (uint32_t)(S_RING + b * kChunkF) * 4;
                        const uint64_t ah = tc::sdesc(xa, 128, 256),
                                       al = tc::sdesc(xa + TT * 8 * 4, 128, 256);
                        tc::mma_tf32_ss(D, ah, bd(W1H, c, K1), id1, c == 0 ? 0u : 1u);
                        tc::mma_tf32_ss(D, ah, bd(W1L, c, K1), id1, 1u);
                        tc::mma_tf32_ss(D, al, bd(W1H, c, K1), id1, 1u);
                        tc::commit(mb + MB_XEMPTY + b);
                        ++g;
                        ++n_k;
                    }
                    tc::commit(mb + MB_D1F + sl);
                    TRACE(1, t);
                }
                if (J.counters) {
                    atomicAdd(J.counters + 0, n_k);
                    atomicAdd(J.counters + 2, (unsigned long long)my_tiles);
                }
            } else {
                for (int64_t t = 0; t < my_tiles; ++t) {
                    const int sl = (int)(t & 1);
                    const uint32_t S = tbase + (uint32_t)(sl * SLOT_COLS);
                    const uint32_t ph = (uint32_t)((t >> 1) & 1);
                    // D2 is free once the previous tile's epilogue has read it
                    if (t >= 1) mbar_wait(mb + MB_D2FREE, (uint32_t)((t - 1) & 1));
                    for (int c2 = 0; c2 < 13; ++c2) {
                        mbar_wait(mb + MB_A2R + 13 * sl + c2, ph);
                        tc::fence_after();
                        tc::mma_tf32_ts(tbase + TD2, S + 8 * c2, bd(W2H, c2, K2), id2, c2 > 0 ? 1u : 0u);
                        if (c2 == 0) TRACE(2, t);
                        tc::mma_tf32_ts(tbase + TD2, S + 8 * c2, bd(W2L, c2, K2), id2, 1u);
                        tc::mma_tf32_ts(tbase + TD2, S + A2LO + 8 * c2, bd(W2H, c2, K2), id2, 1u);
                        ++n_k;
                    }
                    tc::commit(mb + MB_D2F + sl);
                    TRACE(3, t);
                }
                if (J.counters) atomicAdd(J.counters + 1, n_k);
            }
        }
        __syncwarp();
    } else if ((warp >> 2) == MMA_WG) {
        // idle warps (they only hand their registers to the other roles)
    } else if ((warp >> 2) == PROD_WG) {
        // ================================ producers ================================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegProd));
        const uint8_t* pos_of = reinterpret_cast<const uint8_t*>(sm + S_PERM);
        const uint8_t* slot_at = pos_of + 128;
        const int ptid = tid - PROD_WG * kGroupT, pw = warp & 3;
        const int row = ptid;  // kernel of the tile; TMEM lane quadrant = pw
        const uint32_t tq = tbase + ((uint32_t)(32 * pw) << 16);
        uint32_t g = 0;  // ring chunks produced
        Entries E;
        if (MODE == MODE_CSR && my_tiles > 0) {
            EntriesRaw R0;
            tc_csr_prefetch(J, t0_of(0) + row, R0);
            tc_csr_take(J, t0_of(0) + row, R0, E);
        }
        // CSR: thread 0 bulk-copies tile i's entry range, widened to 16-byte boundaries,
        // into stage buffer i & 1 (one cp.async.bulk completing on MB_ESTAGE + (i & 1));
        // when the widened range does not fit, or would leave the batch's entry array,
        // it only arrives and the tile reads its entries from global
        uint64_t ent_total = 0;  // entries of the batch (thread 0)
        if (MODE == MODE_CSR && ptid == 0) ent_total = __ldg(J.row_ptr + J.n) - J.ent_base;
        auto stage = [&](int64_t i) {
            if (MODE != MODE_CSR || ptid != 0) return;
            const int sb = (int)(i & 1);
            const int64_t t0i = t0_of(i), t1i = t0i + TT < J.n ? t0i + TT : J.n;
            const uint64_t a = __ldg(J.row_ptr + t0i) - J.ent_base, b = __ldg(J.row_ptr + t1i) - J.ent_base;
            const uint64_t mis = (reinterpret_cast<uintptr_t>(J.entries + a) & 15) >> 2;
            const uint64_t a4 = a - mis, b4 = a4 + ((b - a4 + 3) & ~3ull);
            uint32_t* meta = reinterpret_cast<uint32_t*>(sm + S_EMETA) + 4 * sb;
            const bool ok = b > a && a >= mis && b4 <= ent_total && b4 - a4 <= (uint64_t)kStageEnt;
            meta[0] = (uint32_t)a4;
            meta[1] = (uint32_t)(a4 >> 32);
            meta[2] = ok ? 1u : 0u;
            const uint32_t bar = smem_u32(mb + MB_ESTAGE + sb);
            if (ok) {
                const uint32_t bytes = (uint32_t)(b4 - a4) * 4u;
                // the buffer was last read through the generic proxy (the barrier before
                // this call ordered every producer's reads); the bulk copy writes it
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                             "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(sm + S_ESTAGE + sb * kStageEnt)),
                    "l"(J.entries + a4), "r"(bytes), "r"(bar)
                    : "memory");
            } else {
                mb_arrive(mb + MB_ESTAGE + sb);
            }
        };
        if (my_tiles > 0) stage(0);
        for (int64_t t = 0; t < my_tiles; ++t) {
            const int64_t k = t0_of(t) + row;
            const int sl = (int)(t & 1);
            EntriesRaw NE;  // next tile's row extent and DCGM, in flight during this tile
            if (MODE == MODE_CSR && t + 1 < my_tiles) tc_csr_prefetch(J, t0_of(t + 1) + row, NE);
            // predict / dense: the input rows of tile t+2 into L2 (bulk prefetches, one
            // 512-byte row segment per thread, no registers or shared memory held), so
            // the chunk loads below hit L2 rather than HBM
            if (MODE != MODE_CSR && t + 2 < my_tiles) {
                const int64_t tp = t0_of(t + 2);
                const int nrows = MODE == MODE_PRED ? DSO_FUSED_ROWS : DSO_COUNT_ROWS + 8;
                if (tp + TT <= J.n && (J.ld & 3) == 0 && row < nrows) {
                    const void* src = MODE == MODE_PRED
                                          ? (const void*)(J.fused + (int64_t)row * J.ld + tp)
                                      : row < 8 ? (const void*)(J.dcgm + (int64_t)row * J.ld + tp)
                                                : (const void*)(J.counts + (int64_t)(row - 8) * J.ld + tp);
                    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src),
                                     "r"((uint32_t)(TT * 4))
                                     : "memory");
                }
                if (row + kGroupT < nrows) {  // (rows 128..133 of the fused input)
                    const int r2 = row + kGroupT;
                    const void* src2 = MODE == MODE_PRED
                                           ? (const void*)(J.fused + (int64_t)r2 * J.ld + tp)
                                           : (const void*)(J.counts + (int64_t)(r2 - 8) * J.ld + tp);
                    if (tp + TT <= J.n && (J.ld & 3) == 0 && (reinterpret_cast<uintptr_t>(src2) & 15) == 0)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src2),
                                     "r"((uint32_t)(TT * 4))
                                     : "memory");
                }
            }
            TPT_BEGIN(p_t);
            if (ptid == 0) TRACE(4, t);
            // ---- per-kernel preparation: totals, chunk mask, non-finite rows ----
            float tf[3] = {0.f, 0.f, 0.f}, rr[3] = {0.f, 0.f, 0.f};
            uint32_t mask = 1u;   // chunks this kernel touches (chunk 0: DCGM)
            bool uns = false;     // CSR: general path (unsorted / duplicate slots, > 64
                                  // entries, a category total >= 2^24)
            bool bad = false;     // a non-finite feature: FMA-pipe forward
            uint64_t nib = 0;     // CSR: live entries per chunk 1..16, 4 bits each
            uint64_t cbits = 0;   // CSR: row positions of the entries in the common
            uint64_t obits = 0;   //   categories (chunks 1-3) and of the others (4-16)
            const int sb = (int)(t & 1);
            bool staged = false;
            const uint32_t* s_row = nullptr;  // CSR: this kernel's staged entries
            if (MODE == MODE_CSR) {
                TPT_BEGIN(p_l);
                mbar_wait(mb + MB_ESTAGE + sb, (uint32_t)((t >> 1) & 1));
                {
                    const uint32_t* meta = reinterpret_cast<const uint32_t*>(sm + S_EMETA) + 4 * sb;
                    staged = meta[2] != 0;
                    const uint64_t base = meta[0] | ((uint64_t)meta[1] << 32);
                    // (an empty row, e.g. past the batch end, points at the buffer start:
                    // pass B reads a valid word for its predicated-off slots)
                    s_row = reinterpret_cast<const uint32_t*>(sm + S_ESTAGE + sb * kStageEnt) +
                            (E.cnt > 0 ? E.first - base : 0);
                }
                // pass A, one visit per entry: category totals (suffix sums over the slot
                // order: all, dtype + memspace (slot >= 101), memspace (slot >= 118)),
                // live entries per chunk (one table add), and which entries are common-
                // category ones (K positions 0..23, chunks 1-3, first; the others follow;
                // both in slot order).  Positions past the row read the sentinel 127
                // (count 0, table 0).  Unsorted / duplicate / out-of-range slots, rows over
                // 64 entries and totals >= 2^24 take the general path below.
                const uint64_t* chunk_one = reinterpret_cast<const uint64_t*>(sm + S_SLOTLUT);
                uint32_t ta = 0u, t12 = 0u, t2 = 0u;
                int prev = -1;
                const int ce = E.cnt;
                uns = ce > 64;
                auto group = [&](const uint32_t (&en)[4], int e0) {
                    uint32_t cb4 = 0u;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int slot = (int)(en[u] & 127u);
                        const uint32_t c = en[u] >> 7;
                        const bool tail = e0 + u >= ce;
                        uns |= !tail && (slot <= prev || slot >= DSO_COUNT_ROWS);
                        prev = slot;
                        ta += c;
                        t12 += slot >= DSO_INSTR_SLOTS ? c : 0u;
                        t2 += slot >= DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS ? c : 0u;
                        const uint64_t one = chunk_one[slot];
                        nib += one;
                        cb4 |= ((uint32_t)one & 0xFFFu) ? 1u << u : 0u;
                    }
                    cbits |= (uint64_t)cb4 << e0;
                };
                if (!uns) {
                    if (staged) {
#ifdef DSO_TC_PA8
#pragma unroll 1
                        for (int e0 = 0; e0 < ce; e0 += 8) {
                            uint32_t en[4], en2[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t v = s_row[e0 + u < ce ? e0 + u : 0];
                                const uint32_t v2 = s_row[e0 + 4 + u < ce ? e0 + 4 + u : 0];
                                en[u] = e0 + u < ce ? v : 127u;
                                en2[u] = e0 + 4 + u < ce ? v2 : 127u;
                            }
                            group(en, e0);
                            group(en2, e0 + 4);
                        }
#else
#pragma unroll 1
                        for (int e0 = 0; e0 < ce; e0 += 4) {
                            uint32_t en[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t v = s_row[e0 + u < ce ? e0 + u : 0];
                                en[u] = e0 + u < ce ? v : 127u;
                            }
                            group(en, e0);
                        }
#endif
                    } else {
                        const uint32_t* gp = J.entries + E.first;
#pragma unroll 1
                        for (int e0 = 0; e0 < ce; e0 += 4) {
                            uint32_t en[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t v = __ldg(gp + (e0 + u < ce ? e0 + u : 0));
                                en[u] = e0 + u < ce ? v : 127u;
                            }
                            group(en, e0);
                        }
                    }
                    obits = (ce == 64 ? ~0ull : (1ull << ce) - 1ull) & ~cbits;
                    const uint64_t tot[3] = {ta - t12, t12 - t2, t2};
                    cat_scales(tot, tf, rr);
                    uns |= tf[0] < 0.f || tf[1] < 0.f || tf[2] < 0.f;  // a total >= 2^24
                }
                // chunk mask from the per-chunk counts
#pragma unroll
                for (int c = 1; c <= 16; ++c) mask |= ((nib >> (4 * c - 4)) & 15u) ? 1u << c : 0u;
                if (uns) {
                    // general path: totals (64-bit, duplicates added, slots >= 126 ignored)
                    // and chunk mask over every entry
                    uint64_t tot[3] = {0, 0, 0};
                    mask = 1u;
                    for (int idx = 0; idx < ce; ++idx) {
                        const uint32_t en = __ldg(J.entries + E.first + idx);
                        const int slot = (int)(en & 127u);
                        if (slot < DSO_COUNT_ROWS) {
                            const int cat = cat_of_row(slot);
                            tot[0] += cat == 0 ? (en >> 7) : 0u;
                            tot[1] += cat == 1 ? (en >> 7) : 0u;
                            tot[2] += cat == 2 ? (en >> 7) : 0u;
                            mask |= 1u << ((8 + pos_of[slot]) >> 3);
                        }
                    }
                    cat_scales(tot, tf, rr);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) bad |= !isfinite(E.dg[j]);
                TPT_END(16, p_l);
            } else if (MODE == MODE_DENSE) {
                uint64_t tot[3] = {0, 0, 0};
                if (k < J.n) {
#pragma unroll 1
                    for (int r0 = 0; r0 < DSO_COUNT_ROWS; r0 += 42) {
                        uint32_t cv[42];
#pragma unroll
                        for (int u = 0; u < 42; ++u)
                            cv[u] = __ldg(J.counts + (int64_t)(r0 + u) * J.ld + k);
#pragma unroll
                        for (int u = 0; u < 42; ++u) {
                            const int cat = cat_of_row(r0 + u);
                            tot[0] += cat == 0 ? cv[u] : 0u;
                            tot[1] += cat == 1 ? cv[u] : 0u;
                            tot[2] += cat == 2 ? cv[u] : 0u;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) bad |= !isfinite(__ldg(J.dcgm + (int64_t)j * J.ld + k));
                }
                cat_scales(tot, tf, rr);
                mask = 0x1FFFFu;
            } else {
                mask = 0x1FFFFu;
            }
            TPT_BEGIN(p_m);
            // the tile's chunk mask (OR over the 128 kernels), published for the MMA
            // thread before the tile's first chunk
            {
                const uint32_t wm = __reduce_or_sync(0xffffffffu, mask);
                if (lane == 0) misc[10 + 4 * sl + pw] = wm;
                // (also: every producer has finished tile t-1, whose stage buffer the
                // copy for tile t+1 reuses)
                bar_sync(1, kGroupT);
                mask = misc[10 + 4 * sl] | misc[11 + 4 * sl] | misc[12 + 4 * sl] | misc[13 + 4 * sl];
                if (ptid == 0) misc[sl] = mask;
                if (t + 1 < my_tiles) stage(t + 1);
            }
            // kernels with a non-finite feature: forward on the FMA pipe, into the
            // slot's spare TMEM columns (after the epilogue of tile t-2 read them);
            // runs before the tile's last chunk is handed to the MMA thread
            auto slow_block = [&]() {
                if (!__any_sync(0xffffffffu, bad)) return;
                if (t >= 2) mbar_wait(mb + MB_SLOWFREE + sl, (uint32_t)(((t >> 1) - 1) & 1));
                float out[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (bad) {
                    float x[DSO_FUSED_ROWS];
                    if (MODE == MODE_PRED) {
                        for (int c = 0; c < DSO_FUSED_ROWS; ++c) x[c] = J.fused[(int64_t)c * J.ld + k];
                    } else {
                        for (int j = 0; j < 8; ++j) x[j] = J.dcgm[(int64_t)j * J.ld + k];
                        for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
                            uint32_t cnt = 0;
                            if (MODE == MODE_DENSE) {
                                cnt = J.counts[(int64_t)r * J.ld + k];
                            } else {
                                for (int idx = 0; idx < E.cnt; ++idx) {
                                    const uint32_t en = J.entries[E.first + idx];
                                    if ((int)(en & 127u) == r) cnt += en >> 7;
                                }
                            }
                            x[8 + r] = norm_slot(cnt, r, tf, rr);
                        }
                    }
                    tc_forward_x(sm, x, out);
                    out[7] = 1.f;
                }
                tc::fence_after();
                tc::st8(tq + TSLOW + 8 * sl, out);
                tc::wait_st();
                tc::fence_before();
                const uint32_t bm = __ballot_sync(0xffffffffu, bad);
                if (lane == 0) misc[2 + 4 * sl + pw] = bm;
            };
            TPT_END(18, p_m);
            if (ptid == 0) TRACE(5, t);
            TPT_BEGIN(p_s);
            if (MODE == MODE_CSR) slow_block();
            TPT_END(19, p_s);
            TPT_END(14, p_t);
            // the next tile's entries into L2 while this tile's chunks are produced
            // (its row extent, loaded at this tile's start, has arrived by now)
            if (MODE == MODE_CSR && t + 1 < my_tiles && t0_of(t + 1) + row < J.n && NE.b > NE.a) {
                const uint32_t* ep = J.entries + (NE.a - J.ent_base);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ep));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ep + (NE.b - NE.a) - 1));
            }
            TPT_BEGIN(p_c);
            // ---- chunks -> ring ----------------------------------------------------
            auto hand_over = [&](int b) {  // the chunk in ring buffer b is complete
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mb_arrive(mb + MB_XFULL + b);
                ++g;
            };
            auto claim = [&]() {  // next ring buffer, once the MMAs reading it are done
                const int b = (int)(g % kRing);
                TPT_BEGIN(p_w);
                if (g >= kRing) mbar_wait(mb + MB_XEMPTY + b, ((g / kRing) - 1) & 1u);
                TPT_END(0, p_w);
                return b;
            };
            const int o = (row >> 3) * 64 + (row & 7) * 4;  // this kernel's core-matrix rows
            if (MODE == MODE_CSR) {
                // pass B: chunk c's entries are the next n_c common-category entries
                // (c = 1..3) or the next n_c others (c = 4..16) in row order: their
                // positions are popped off cbits / obits, four per step
                const float tf0 = tf[0], tf1 = tf[1], tf2 = tf[2], rr0 = rr[0], rr1 = rr[1],
                            rr2 = rr[2];
                const uint32_t buf_row = smem_u32(sm + S_RING) + 4u * (uint32_t)o;
                const uint8_t* offl = reinterpret_cast<const uint8_t*>(sm + S_OFFL);
                // global reads of an empty row go to entry 0 (some kernel of the tile has
                // entries whenever pass B runs, so the array is not empty)
                const uint64_t g_first = E.cnt > 0 ? E.first : 0;
                // rows of at most 32 entries in the whole warp: 32-bit position cursors
                const bool w64 = __any_sync(0xffffffffu, E.cnt > 32);
                // pass B, branch-free: positions beyond n_c read a valid word (position 0)
                // and their stores are predicated off
#ifndef DSO_TC_PBW
#define DSO_TC_PBW 4
#endif
                auto take = [&](auto stg, auto wide, uint64_t& rem, int n_c, int nmax, uint32_t bufa) {
                    constexpr int WD = DSO_TC_PBW;  // entries per step
#pragma unroll 1
                    for (int i0 = 0; i0 < nmax; i0 += WD) {
                        uint32_t en[WD];
                        bool on[WD];
#pragma unroll
                        for (int u = 0; u < WD; ++u) {
                            on[u] = i0 + u < n_c;
                            int e;
                            if constexpr (decltype(wide)::value) {
                                const uint32_t lo = (uint32_t)rem, hi = (uint32_t)(rem >> 32);
                                e = lo ? __ffs(lo) - 1 : 31 + __ffs(hi);
                                rem = on[u] ? rem & (rem - 1) : rem;
                            } else {
                                const uint32_t lo = (uint32_t)rem;
                                e = __ffs(lo) - 1;
                                rem = on[u] ? (uint64_t)(lo & (lo - 1u)) : rem;
                            }
                            e = on[u] ? e : 0;
                            if constexpr (decltype(stg)::value)
                                en[u] = s_row[e];
                            else
                                en[u] = __ldg(J.entries + g_first + e);
                        }
#pragma unroll
                        for (int u = 0; u < WD; ++u) {
                            const int slot = (int)(en[u] & 127u);
                            float t = tf0, r = rr0;
                            t = slot >= DSO_INSTR_SLOTS ? tf1 : t;
                            r = slot >= DSO_INSTR_SLOTS ? rr1 : r;
                            t = slot >= DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS ? tf2 : t;
                            r = slot >= DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS ? rr2 : r;
                            // count / total correctly rounded (totals < 2^24: the count
                            // converts exactly; Markstein correction of count * (1/total))
                            const float cf = __uint2float_rn(en[u] >> 7);
                            const float qq = __fmul_rn(cf, r);
                            const float f = fmaf(fmaf(-qq, t, cf), r, qq);
                            const float h = tc::tf32_hi_finite(f);
                            const uint32_t a4 = bufa + 4u * (uint32_t)offl[slot];
                            sts_pred(a4, h, on[u]);
                            sts_pred(a4 + 4u * TT * 8, f - h, on[u]);
                        }
                    }
                };
                auto take_any = [&](uint64_t& rem, int n_c, int nmax, uint32_t bufa) {
                    if (staged) {
                        if (w64) take(std::true_type{}, std::true_type{}, rem, n_c, nmax, bufa);
                        else take(std::true_type{}, std::false_type{}, rem, n_c, nmax, bufa);
                    } else {
                        if (w64) take(std::false_type{}, std::true_type{}, rem, n_c, nmax, bufa);
                        else take(std::false_type{}, std::false_type{}, rem, n_c, nmax, bufa);
                    }
                };
#pragma unroll 1
                for (uint32_t mrem = mask; mrem; mrem &= mrem - 1u) {
                    const int c = __ffs(mrem) - 1;
                    const int b = claim();
                    float* buf = sm + S_RING + b * kChunkF;
                    const int n_c = (c == 0 || uns) ? 0 : (int)((nib >> (4 * (c - 1))) & 15u);
                    const int nmax = __reduce_max_sync(0xffffffffu, n_c);
                    if (c == 0) {
                        put_chunk(buf, row, E.dg);
                    } else if (!uns) {
                        // zeros, then this chunk's entries in place
                        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
                        *reinterpret_cast<float4*>(buf + o) = z4;
                        *reinterpret_cast<float4*>(buf + o + 32) = z4;
                        *reinterpret_cast<float4*>(buf + TT * 8 + o) = z4;
                        *reinterpret_cast<float4*>(buf + TT * 8 + o + 32) = z4;
                        if (c < 4)
                            take_any(cbits, n_c, nmax, buf_row + 4u * b * kChunkF);
                        else
                            take_any(obits, n_c, nmax, buf_row + 4u * b * kChunkF);
                    } else {
                        // duplicate / unsorted / long rows: sum the counts per slot
                        uint32_t acc[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                        for (int idx = 0; idx < E.cnt; ++idx) {
                            const uint32_t en = __ldg(J.entries + E.first + idx);
                            const int slot = (int)(en & 127u);
                            if (slot >= DSO_COUNT_ROWS) continue;
                            const int col = 8 + pos_of[slot];
                            if ((col >> 3) == c)
#pragma unroll
                                for (int j = 0; j < 8; ++j) acc[j] += (col & 7) == j ? (en >> 7) : 0u;
                        }
                        float v[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int p = 8 * c + j - 8;
                            v[j] = (p < DSO_COUNT_ROWS) ? norm_slot(acc[j], slot_at[p], tf, rr) : 0.f;
                        }
                        put_chunk(buf, row, v);
                    }
                    TPT_BEGIN(p_p);
                    hand_over(b);
                    TPT_END(1, p_p);
                }
            } else {
                // predict / dense: chunk values loaded kAhead chunks in advance
                constexpr int kAhead = 4;
                float pf[kAhead][8];
                auto load_chunk = [&](int c, float (&v)[8]) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int col = 8 * c + j;
                        float x = 0.f;
                        if (k < J.n && col < DSO_FUSED_ROWS) {
                            const int sl8 = col < 8 ? col : 8 + slot_at[col - 8];  // feature row
                            if (MODE == MODE_PRED) {
                                x = __ldg(J.fused + (int64_t)sl8 * J.ld + k);
                            } else if (col < 8) {
                                x = __ldg(J.dcgm + (int64_t)col * J.ld + k);
                            } else {
                                const uint32_t cnt = __ldg(J.counts + (int64_t)(sl8 - 8) * J.ld + k);
                                x = norm_slot(cnt, sl8 - 8, tf, rr);
                            }
                        }
                        v[j] = x;
                    }
                };
#pragma unroll
                for (int a = 0; a < kAhead; ++a) load_chunk(a, pf[a]);
#pragma unroll
                for (int c = 0; c < 17; ++c) {
                    float v[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        v[j] = pf[c % kAhead][j];
                        bad |= !isfinite(v[j]);
                    }
                    if (c + kAhead < 17) load_chunk(c + kAhead, pf[c % kAhead]);
                    if (c == 16) slow_block();
                    const int b = claim();
                    put_chunk(sm + S_RING + b * kChunkF, row, v);
                    TPT_BEGIN(p_p);
                    hand_over(b);
                    TPT_END(1, p_p);
                }
            }
            TPT_END(15, p_c);
            if (ptid == 0) TRACE(7, t);
            if (MODE == MODE_CSR && t + 1 < my_tiles) tc_csr_take(J, t0_of(t + 1) + row, NE, E);
        }
    } else {
        // ============================ epilogue groups ============================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegEpi));
        const int grp = (warp >> 2) - EPI_WG0, q = warp & 3;
        const int row = 32 * q + lane;
        const uint32_t tq = tbase + ((uint32_t)(32 * q) << 16);
        const uint32_t S = tq + (uint32_t)(grp * SLOT_COLS);
        const float4* s_core = reinterpret_cast<const float4*>(sm + S_TABLES);
        const float2* s_mem = reinterpret_cast<const float2*>(sm + S_TABLES + 4 * J.nc);
        const float4* s_pair =
            J.pairs ? reinterpret_cast<const float4*>(sm + tc_pairs_offset(J.nc, J.nm)) : nullptr;
        // pipeline modes: clamped parameters of the tile's kernels -> grid sweep
        // (a sweep of the previous tile placed in this tile's layer-2 wait measured
        // slower: the producers, not the layer-2 hand-off, bound the engine)
        struct Pending {
            int64_t k;
            float pr[7];
            bool cl;
        } pend;
        auto sweep_out = [&](const Pending& P) {
            const KParams p{P.pr[0], P.pr[1], P.pr[2], P.pr[3], P.pr[4], P.pr[5], P.pr[6]};
#ifdef DSO_TCV_NOSWEEP
            const Best r{P.pr[0], P.pr[1], (int)(P.pr[2] > 1.f)};
#else
            const Best r = sweep_dispatch<DSO_TC_SWEEP_UNR>(p, s_core, s_mem, s_pair, J, 0, J.nc);
#endif
#pragma unroll
            for (int d = 0; d < 4; ++d) write_result(J, P.k, d, r, P.cl, P.pr, p, s_core, s_mem);
        };
        for (int64_t t = grp; t < my_tiles; t += 2) {
            const uint32_t ph = (uint32_t)((t >> 1) & 1);
            const int64_t k = t0_of(t) + row;
            TPT_BEGIN(e_w1);
            if (q == 0 && lane == 0) TRACE(8, t);
            wait_acq(mb + MB_D1F + grp, ph);
            TPT_END(2, e_w1);
            if (q == 0 && lane == 0) TRACE(9, t);
            TPT_BEGIN(e_1);
            {
                // batches of kEpi1Batch chunks: the batch's TMEM loads back to back, one
                // wait, activations split and stored as A2, one store wait, then the
                // batch's chunks are signalled (tcgen05 load / store latencies paid once
                // per batch instead of once per chunk)
#pragma unroll kEpi1Unroll
                for (int c0 = 0; c0 < 13; c0 += kEpi1Batch) {
                    float v[kEpi1Batch][8];
#pragma unroll
                    for (int u = 0; u < kEpi1Batch; ++u)
                        if (c0 + u < 13) tc::ld8(S + 8 * (c0 + u), v[u]);
                    tc::wait_ld_tie(v[0]);
#pragma unroll
                    for (int u = 1; u < kEpi1Batch; ++u) tc::tie8(v[u]);
#pragma unroll
                    for (int u = 0; u < kEpi1Batch; ++u)
                        if (c0 + u < 13)
                            epi_act_store<H1>(v[u], c0 + u, sm + NB1, S + 8 * (c0 + u),
                                              S + A2LO + 8 * (c0 + u));
                    tc::wait_st();
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0)
#pragma unroll
                        for (int u = 0; u < kEpi1Batch; ++u)
                            if (c0 + u < 13) mb_arrive(mb + MB_A2R + 13 * grp + c0 + u);
                }
            }
            TPT_END(3, e_1);
            if (q == 0 && lane == 0) TRACE(10, t);
            TPT_BEGIN(e_w2);
            wait_acq(mb + MB_D2F + grp, ph);
            TPT_END(4, e_w2);
            if (q == 0 && lane == 0) TRACE(11, t);
            TPT_BEGIN(e_2);
            // L2 outputs: sigmoid of D2 into registers; D2 is then free for the next tile
            float h2[56];
            {
                // all of D2 into registers with one wait, then D2 is released at once
                // (the next tile's layer 2 may start) and the activations follow
                float v[7][8];
#pragma unroll
                for (int c = 0; c < 7; ++c) tc::ld8(tq + TD2 + 8 * c, v[c]);
                tc::wait_ld_tie(v[0]);
#pragma unroll
                for (int c = 1; c < 7; ++c) tc::tie8(v[c]);
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mb_arrive(mb + MB_D2FREE);
                if (q == 0 && lane == 0) TRACE(12, t);
#pragma unroll
                for (int c = 0; c < 7; ++c)
#pragma unroll
                for (int j = 0; j < 8; ++j) h2[8 * c + j] = v[c][j];
            }
#pragma unroll
            for (int c = 0; c < 7; ++c) {
                float v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = h2[8 * c + j];
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                    const float2 z = ffma2(make_float2(v[j], v[j + 1]), make_float2(kNL2E, kNL2E),
                                           make_float2(sm[NB2 + 8 * c + j], sm[NB2 + 8 * c + j + 1]));
                    float e0, e1, r0, r1;
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(z.x));
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(z.y));
                    const float2 d = fadd2(make_float2(1.f, 1.f), make_float2(e0, e1));
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
                    h2[8 * c + j] = r0;
                    h2[8 * c + j + 1] = r1;
                }
            }
            TPT_END(5, e_2);
            TPT_BEGIN(e_3);
            // L3 (50 -> 25, sigmoid) and L4 (25 -> 7) on the FMA pipe, FP32, neuron
            // pairs per FFMA2, weights as shared-memory broadcasts
            float raw[8];
#ifdef DSO_TCV_NOL34
#pragma unroll
            for (int j = 0; j < 8; ++j) raw[j] = h2[j] * sm[S_STATS + 8 + (j & 7)] + h2[8 + j];
            if (false)
#endif
            {
                float2 a3[14];
#pragma unroll
                for (int u = 0; u < 14; ++u) a3[u] = make_float2(0.f, 0.f);
#pragma unroll kL3Unroll
                for (int kk = 0; kk < H2; ++kk) {
                    const float4* wr = reinterpret_cast<const float4*>(sm + W3T + kk * 28);
                    const float2 x2 = make_float2(h2[kk], h2[kk]);
#pragma unroll
                    for (int u = 0; u < 7; ++u) {
                        const float4 w4 = wr[u];
                        a3[2 * u] = ffma2(x2, make_float2(w4.x, w4.y), a3[2 * u]);
                        a3[2 * u + 1] = ffma2(x2, make_float2(w4.z, w4.w), a3[2 * u + 1]);
                    }
                }
                float h3[28];
#pragma unroll
                for (int u = 0; u < 14; ++u) {
                    const float2 z = ffma2(a3[u], make_float2(kNL2E, kNL2E),
                                           make_float2(sm[NB3 + 2 * u], sm[NB3 + 2 * u + 1]));
                    float e0, e1, r0, r1;
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(z.x));
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(z.y));
                    const float2 d = fadd2(make_float2(1.f, 1.f), make_float2(e0, e1));
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
                    h3[2 * u] = r0;
                    h3[2 * u + 1] = r1;
                }
                float2 a4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                make_float2(0.f, 0.f)};
#pragma unroll
                for (int kk = 0; kk < H3; ++kk) {
                    const float4* wr = reinterpret_cast<const float4*>(sm + W4T + kk * 8);
                    const float2 x2 = make_float2(h3[kk], h3[kk]);
                    const float4 w0 = wr[0], w1 = wr[1];
                    a4[0] = ffma2(x2, make_float2(w0.x, w0.y), a4[0]);
                    a4[1] = ffma2(x2, make_float2(w0.z, w0.w), a4[1]);
                    a4[2] = ffma2(x2, make_float2(w1.x, w1.y), a4[2]);
                    a4[3] = ffma2(x2, make_float2(w1.z, w1.w), a4[3]);
                }
                const float z4[8] = {a4[0].x, a4[0].y, a4[1].x, a4[1].y, a4[2].x, a4[2].y, a4[3].x, a4[3].y};
#pragma unroll
                for (int j = 0; j < 7; ++j)
                    raw[j] = fmaf(z4[j] + sm[B4 + j], sm[S_STATS + 8 + j], sm[S_STATS + j]);
            }
            TPT_END(7, e_3);
            if (q == 0 && lane == 0) TRACE(13, t);
            TPT_BEGIN(e_4);
            {
                const uint32_t bm = *reinterpret_cast<volatile uint32_t*>(misc + 2 + 4 * grp + q);
                if (bm) {  // kernels predicted on the FMA pipe by the producer
                    float w[8];
                    tc::ld8(tq + TSLOW + 8 * grp, w);
                    tc::wait_ld();
                    if ((bm >> lane) & 1u)
#pragma unroll
                        for (int j = 0; j < 7; ++j) raw[j] = w[j];
                    __syncwarp();
                    if (lane == 0) misc[2 + 4 * grp + q] = 0u;
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mb_arrive(mb + MB_SLOWFREE + grp);
            }
            if (MODE == MODE_PRED) {
                if (k < J.n) {
                    if (J.raw)
#pragma unroll
                        for (int j = 0; j < 7; ++j) J.raw[j * J.ld_out + k] = raw[j];
                    const bool cl = clamp_params(raw);
#pragma unroll
                    for (int j = 0; j < 7; ++j) J.params[j * J.ld_out + k] = raw[j];
                    if (J.clamped) J.clamped[k] = cl ? 1 : 0;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 7; ++j) pend.pr[j] = raw[j];
                pend.cl = clamp_params(pend.pr);
                pend.k = k;
                TPT_END(10, e_4);
                TPT_BEGIN(e_s);
                sweep_out(pend);
                TPT_END(9, e_s);
            }
            if (q == 0 && lane == 0) TRACE(14, t);
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == MMA_WARP) tc::tmem_dealloc<512>(tbase);
}

inline size_t tc_smem_bytes(int nc, int nm, bool pairs) {
    return pairs ? (size_t)(tc_pairs_offset(nc, nm) + 8 * ((nc + 1) / 2)) * sizeof(float)
                 : (size_t)(S_TABLES + 4 * nc + 2 * nm) * sizeof(float);
}

// Packed tc model from the reference-layout master (f32): hi/lo splits with
// the device's cvt.rna.tf32, padding zero, non-finite weights counted.
__global__ void tc_repack_kernel(const float* __restrict__ master, float* __restrict__ pk) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    auto put = [&](int hi, int lo, int n, int k, int K, float w) {
        const float h = tc::tf32_hi(w);
        pk[hi + cm(n, k, K)] = h;
        pk[lo + cm(n, k, K)] = isfinite(w) ? w - h : 0.f;
        if (!isfinite(w)) atomicAdd(reinterpret_cast<int*>(pk + FLAG), 1);
    };
    if (e < MW2) {
        const int c = e % 134;
        put(W1H, W1L, e / 134, c < 8 ? c : 8 + tc_pos(c - 8), K1, master[e]);
    } else if (e < MW3) {
        const int f = e - MW2;
        put(W2H, W2L, f / 100, f % 100, K2, master[e]);
    } else if (e < MW4) {
        const int f = e - MW3;
        pk[W3T + (f % 50) * 28 + f / 50] = master[e];
        if (!isfinite(master[e])) atomicAdd(reinterpret_cast<int*>(pk + FLAG), 1);
    } else if (e < MB1) {
        const int f = e - MW4;
        pk[W4T + (f % 25) * 8 + f / 25] = master[e];
        if (!isfinite(master[e])) atomicAdd(reinterpret_cast<int*>(pk + FLAG), 1);
    } else if (e < MB2) {
        pk[NB1 + e - MB1] = master[e] * kNL2E;
    } else if (e < MB3) {
        pk[NB2 + e - MB2] = master[e] * kNL2E;
    } else if (e < MB4) {
        pk[NB3 + e - MB3] = master[e] * kNL2E;
    } else if (e < kMasterFloats) {
        pk[B4 + e - MB4] = master[e];
    }
}

}  // namespace tce
