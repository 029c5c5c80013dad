// Forward, ping-pong tcgen05 kernel (moba_forward, src/attention.py:147-182;
// paper Alg. 1), key-block-major, for block sizes <= 128.
//
// Work item = (head, key block j, 128-row tile of block j's varlen slice);
// items are sorted by (head, block) and every persistent CTA takes a
// contiguous range, so consecutive items share K_j / V_j. An item record
// carries everything the roles need (block, tile start in the flat slice,
// row count), so no role walks a chain of dependent global loads per item.
//
//   S(i)  = Q_g K_j^T            SS-MMA  -> TMEM slot i&1 (fp32, BP columns)
//   P(i)  = exp2(S*scale*log2e - m)      -> bf16 pairs written back over the
//                                           first BP/2 columns of the slot
//   O(i)  = P V_j                TS-MMA  (A = P from TMEM, B = V in smem)
//                                        -> TMEM O buffer i&1
// Each query row of an item sees the whole (<= 128-key) block at once, so
// the softmax is single pass (SoftmaxState.update with one chunk,
// src/attention.py:60-68): row max, exp, sum, and the partial is stored
// normalised with its LSE; moba_combine merges a query's partials
// (SoftmaxState.finalize, src/attention.py:70-74).
//
// Warps (512 threads):
//   0      MMA issuer (one elected lane)
//   1-3    producers: coalesced cp.async gather of the item's 128 query rows
//          (8 lanes per 128-B row segment) plus their query ids into smem,
//          one item of index prefetch ahead; warp 1 lane 0 also loads
//          K_j / V_j with 3-D TMA (rows past the head's end are zero filled)
//   4-7    softmax for even items   (TMEM lane quadrant warp%4)
//   8-11   softmax for odd items
//   12-15  epilogue: O from TMEM -> normalised bf16 partial (TMA store) + LSE
// The two softmax warpgroups ping-pong: while one runs exp on item i, the
// tensor pipe computes S(i+1) / O(i-1) for the other. P never touches
// shared memory (the SS-MMA of P V would read 32 KB more per item through
// the smem port than the whole Q gather writes).
#include "common.cuh"
#include "sm100.cuh"
#include <cstdio>
#include <cstdlib>

namespace moba {
namespace fwdts {

constexpr int kM = 128;
constexpr int kThreads = 512;
constexpr int kMma = 0;
constexpr int kPr0 = 1, kPrN = 3;
constexpr int kSm0 = 4;       // softmax warps 4-11
constexpr int kEp0 = 12;      // epilogue warps 12-15
constexpr float kLn2 = 0.6931471805599453f;
constexpr uint32_t kStg = 32 * 128;    // per-warp O staging: 32 rows x one 64-column SW128 slab

struct Bars {
    uint64_t q_full[4], q_empty[4];
    uint64_t kv_full[3], kv_empty[3];
    uint64_t s_full[2], s_free[2], p_full[2], p_free[2], o_full[2], o_empty[2];
    uint32_t tmem;
};

// hj = head * n_blocks + j; fl = head-local flat position of the tile's
// first row (offsets[hj] + row0); rows = live rows of the tile (1..128)
struct __align__(16) Item {
    int32_t hj, fl, rows, pad;
};

template <int D>
struct Cfg {
    static constexpr int QS = (D == 64) ? 4 : 2;          // Q gather stages
    static constexpr uint32_t kQBytes = kM * D * 2;
    // d = 64: S, P and O each have their own TMEM columns, so S(i+2) can be
    // issued as soon as the softmax has read S(i) (before P(i) is consumed):
    //   S [0, 256)  P [256, 384)  O [384, 512)
    // d = 128: P aliases the first half of its S slot (S(i+2) waits for the
    // O MMA of item i):   S/P [0, 256)  O [256, 512)
    static constexpr bool kSplit = (D == 64);
    static constexpr int KVS = kSplit ? 3 : 2;             // K/V stages (S runs up to 2 items ahead)
    static constexpr uint32_t kPCol = kSplit ? 256 : 0;
    static constexpr uint32_t kPStride = kSplit ? 64 : 128;
    static constexpr uint32_t kOCol = kSplit ? 384 : 256;
};

MOBA_DEV void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// 3-D tiled store {c0, c1, c2} of an SW128 box from smem (bulk-group completion)
MOBA_DEV void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map),
                 "r"(c0), "r"(c1), "r"(c2), "r"(src)
                 : "memory");
}

MOBA_DEV Item load_item(const Item* p) {
    int4 v = __ldg(reinterpret_cast<const int4*>(p));
    return Item{v.x, v.y, v.z, v.w};
}

// NCH = ceil(BP / 32): 32-column chunks of S the softmax reads
template <int D, int NCH>
__global__ void __launch_bounds__(kThreads, 1)
moba_fwd_ts_kernel(const __nv_bfloat16* __restrict__ Q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, int64_t N, int B, int BP, int width, int kv_group, int slabs,
                   const int32_t* __restrict__ flat, const Item* __restrict__ items,
                   const int32_t* __restrict__ item_lo, const int32_t* __restrict__ item_hi, float scale_log2,
                   __nv_bfloat16* __restrict__ part_o, float* __restrict__ part_lse,
                   const __grid_constant__ CUtensorMap tm_po, long long* __restrict__ trace, int trace_cta) {
    using namespace sm100;
    using C = Cfg<D>;
    // debug timeline (MOBA_FWD_TRACE): CTA trace_cta (MOBA_FWD_TRACE_CTA,
    // default 0), lane 0 of the recording warp, its first 256 items
#ifdef MOBA_TIMELINE
#define TR(li, ev)                                                                          \
    do {                                                                                    \
        if (trace != nullptr && blockIdx.x == trace_cta && lane == 0 && (li) < 256)         \
            trace[(li) * 16 + (ev)] = clock64();                                            \
    } while (0)
#else
    // compiled out of the product build (make EXTRA=-DMOBA_TIMELINE for timelines)
    (void)trace;
    (void)trace_cta;
#define TR(li, ev) do { } while (0)
#endif
    constexpr int SL = D / 64;
    constexpr int QS = C::QS;
    constexpr int NC = NCH * 32;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t kv_bytes = (uint32_t)BP * D * 2;              // one of K / V
    const uint32_t oQ = 0, oKV = QS * C::kQBytes;
    const uint32_t oSTG = oKV + C::KVS * 2 * kv_bytes;           // [4 epilogue warps][32 rows][128 B] O staging
    const uint32_t oID = oSTG + 4 * kStg;                        // [QS][128] query ids
    const uint32_t oST = oID + QS * kM * 4;                      // [4][128] (1/l, lse) per row
    Bars* bars = reinterpret_cast<Bars*>(smem + oST + 4 * kM * 8);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_blocks = (int)((N + B - 1) / B);
    const int lo = *item_lo;
    const int n_items = *item_hi - lo;
    const int per = (n_items + gridDim.x - 1) / gridDim.x;
    const int it0 = min(n_items, (int)blockIdx.x * per);
    const int n_local = min(n_items, it0 + per) - it0;
    const Item* my_items = items + lo + it0;

    if (warp == kMma) tmem_alloc(&bars->tmem, 512);
    if (tid == 0) {
        for (int s = 0; s < QS; ++s) {
            mbar_init(&bars->q_full[s], 2 * 32 * kPrN);     // cp.async (noinc) + plain arrival per producer lane
            mbar_init(&bars->q_empty[s], 1 + 4);            // S MMA commit + the 4 softmax warps (ids read)
        }
        for (int s = 0; s < C::KVS; ++s) {
            mbar_init(&bars->kv_full[s], 1);
            mbar_init(&bars->kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars->s_full[s], 1);
            mbar_init(&bars->s_free[s], 4);
            mbar_init(&bars->p_free[s], 1);
            mbar_init(&bars->p_full[s], 4);
            mbar_init(&bars->o_full[s], 1);
            mbar_init(&bars->o_empty[s], 4);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    // register budget (setmaxnreg per warpgroup, executed before the roles
    // diverge): 128 x 104 (MMA + producers) + 256 x 168 (softmax) + 128 x 72
    // (epilogue) = 64K
    auto run_producer = [&]() {
            // ------------------------------------------------------------ producers
            const int pw = warp - kPr0;
            const int sub = lane & 7, rsub = lane >> 3;
            constexpr int NI = (kM / 4 + kPrN - 1) / kPrN;    // 4-row groups per warp
            int prev_hj = -1, kv_uses = -1;
            // rows of this lane: r_i = 4 * (pw + kPrN * i) + rsub; the id of
            // row r_i is written by the sub == 0 lane
            auto load_ids = [&](const Item& it, int (&qr)[NI]) {
                const int32_t* fl = flat + (int64_t)(it.hj / n_blocks) * N * width + it.fl;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int r = 4 * (pw + kPrN * i) + rsub;
                    qr[i] = (r < it.rows) ? __ldg(fl + r) : -1;
                }
            };
            Item cur = load_item(my_items);
            int qrow[NI];
            load_ids(cur, qrow);
            for (int li = 0; li < n_local; ++li) {
                const Item nxt = (li + 1 < n_local) ? load_item(my_items + li + 1) : cur;
                const int64_t h = cur.hj / n_blocks;
                const int j = cur.hj - (int)h * n_blocks;
                const int kvkey = cur.hj * slabs + cur.pad;          // (block, 128-key slab)
                const int krow = j * B + cur.pad * kM;
                if (kvkey != prev_hj) {
                    prev_hj = kvkey;
                    ++kv_uses;
                    if (pw == 0 && lane == 0) {
                        const int ks = kv_uses % C::KVS;
                        mbar_wait(&bars->kv_empty[ks], ((kv_uses / C::KVS) & 1) ^ 1);
                        mbar_expect_tx(&bars->kv_full[ks], 2 * kv_bytes);
                        const uint32_t kb = sbase + oKV + ks * 2 * kv_bytes;
#pragma unroll
                        for (int sl = 0; sl < SL; ++sl) {
                            // GQA: query head h reads K/V head h / kv_group
                            const int hk = (int)(h / kv_group);
                            tma_load_3d(kb + sl * BP * 128, &tm_k, sl * 64, krow, hk, &bars->kv_full[ks]);
                            tma_load_3d(kb + kv_bytes + sl * BP * 128, &tm_v, sl * 64, krow, hk,
                                        &bars->kv_full[ks]);
                        }
                    }
                }
                const int qs = li % QS;
                const __nv_bfloat16* Qh = Q + h * N * D;
                if (pw == 0) TR(li, 4);
                mbar_wait(&bars->q_empty[qs], ((li / QS) & 1) ^ 1);
                if (pw == 0) TR(li, 5);
                const uint32_t qb = sbase + oQ + qs * C::kQBytes;
                const uint32_t ib = sbase + oID + qs * kM * 4;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int r = 4 * (pw + kPrN * i) + rsub;
                    if (r < kM) {
                        const int q = qrow[i];
                        const __nv_bfloat16* src = Qh + (int64_t)max(q, 0) * D + sub * 8;
                        const uint32_t dst = qb + r * 128 + ((sub ^ (r & 7)) << 4);
#pragma unroll
                        for (int sl = 0; sl < SL; ++sl) cp_async16(dst + sl * kM * 128, src + sl * 64, q >= 0);
                        if (sub == 0) sts32(ib + r * 4, (uint32_t)q);
                    }
                }
                cpasync_arrive_noinc(&bars->q_full[qs]);
                mbar_arrive(&bars->q_full[qs]);
                if (pw == 0) TR(li, 6);
                if (li + 1 < n_local) load_ids(nxt, qrow);
                if (pw == 0) TR(li, 15);
                cur = nxt;
            }
    };

    if (warp < kSm0) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
        if (n_local > 0 && warp == kMma) {
            // ------------------------------------------------------------ MMA issuer
            // warp-uniform: every lane runs the loop, one elected lane issues;
            // descriptors advance by constants (start address field, 16 B units)
            const uint32_t idesc_s = idesc_bf16(kM, BP, false, false);
            const uint32_t idesc_o = idesc_bf16(kM, D, false, true);
            int s_hj = -1, s_kv = -1;
            int kv_of[4] = {0, 0, 0, 0};
            // block ids of items li, li+1, li+2 (loaded two issues ahead)
            auto kvkey = [&](int li) { return my_items[li].hj * slabs + my_items[li].pad; };
            int hj0 = kvkey(0);
            int hj1 = n_local > 1 ? kvkey(1) : -1;
            int hj2 = n_local > 2 ? kvkey(2) : -1;
            auto issue_s = [&](int li) {
                const int hj = hj0;
                const bool last = hj1 != hj;
                hj0 = hj1;
                hj1 = hj2;
                hj2 = (li + 3 < n_local) ? kvkey(li + 3) : -1;
                if (hj != s_hj) {
                    s_hj = hj;
                    ++s_kv;
                    mbar_wait(&bars->kv_full[s_kv % C::KVS], (s_kv / C::KVS) & 1);
                }
                kv_of[li & 3] = s_kv | (last ? (1 << 30) : 0);   // bit 30: last use of the K/V buffer
                const int qs = li % QS;
                TR(li, 0);
                mbar_wait(&bars->q_full[qs], (li / QS) & 1);
                TR(li, 1);
                tc_fence_after();
                fence_proxy_async_smem();
                const uint64_t dq = desc_kmajor(sbase + oQ + qs * C::kQBytes, 0);
                const uint64_t dk = desc_kmajor(sbase + oKV + (s_kv % C::KVS) * 2 * kv_bytes, 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const int sl = kk >> 2, ke = kk & 3;
                    umma_bf16_w(tmem + (li & 1) * 128, dq + (uint64_t)(sl * (kM * 128 >> 4) + ke * 2),
                                dk + (uint64_t)(sl * (BP * 128 >> 4) + ke * 2), idesc_s, kk > 0);
                }
                umma_commit_w(&bars->s_full[li & 1]);
                umma_commit_w(&bars->q_empty[qs]);
                TR(li, 13);
            };
            // inputs of S(li+2) (slot free, its K/V block and query tile
            // landed) — probed without blocking
            auto s_ready = [&](int li2) {
                const int b2 = li2 & 1;
                if (!mbar_test_wait(&bars->s_free[b2], ((li2 >> 1) - 1) & 1)) return false;
                if (hj0 != s_hj) {
                    const int nk = s_kv + 1;
                    if (!mbar_test_wait(&bars->kv_full[nk % C::KVS], (nk / C::KVS) & 1)) return false;
                }
                return mbar_test_wait(&bars->q_full[li2 % QS], (li2 / QS) & 1);
            };
            auto issue_pv = [&](int li) {
                const int b = li & 1;
                const int kvu = kv_of[li & 3] & ~(1 << 30);
                const bool last_use = (kv_of[li & 3] >> 30) & 1;
                TR(li, 3);
                tc_fence_after();
                const uint64_t dv = desc_mnmajor(sbase + oKV + (kvu % C::KVS) * 2 * kv_bytes + kv_bytes, 0, BP * 128);
                const uint32_t ta = tmem + C::kPCol + b * C::kPStride;
                for (int kk = 0; kk < BP / 16; ++kk)
                    umma_bf16_ts_w(tmem + C::kOCol + b * D, ta + 8 * kk, dv + (uint64_t)(kk * 128), idesc_o, kk > 0);
                umma_commit_w(&bars->o_full[b]);
                umma_commit_w(&bars->p_free[b]);
                if (last_use) umma_commit_w(&bars->kv_empty[kvu % C::KVS]);
                TR(li, 12);
            };
            issue_s(0);
            if (n_local > 1) issue_s(1);
            for (int li = 0; li < n_local; ++li) {
                const int b = li & 1;
                TR(li, 2);
                if (C::kSplit && NCH <= 2) {
                    // d = 64, blocks of <= 64 keys: S(li+2) (slot b) and
                    // O(li) = P(li) V (P / O columns) touch different TMEM, so
                    // they are issued in the order their inputs arrive: a late
                    // query gather no longer holds back the P.V of a finished
                    // softmax (C3, B = 64: fwd 0.75 -> 0.67 ms; with 128-key
                    // blocks the fixed order below is 1.5% faster)
                    bool s_pending = li + 2 < n_local, pv_pending = true;
                    while (s_pending || pv_pending) {
                        bool progress = false;
                        if (pv_pending && mbar_test_wait(&bars->p_full[b], (li >> 1) & 1) &&
                            mbar_test_wait(&bars->o_empty[b], ((li >> 1) & 1) ^ 1)) {
                            issue_pv(li);
                            pv_pending = false;
                            progress = true;
                        }
                        if (s_pending && s_ready(li + 2)) {
                            issue_s(li + 2);
                            s_pending = false;
                            progress = true;
                        }
                        // nothing ready: park briefly on the softmax's P
                        // (the usual next event) instead of spinning on the
                        // issue slots this warp shares with a softmax warp
                        if (!progress && pv_pending) mbar_try_wait_hint(&bars->p_full[b], (li >> 1) & 1, 256u);
                    }
                } else if (C::kSplit) {
                    if (li + 2 < n_local) {
                        // S(li+2) goes into slot b once the softmax has read S(li)
                        mbar_wait(&bars->s_free[b], (li >> 1) & 1);
                        issue_s(li + 2);
                    }
                    mbar_wait(&bars->p_full[b], (li >> 1) & 1);
                    mbar_wait(&bars->o_empty[b], ((li >> 1) & 1) ^ 1);
                    issue_pv(li);
                } else {
                    mbar_wait(&bars->p_full[b], (li >> 1) & 1);
                    mbar_wait(&bars->o_empty[b], ((li >> 1) & 1) ^ 1);
                    issue_pv(li);
                    // d = 128: S(li+2) reuses slot b, whose P(li) has been consumed
                    // by the O MMA issued above (tcgen05.mma executes in issue order)
                    if (li + 2 < n_local) issue_s(li + 2);
                }
            }
        } else if (n_local > 0) {
            run_producer();
        }
    } else if (warp < kEp0) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
        if (n_local > 0) {
            // ------------------------------------------------------------ softmax
            // a thread holds its whole S row (setmaxnreg gives these two
            // warpgroups 168 registers, taken from the producer/MMA and
            // epilogue warpgroups)
            const int wg = (warp - kSm0) >> 2;            // 0: even items, 1: odd items
            const int quad = warp & 3;
            const int row = 32 * quad + lane;
            const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
            const uint32_t slot = tmem + wg * 128 + lane_off;
            const uint32_t pslot = tmem + C::kPCol + wg * C::kPStride + lane_off;
            Item nxt = load_item(my_items + min(wg, n_local - 1));
            for (int li = wg; li < n_local; li += 2) {
                const Item cur = nxt;
                if (li + 2 < n_local) nxt = load_item(my_items + li + 2);
                const int64_t h = cur.hj / n_blocks;
                const int64_t k0 = (int64_t)(cur.hj - (int)h * n_blocks) * B + (int64_t)cur.pad * kM;   // slab start
                const int64_t slab_len = min64(min64((int64_t)B - (int64_t)cur.pad * kM, (int64_t)kM), N - k0);
                const bool live = row < cur.rows;
                const int qs = li % QS;
                if (quad == 0) TR(li, 7);
                mbar_wait(&bars->s_full[wg], (li >> 1) & 1);
                if (quad == 0) TR(li, 8);
                tc_fence_after();
                const int q = lds32i(sbase + oID + qs * kM * 4 + row * 4);
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->q_empty[qs]);
                // visible keys of this row: columns [0, lim); columns
                // [lim, NC) are masked (past the block end, token-causal in
                // the own block, or never written by the MMA)
                const int lim = live ? (int)max64(0, min64(slab_len, (int64_t)q - k0 + 1)) : 0;
                const bool masked = lim < NC;
                float sv[NC];
#pragma unroll
                for (int c = 0; c < NCH; ++c) tmem_ld32(slot + c * 32, *reinterpret_cast<float(*)[32]>(&sv[c * 32]));
                tmem_ld_wait();
                if (C::kSplit) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->s_free[wg]);
                }
                if (masked) {
#pragma unroll
                    for (int c = 0; c < NC; ++c) sv[c] = (c < lim) ? sv[c] : -INFINITY;
                }
                float mx[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) mx[u] = sv[u];
#pragma unroll
                for (int c = 8; c < NC; ++c) mx[c & 7] = fmaxf(mx[c & 7], sv[c]);
                const float m = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                      fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
                const float msl = (m == -INFINITY) ? 0.f : m * scale_log2;
                // P slot b is free once the O MMA of item li - 2 has run
                if (C::kSplit && li >= 2) {
                    mbar_wait(&bars->p_free[wg], ((li >> 1) - 1) & 1);
                    tc_fence_after();
                }
                // x*scale - m and the row sum in packed fp32x2 (FFMA2 / FADD2).
                // Per 32-column chunk all shifts, then all 32 exponentials,
                // then sums / packing: the MUFU ops are independent and back
                // to back (the softmax is latency-bound, not MUFU-bound).
                float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    float* t = &sv[c * 32];
#pragma unroll
                    for (int i = 0; i < 32; i += 2) ffma2(t[i], t[i + 1], t[i], t[i + 1], scale_log2, scale_log2, -msl, -msl);
#pragma unroll
                    for (int i = 0; i < 32; ++i) t[i] = fast_exp2(t[i]);
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const int a = (i >> 1) & 2;
                        fadd2(ls[a], ls[a + 1], ls[a], ls[a + 1], t[i], t[i + 1]);
                        fadd2(ls[a], ls[a + 1], ls[a], ls[a + 1], t[i + 2], t[i + 3]);
                        pk[i >> 1] = pack_bf16(t[i], t[i + 1]);
                        pk[(i >> 1) + 1] = pack_bf16(t[i + 2], t[i + 3]);
                    }
                    tmem_st16(pslot + c * 16, pk);
                }
                const float l = (ls[0] + ls[1]) + (ls[2] + ls[3]);
                // row statistics for the epilogue warps (slot li & 3: the
                // epilogue of li has read them before S(li + 4) can exist)
                {
                    const uint32_t st = sbase + oST + ((li & 3) * kM + row) * 8;
                    asm volatile("st.shared.v2.f32 [%0], {%1, %2};\n" ::"r"(st), "f"(l > 0.f ? 1.f / l : 0.f),
                                 "f"(l > 0.f ? (msl + __log2f(l)) * kLn2 : -INFINITY)
                                 : "memory");
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full[wg]);
                if (quad == 0) TR(li, 9);
            }
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::: "memory");
        if (n_local > 0) {
            // ------------------------------------------------------------ epilogue
            // normalised partial O (bf16) and its LSE. A warp whose 32 rows
            // are all live stages them in SW128 smem and writes 4 KB per slab
            // with one TMA store (the rows are contiguous flat positions); the
            // tail warp of a block's last tile stores its live rows directly.
            const int quad = warp & 3;
            const int row = 32 * quad + lane;
            const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
            const uint32_t stg = sbase + oSTG + quad * kStg;
            Item nxt = load_item(my_items);
            for (int li = 0; li < n_local; ++li) {
                const Item cur = nxt;
                if (li + 1 < n_local) nxt = load_item(my_items + li + 1);
                const int b = li & 1;
                // partial of (flat position p, slab) at p * slabs + slab
                const int64_t pb = ((int64_t)(cur.hj / n_blocks) * N * width + cur.fl + row) * slabs + cur.pad;
                const bool live = row < cur.rows;
                const bool full_warp = 32 * quad + 32 <= cur.rows;
                const uint32_t obuf = tmem + C::kOCol + b * D + lane_off;
                mbar_wait(&bars->o_full[b], (li >> 1) & 1);
                if (quad == 0) TR(li, 10);
                tc_fence_after();
                float st0, st1;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n"
                             : "=f"(st0), "=f"(st1)
                             : "r"(sbase + oST + ((li & 3) * kM + row) * 8));
                const float inv = st0;
                if (live) part_lse[pb] = st1;
#pragma unroll
                for (int sl = 0; sl < SL; ++sl) {
                    if (full_warp) {
                        if (lane == 0) bulk_wait_read0();            // previous store has read the staging slab
                        __syncwarp();
                    }
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        float ov[32];
                        tmem_ld32(obuf + sl * 64 + hh * 32, ov);
                        tmem_ld_wait();
                        if (sl == SL - 1 && hh == 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&bars->o_empty[b]);
                        }
                        uint4 pk[4];
#pragma unroll
                        for (int g = 0; g < 4; ++g)
                            pk[g] = make_uint4(pack_bf16(ov[8 * g] * inv, ov[8 * g + 1] * inv),
                                               pack_bf16(ov[8 * g + 2] * inv, ov[8 * g + 3] * inv),
                                               pack_bf16(ov[8 * g + 4] * inv, ov[8 * g + 5] * inv),
                                               pack_bf16(ov[8 * g + 6] * inv, ov[8 * g + 7] * inv));
                        if (full_warp) {
#pragma unroll
                            for (int g = 0; g < 4; ++g)
                                sts128(stg + lane * 128 + (((hh * 4 + g) ^ (lane & 7)) << 4), pk[g]);
                        } else if (live) {
                            __nv_bfloat16* po = part_o + pb * D + sl * 64 + hh * 32;
#pragma unroll
                            for (int g = 0; g < 4; ++g) *reinterpret_cast<uint4*>(po + g * 8) = pk[g];
                        }
                    }
                    if (quad == 0 && sl == 0) TR(li, 14);
                    if (full_warp) {
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_3d(&tm_po, stg, sl * 64, cur.pad, (int)((pb - cur.pad) / slabs - lane));
                            bulk_commit();
                        }
                    }
                }
                if (quad == 0) TR(li, 11);
            }
            if (lane == 0) bulk_wait0();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMma) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// one thread per (head, block): its tiles' item records, at item_off[hj]
__global__ void fwd_ts_items_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                                    const int32_t* __restrict__ item_off, int64_t total, int slabs,
                                    Item* __restrict__ items) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= total) return;
    const int cnt = counts[b], off = offsets[b];
    Item* dst = items + item_off[b];
    const int tiles = (cnt + kM - 1) / kM;
    for (int sl = 0; sl < slabs; ++sl)
        for (int t = 0; t < tiles; ++t) dst[sl * tiles + t] = Item{(int32_t)b, off + t * kM, min(kM, cnt - t * kM), sl};
}

}  // namespace fwdts

bool make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t heads, uint64_t rows, uint32_t cols,
                       uint32_t box_rows);
bool make_tmap_bf16_3d_box(CUtensorMap* map, const void* base, uint64_t outer, uint64_t mid, uint32_t cols,
                           uint32_t box_mid, uint32_t box_outer);

size_t fwd_ts_item_bytes() { return sizeof(fwdts::Item); }

// item records for every (head, block): item_off = exclusive scan of the
// per-(head, block) counts of 128-row tiles
void fwd_ts_fill_items(const int32_t* counts, const int32_t* offsets, const int32_t* item_off, int64_t total,
                       int slabs, void* items, cudaStream_t s) {
    fwdts::fwd_ts_items_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, s>>>(counts, offsets, item_off, total, slabs,
                                                                             (fwdts::Item*)items);
}

// d in {64, 128}, ceil16(B) <= 128; runs the items [*item_lo, *item_hi)
// (device values) — a contiguous range of heads.
template <int D>
int launch_fwd_ts(const void* q, const void* k, const void* v, int64_t bh, int kv_group, int64_t N, int B, int width,
                  const int32_t* flat, const void* items, const int32_t* item_lo, const int32_t* item_hi,
                  float scale_log2, void* part_o, float* part_lse, cudaStream_t s) {
    using namespace fwdts;
    const int slabs = (int)ceil_div(B, kM);          // keys of a block in slabs of <= 128
    const int BP = (int)ceil_div(std::min(B, kM), 16) * 16;
    CUtensorMap tm_k, tm_v;
    if (!make_tmap_bf16_3d(&tm_k, k, (uint64_t)(bh / kv_group), (uint64_t)N, D, BP) ||
        !make_tmap_bf16_3d(&tm_v, v, (uint64_t)(bh / kv_group), (uint64_t)N, D, BP))
        return MOBA_ERR_CUDA;
    CUtensorMap tm_po;
    // partials [bh * N * width][slabs][D]: 3-D map, box {64, 1 slab, 32 positions}
    if (!make_tmap_bf16_3d_box(&tm_po, part_o, (uint64_t)(bh * N * width), (uint64_t)slabs, D, 1, 32))
        return MOBA_ERR_CUDA;
    const size_t smem = 1024 + (size_t)Cfg<D>::QS * (Cfg<D>::kQBytes + kM * 4) + 2 * Cfg<D>::KVS * (size_t)BP * D * 2 + 4 * kStg +
                        4 * kM * 8 + sizeof(Bars);
    if (smem > 232448) return MOBA_ERR_UNSUPPORTED;
    const int nch = (BP + 31) / 32;
    auto kern = nch == 1 ? moba_fwd_ts_kernel<D, 1>
              : nch == 2 ? moba_fwd_ts_kernel<D, 2>
              : nch == 3 ? moba_fwd_ts_kernel<D, 3>
                         : moba_fwd_ts_kernel<D, 4>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = kNumSMs;
    static long long* trace = nullptr;
    const char* trace_path = std::getenv("MOBA_FWD_TRACE");
    if (trace_path != nullptr && trace == nullptr) cudaMalloc(&trace, 256 * 16 * sizeof(long long));
    if (trace_path != nullptr) cudaMemsetAsync(trace, 0, 256 * 16 * sizeof(long long), s);
    {
        StageTimer tm(T_FWD, s);
        kern<<<grid, kThreads, smem, s>>>((const __nv_bfloat16*)q, tm_k, tm_v, N, B, BP, width, kv_group, slabs, flat,
                                          (const Item*)items, item_lo, item_hi, scale_log2, (__nv_bfloat16*)part_o,
                                          part_lse, tm_po, trace_path != nullptr ? trace : nullptr,
                                          std::getenv("MOBA_FWD_TRACE_CTA") ? std::atoi(std::getenv("MOBA_FWD_TRACE_CTA")) : 0);
    }
    int st = check_launch("moba_fwd_ts_kernel");
    if (st == 0 && trace_path != nullptr) {
        static long long host[256 * 16];
        cudaMemcpyAsync(host, trace, sizeof(host), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (FILE* f = std::fopen(trace_path, "wb")) {
            std::fwrite(host, sizeof(host), 1, f);
            std::fclose(f);
        }
    }
    return st;
}

template int launch_fwd_ts<64>(const void*, const void*, const void*, int64_t, int, int64_t, int, int,
                               const int32_t*, const void*, const int32_t*, const int32_t*, float, void*, float*,
                               cudaStream_t);
template int launch_fwd_ts<128>(const void*, const void*, const void*, int64_t, int, int64_t, int, int,
                                const int32_t*, const void*, const int32_t*, const int32_t*, float, void*, float*,
                                cudaStream_t);

}  // namespace moba
