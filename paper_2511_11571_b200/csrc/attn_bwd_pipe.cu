// Backward, pipelined tcgen05 kernel for d = 64 (moba_backward,
// src/attention.py:239-302; Alg. 5 per key block, src/attention.py:185-236).
//
// Work item = (head, key block j, 128-key slab). Items are handed out by an
// atomic counter in block-major order (block 0 of every head first): early
// blocks are selected by the most queries, so this is close to longest-first
// and the persistent CTAs finish together.
//
// Per 128-query tile g of an item's varlen slice (gathered rows):
//   S^T(g)  = K Q^T          -> TMEM slot g&1         (issued one tile ahead)
//   phase A : P^T = exp2(S^T*scale*log2e - L)  -> bf16 pairs in slot[0:64)
//   dP^T(g) = V dO^T         -> TMEM Y
//   phase B : dS^T = P^T (dP^T - D) (fp32 P)   -> bf16 pairs in Y[0:64) and
//                                                 an SW128 smem tile (A of dQ)
//   dV += P^T dO, dK += dS^T Q  (TS-MMAs, TMEM accumulators over the item)
//   dQ(g)   = dS K           -> slot[64:128), drained by the epilogue warps
//             with one 256-B bulk fp32 reduce-add per row
// S^T(g+1) runs on the tensor pipe while the softmax warps do phase A of g;
// dP^T(g+1) is issued right behind the dV/dK/dQ MMAs of g (tcgen05.mma
// executes in issue order, so Y and the slots are reused without waits).
//
// TMEM (512 columns): slot0 [0,128) slot1 [128,256) Y [256,384)
//                     dV [384,448) dK [448,512)
// Warps: 0-2 gather producers (warp 0 lane 0 also fetches items and loads
// K/V by TMA), 3 MMA issuer, 4-11 softmax (pairs share a TMEM lane quadrant
// and split the 128 query columns), 12-15 epilogue (dQ per tile, dK/dV per
// item).
#include "common.cuh"
#include "sm100.cuh"
#include <cstdio>
#include <cstdlib>

namespace moba {
namespace bwdp {

constexpr int D = 64;
constexpr int KT = 128;                 // keys per item
constexpr int MQ = 128;                 // gathered queries per tile
constexpr int kPr = 3;                  // producer warps
constexpr int kMma = 3;                 // MMA warp
constexpr int kSm0 = 4, kSmN = 8;       // softmax warps
constexpr int kEp0 = 12, kEpN = 4;      // epilogue warps (16 warps: 128 registers per thread)
constexpr int kThreads = 32 * (kEp0 + kEpN);
constexpr int kQSt = 3;                 // Q/dO stages
constexpr int kRing = 8;                // item ring depth
constexpr int kRingConsumers = (kPr - 1) + 1 + kSmN + kEpN;
constexpr uint32_t kTile = 128 * 64 * 2;     // one 128 x 64 bf16 SW128 tile (16 KB)
constexpr uint32_t cS0 = 0, cY = 256, cDV = 384, cDK = 448;
constexpr uint32_t kStgRow = 64 * 4 + 16;    // full-row dQ staging (fp32) + pad
constexpr uint32_t kStgRows = 16;            // staged rows per epilogue warp (two rounds of 16 lanes)
constexpr float kLog2e = 1.4426950408889634f;

struct Bars {
    uint64_t ring_full[kRing], ring_empty[kRing];
    uint64_t kv_full[2], kv_empty[2];
    uint64_t qd_full[kQSt], qd_empty[kQSt];
    uint64_t s_full[2], pa_full[2], dp_full, p_full;
    uint64_t dq_full[2], dq_empty[2];
    uint64_t dkv_full, dkv_empty;
    int ring[kRing];
    uint32_t tmem;
};

// smem layout (offsets from the 1 KB aligned base)
constexpr uint32_t oKV = 0;                                  // [2][K | V]
constexpr uint32_t oQD = oKV + 2 * 2 * kTile;                // [kQSt][Q | dO]
constexpr uint32_t oDS = oQD + kQSt * 2 * kTile;             // dS^T [2 query slabs][128 keys][128 B]
constexpr uint32_t oLDI = oDS + 2 * kTile;                   // [kQSt][L | D | id] x 128 x 4 B
constexpr uint32_t oSTG = oLDI + kQSt * 3 * MQ * 4;          // dQ staging kEpN x kStgRows x kStgRow
constexpr uint32_t oBAR = oSTG + kEpN * kStgRows * kStgRow;
constexpr uint32_t kSmem = 1024 + oBAR + sizeof(Bars);

struct Item {
    int64_t h;
    int j, slab, cnt, n_tiles, klen;
    int64_t kb0, fl_base;   // first key row (head-local), head-local flat base of the slice
};

// Items run in groups of `hg` heads (the group's fp32 dQ rows fit in L2, so
// the dQ reductions stay on chip when N is large), block-major inside a
// group: block 0 of every head of the group first (early blocks are selected
// by the most queries, so this is close to longest-first).
MOBA_DEV Item decode(int it, int64_t bh, int hg, int n_blocks, int slabs, int B, int64_t N, int width,
                     const int32_t* counts, const int32_t* offsets) {
    Item x;
    const int per_group = hg * n_blocks * slabs;
    const int g = it / per_group;
    const int r = it - g * per_group;
    const int h0 = g * hg;
    const int hn = (int)min64(hg, bh - h0);
    const int per_j = hn * slabs;
    x.j = r / per_j;
    const int rem = r % per_j;
    x.h = h0 + rem / slabs;
    x.slab = rem % slabs;
    const int64_t hj = x.h * n_blocks + x.j;
    x.cnt = counts[hj];
    x.n_tiles = (x.cnt + MQ - 1) / MQ;
    x.kb0 = (int64_t)x.j * B + x.slab * KT;
    x.klen = (int)max64(0, min64(min64(KT, (int64_t)B - x.slab * KT), N - x.kb0));
    x.fl_base = x.h * N * width + offsets[hj];
    return x;
}

// consumer side of the item ring: every consuming warp reads each entry once
struct RingReader {
    int s = 0;
    MOBA_DEV int next(Bars* bars, int lane) {
        const int slot = s % kRing;
        sm100::mbar_wait(&bars->ring_full[slot], (s / kRing) & 1);
        const int it = *reinterpret_cast<volatile int*>(&bars->ring[slot]);
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&bars->ring_empty[slot]);
        ++s;
        return it;
    }
};

__global__ void __launch_bounds__(kThreads, 1)
moba_bwd_pipe_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ dO,
                     const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const float* __restrict__ lse, const float* __restrict__ Dd, int64_t bh, int hg, int kv_group, int64_t N,
                     int B, int width, const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                     const int32_t* __restrict__ flat, float scale, int n_items, int* __restrict__ sched,
                     float* __restrict__ dq_acc, float* __restrict__ dq_part, int64_t part_stride,
                     __nv_bfloat16* __restrict__ dK, __nv_bfloat16* __restrict__ dV, long long* __restrict__ trace,
                     int trace_g0) {
    using namespace sm100;
    // debug timeline (MOBA_BWD_TRACE): CTA 0, lane 0 of the recording warp,
    // tiles [trace_g0, trace_g0 + 256) of the CTA (MOBA_BWD_TRACE_G0)
#ifdef MOBA_TIMELINE
#define TRB(g, ev)                                                                          \
    do {                                                                                    \
        if (trace != nullptr && blockIdx.x == 0 && lane == 0 && (unsigned)((g) - trace_g0) < 256u) \
            trace[((g) - trace_g0) * 16 + (ev)] = clock64();                                \
    } while (0)
#else
    // compiled out of the product build (the recording branches cost 2-4%;
    // make EXTRA=-DMOBA_TIMELINE for timelines)
    (void)trace;
    (void)trace_g0;
#define TRB(g, ev) do { } while (0)
#endif
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    Bars* bars = reinterpret_cast<Bars*>(smem + oBAR);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_blocks = (int)((N + B - 1) / B);
    const int slabs = (B + KT - 1) / KT;

    if (warp == kMma) tmem_alloc(&bars->tmem, 512);
    if (tid == 0) {
        for (int i = 0; i < kRing; ++i) {
            mbar_init(&bars->ring_full[i], 1);
            mbar_init(&bars->ring_empty[i], kRingConsumers);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->kv_full[i], 1);
            mbar_init(&bars->kv_empty[i], 1);
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->pa_full[i], kSmN);
            mbar_init(&bars->dq_full[i], 1);
            mbar_init(&bars->dq_empty[i], kEpN);
        }
        for (int i = 0; i < kQSt; ++i) {
            mbar_init(&bars->qd_full[i], 2 * 32 * kPr);   // cp.async (noinc) + plain arrival per producer lane
            mbar_init(&bars->qd_empty[i], 1 + kEpN);      // MMA commit + epilogue (ids read)
        }
        mbar_init(&bars->dp_full, 1);
        mbar_init(&bars->p_full, kSmN);
        mbar_init(&bars->dkv_full, 1);
        mbar_init(&bars->dkv_empty, kEpN);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    auto qd_addr = [&](int st) { return sbase + oQD + st * 2 * kTile; };          // Q; dO at +kTile
    auto ldi_addr = [&](int st) { return sbase + oLDI + st * 3 * MQ * 4; };       // L; D at +512; id at +1024
    auto kv_addr = [&](int s) { return sbase + oKV + s * 2 * kTile; };            // K; V at +kTile

    if (warp < kPr) {
        // ---------------------------------------------------------- producers
        RingReader rr;
        int s_fetch = 0, g = 0, kv_use = 0;
        if (warp == 0 && lane == 0) {
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
        }
        for (;;) {
            int it;
            if (warp == 0) {
                if (lane == 0) {
                    const int slot = s_fetch % kRing;
                    mbar_wait(&bars->ring_empty[slot], ((s_fetch / kRing) & 1) ^ 1);
                    int v = atomicAdd(sched, 1);
                    it = v < n_items ? v : -1;
                    bars->ring[slot] = it;
                    mbar_arrive(&bars->ring_full[slot]);
                }
                ++s_fetch;
                it = __shfl_sync(0xffffffffu, it, 0);
            } else {
                it = rr.next(bars, lane);
            }
            if (it < 0) break;
            const Item x = decode(it, bh, hg, n_blocks, slabs, B, N, width, counts, offsets);
            if (x.n_tiles == 0) continue;
            if (warp == 0) {
                const int ks = kv_use & 1;
                mbar_wait(&bars->kv_empty[ks], ((kv_use >> 1) & 1) ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(&bars->kv_full[ks], 2 * kTile);
                    const int row0 = (int)((x.h / kv_group) * N + x.kb0);   // GQA: K/V head of query head x.h
                    tma_load_2d(kv_addr(ks), &tm_k, 0, row0, &bars->kv_full[ks]);
                    tma_load_2d(kv_addr(ks) + kTile, &tm_v, 0, row0, &bars->kv_full[ks]);
                }
                __syncwarp();
            }
            ++kv_use;
            const int32_t* fl = flat + x.fl_base;
            const __nv_bfloat16* Qh = Q + x.h * N * D;
            const __nv_bfloat16* dOh = dO + x.h * N * D;
            for (int t = 0; t < x.n_tiles; ++t, ++g) {
                const int st = g % kQSt;
                const int rows = min(MQ, x.cnt - t * MQ);
                // 8 lanes per 128-B row: a warp instruction gathers 4 rows
                const int sub = lane & 7, rsub = lane >> 3;
                constexpr int NI = (MQ / 4 + kPr - 1) / kPr;
                constexpr int NV = (MQ + 32 * kPr - 1) / (32 * kPr);
                int qrow[NI], qv[NV];
                float lv[NV], dv[NV];
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int r = 4 * (warp + kPr * i) + rsub;
                    qrow[i] = (r < rows) ? fl[t * MQ + r] : -1;
                }
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const int r = 32 * (warp + kPr * i) + lane;
                    qv[i] = (r < rows) ? fl[t * MQ + r] : -1;
                    lv[i] = (qv[i] >= 0) ? lse[x.h * N + qv[i]] * kLog2e : 0.f;
                    dv[i] = (qv[i] >= 0) ? Dd[x.h * N + qv[i]] : 0.f;
                }
                if (warp == 0) TRB(g, 0);
                mbar_wait(&bars->qd_empty[st], ((g / kQSt) & 1) ^ 1);
                if (warp == 0) TRB(g, 1);
                const uint32_t qb = qd_addr(st), db = qb + kTile;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int r = 4 * (warp + kPr * i) + rsub, qi = qrow[i];
                    if (r < MQ) {
                        const uint32_t off = sw128_off(r, sub * 8, MQ);
                        cp_async16(qb + off, Qh + (int64_t)max(qi, 0) * D + sub * 8, qi >= 0);
                        cp_async16(db + off, dOh + (int64_t)max(qi, 0) * D + sub * 8, qi >= 0);
                    }
                }
                cpasync_arrive_noinc(&bars->qd_full[st]);
                const uint32_t la = ldi_addr(st);
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const int r = 32 * (warp + kPr * i) + lane;
                    if (r < MQ) {
                        sts32(la + r * 4, __float_as_uint(lv[i]));
                        sts32(la + 512 + r * 4, __float_as_uint(dv[i]));
                        sts32(la + 1024 + r * 4, (uint32_t)qv[i]);
                    }
                }
                mbar_arrive(&bars->qd_full[st]);
                if (warp == 0) TRB(g, 2);
            }
        }
    } else if (warp == kMma) {
        // ---------------------------------------------------------- MMA issuer
        RingReader rr;
        const uint32_t idesc_kq = idesc_bf16(KT, MQ, false, false);   // S^T, dP^T
        const uint32_t idesc_kd = idesc_bf16(KT, D, false, true);     // dV, dK
        const uint32_t idesc_qd = idesc_bf16(MQ, D, true, true);      // dQ
        // tile stream: items with >= 1 tile, flattened
        struct Tile { int kvs, kvu, first, last; };
        int kv_use = 0, t_in = 0, n_in = 0;
        auto next_tile = [&](Tile& tl) -> bool {
            while (t_in == n_in) {
                const int it = rr.next(bars, lane);
                if (it < 0) return false;
                const Item x = decode(it, bh, hg, n_blocks, slabs, B, N, width, counts, offsets);
                if (x.n_tiles == 0) continue;
                n_in = x.n_tiles;
                t_in = 0;
                ++kv_use;
            }
            tl.kvu = kv_use - 1;
            tl.kvs = tl.kvu & 1;
            tl.first = t_in == 0;
            tl.last = t_in + 1 == n_in;
            ++t_in;
            return true;
        };
        auto issue_s = [&](const Tile& tl, int g) {
            if (tl.first) mbar_wait(&bars->kv_full[tl.kvs], (tl.kvu >> 1) & 1);
            mbar_wait(&bars->qd_full[g % kQSt], (g / kQSt) & 1);
            mbar_wait(&bars->dq_empty[g & 1], ((g >> 1) & 1) ^ 1);
            TRB(g, 3);
            tc_fence_after();
            fence_proxy_async_smem();
            // warp-uniform issue (elect.sync in the asm) with descriptors
            // advanced by constant offsets: a few instructions per MMA, which
            // matters because this warp shares its issue slots with softmax
            // and epilogue warps (K-major: +32 B per K16 step)
            const uint64_t dk = desc_kmajor(kv_addr(tl.kvs), 0), dq = desc_kmajor(qd_addr(g % kQSt), 0);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
                umma_bf16_w(tmem + cS0 + (g & 1) * 128, dk + 2 * kk, dq + 2 * kk, idesc_kq, kk > 0);
            umma_commit_w(&bars->s_full[g & 1]);
        };
        auto issue_dp = [&](const Tile& tl, int g) {
            const uint64_t dv = desc_kmajor(kv_addr(tl.kvs) + kTile, 0), ddo = desc_kmajor(qd_addr(g % kQSt) + kTile, 0);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
                umma_bf16_w(tmem + cY, dv + 2 * kk, ddo + 2 * kk, idesc_kq, kk > 0);
            umma_commit_w(&bars->dp_full);
        };
        Tile cur, nxt;
        bool have = next_tile(cur);
        int g = 0;
        if (have) {
            issue_s(cur, 0);
            issue_dp(cur, 0);
        }
        while (have) {
            const bool have_n = next_tile(nxt);
            if (have_n) issue_s(nxt, g + 1);
            // dV(g) needs only P(g): issued as soon as phase A has stored it,
            // so it runs on the tensor pipe while the softmax does phase B
            mbar_wait(&bars->pa_full[g & 1], (g >> 1) & 1);
            if (cur.first) mbar_wait(&bars->dkv_empty, (cur.kvu & 1) ^ 1);
            tc_fence_after();
            const uint32_t slot = tmem + cS0 + (g & 1) * 128;
            // MN-major operands: +16 rows x 128 B = 2 KB per K16 step
            const uint64_t d_k = desc_mnmajor(kv_addr(cur.kvs), 0, KT * 128);
            const uint64_t d_q = desc_mnmajor(qd_addr(g % kQSt), 0, MQ * 128);
            const uint64_t d_do = desc_mnmajor(qd_addr(g % kQSt) + kTile, 0, MQ * 128);
            const uint64_t d_ds = desc_mnmajor(sbase + oDS, 0, KT * 128);
#pragma unroll
            for (int kk = 0; kk < MQ / 16; ++kk)
                umma_bf16_ts_w(tmem + cDV, slot + 8 * kk, d_do + 128 * kk, idesc_kd, !cur.first || kk > 0);
            mbar_wait(&bars->p_full, g & 1);
            TRB(g, 4);
            tc_fence_after();
            fence_proxy_async_smem();
            // dK and dQ interleaved: two independent accumulation chains
#pragma unroll
            for (int kk = 0; kk < MQ / 16; ++kk) {
                umma_bf16_ts_w(tmem + cDK, tmem + cY + 8 * kk, d_q + 128 * kk, idesc_kd, !cur.first || kk > 0);
                umma_bf16_w(slot + 64, d_ds + 128 * kk, d_k + 128 * kk, idesc_qd, kk > 0);
            }
            TRB(g, 13);
            TRB(g, 14);
            umma_commit_w(&bars->dq_full[g & 1]);
            umma_commit_w(&bars->qd_empty[g % kQSt]);
            if (cur.last) {
                umma_commit_w(&bars->dkv_full);
                umma_commit_w(&bars->kv_empty[cur.kvs]);
            }
            TRB(g, 5);
            if (have_n) issue_dp(nxt, g + 1);
            cur = nxt;
            have = have_n;
            ++g;
        }
    } else if (warp < kEp0) {
        // ---------------------------------------------------------- softmax (phase A: P, phase B: dS)
        RingReader rr;
        const int quad = warp & 3;
        const int half = (warp - kSm0) >> 2;
        const int row = 32 * quad + lane;                    // key row of the slab
        const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
        const float sl2 = scale * kLog2e;
        int g = 0;
        for (;;) {
            const int it = rr.next(bars, lane);
            if (it < 0) break;
            const Item x = decode(it, bh, hg, n_blocks, slabs, B, N, width, counts, offsets);
            const int64_t key = x.kb0 + row;
            const bool krow_ok = row < x.klen;
            for (int t = 0; t < x.n_tiles; ++t, ++g) {
                const int st = g % kQSt;
                const uint32_t la = ldi_addr(st), da = la + 512, ia = la + 1024;
                const uint32_t slot = tmem + cS0 + (g & 1) * 128;
                const int rows_t = min(MQ, x.cnt - t * MQ);
                if (warp == kSm0) TRB(g, 6);
                mbar_wait(&bars->s_full[g & 1], (g >> 1) & 1);
                if (warp == kSm0) TRB(g, 7);
                tc_fence_after();
                // slices ascend: a tile whose first query is at or past the
                // slab's last key needs no causal mask
                const bool need_mask = rows_t < MQ || x.klen < KT || (int64_t)lds32i(ia) < x.kb0 + KT - 1;
                float sv[64];
                tmem_ld32(slot + lane_off + 64 * half, *reinterpret_cast<float(*)[32]>(&sv[0]));
                tmem_ld32(slot + lane_off + 64 * half + 32, *reinterpret_cast<float(*)[32]>(&sv[32]));
                tmem_ld_wait();
                // the mask test is hoisted out of the unrolled loop so each
                // variant is straight-line code (a branch per group of four
                // serialised the shared-memory loads and exponentials:
                // phase A 3076 -> 1578 clk per tile)
                if (need_mask) {
                    // padded rows carry id -1 and a dead key row never passes
                    const int kmask = krow_ok ? (int)key : 0x7fffffff;
#pragma unroll
                    for (int i = 0; i < 64; i += 4) {
                        const int c = 64 * half + i;
                        const float4 lv = lds128f(la + c * 4);
                        const int4 iv = lds128i(ia + c * 4);
                        const float l4[4] = {lv.x, lv.y, lv.z, lv.w};
                        const int i4[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float e = fast_exp2(fmaf(sv[i + u], sl2, -l4[u]));
                            sv[i + u] = kmask <= i4[u] ? e : 0.f;
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 64; i += 4) {
                        const int c = 64 * half + i;
                        const float4 lv = lds128f(la + c * 4);
                        const float l4[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            sv[i + u] = fast_exp2(fmaf(sv[i + u], sl2, -l4[u]));
                    }
                }
                // sv now holds P (fp32, kept for phase B); bf16 pairs go to TMEM
                uint32_t pk[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                named_bar(1 + quad, 64);        // both halves have read S^T from the slot
                tmem_st32(slot + lane_off + 32 * half, pk);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->pa_full[g & 1]);
                if (warp == kSm0) TRB(g, 8);
                // ---- phase B
                mbar_wait(&bars->dp_full, g & 1);
                if (warp == kSm0) TRB(g, 9);
                tc_fence_after();
                uint32_t dk[32];
#pragma unroll
                for (int c32 = 0; c32 < 2; ++c32) {
                    float dpv[32];
                    tmem_ld32(tmem + cY + lane_off + 64 * half + 32 * c32, dpv);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const int c = 64 * half + 32 * c32 + i;
                        const float4 dvv = lds128f(da + c * 4);
                        const float d4[4] = {dvv.x, dvv.y, dvv.z, dvv.w};
                        const int e = 16 * c32 + (i >> 1), q0 = 32 * c32 + i;
                        dk[e] = pack_bf16(sv[q0] * (dpv[i] - d4[0]), sv[q0 + 1] * (dpv[i + 1] - d4[1]));
                        dk[e + 1] = pack_bf16(sv[q0 + 2] * (dpv[i + 2] - d4[2]), sv[q0 + 3] * (dpv[i + 3] - d4[3]));
                    }
                }
                // dS^T row (this key, 64 queries of this half) -> SW128 slab `half` of the dQ A operand
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    sts128(sbase + oDS + sw128_off(row, 64 * half + 8 * c, KT),
                           make_uint4(dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]));
                named_bar(1 + quad, 64);        // both halves have read dP^T from Y
                tmem_st32(tmem + cY + lane_off + 32 * half, dk);
                tmem_st_wait();
                tc_fence_before();
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_full);
                if (warp == kSm0) TRB(g, 10);
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue: dQ per tile, dK/dV per item
        RingReader rr;
        const int quad = warp & 3;
        const int row = 32 * quad + lane;
        const uint32_t lane_off = (uint32_t)(32 * quad) << 16;
        const uint32_t srow = sbase + oSTG + (quad * kStgRows + (lane & 15)) * kStgRow;
        int g = 0, kv_use = 0;
        for (;;) {
            const int it = rr.next(bars, lane);
            if (it < 0) break;
            const Item x = decode(it, bh, hg, n_blocks, slabs, B, N, width, counts, offsets);
            for (int t = 0; t < x.n_tiles; ++t, ++g) {
                const int st = g % kQSt;
                mbar_wait(&bars->dq_full[g & 1], (g >> 1) & 1);
                if (warp == kEp0) TRB(g, 11);
                tc_fence_after();
                if (t + 1 == x.n_tiles) {
                    mbar_wait(&bars->dkv_full, kv_use & 1);
                    tc_fence_after();
                    const bool live = row < x.klen;
                    __nv_bfloat16* dk_row = dK + (x.h * N + x.kb0 + row) * D;
                    __nv_bfloat16* dv_row = dV + (x.h * N + x.kb0 + row) * D;
#pragma unroll
                    for (int which = 0; which < 2; ++which) {
                        float a[64];
                        const uint32_t col = which ? cDK : cDV;
                        tmem_ld32(tmem + col + lane_off, *reinterpret_cast<float(*)[32]>(&a[0]));
                        tmem_ld32(tmem + col + 32 + lane_off, *reinterpret_cast<float(*)[32]>(&a[32]));
                        tmem_ld_wait();
                        if (which == 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&bars->dkv_empty);
                        }
                        const float mul = which ? scale : 1.f;
                        __nv_bfloat16* dst = which ? dk_row : dv_row;
                        if (live) {
#pragma unroll
                            for (int c = 0; c < 8; ++c)
                                *reinterpret_cast<uint4*>(dst + 8 * c) =
                                    make_uint4(pack_bf16(a[8 * c] * mul, a[8 * c + 1] * mul),
                                               pack_bf16(a[8 * c + 2] * mul, a[8 * c + 3] * mul),
                                               pack_bf16(a[8 * c + 4] * mul, a[8 * c + 5] * mul),
                                               pack_bf16(a[8 * c + 6] * mul, a[8 * c + 7] * mul));
                        }
                    }
                    ++kv_use;
                }
                const int qi = lds32i(ldi_addr(st) + 1024 + row * 4);
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->qd_empty[st]);
                float v[64];
                tmem_ld32(tmem + cS0 + (g & 1) * 128 + 64 + lane_off, *reinterpret_cast<float(*)[32]>(&v[0]));
                tmem_ld32(tmem + cS0 + (g & 1) * 128 + 96 + lane_off, *reinterpret_cast<float(*)[32]>(&v[32]));
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->dq_empty[g & 1]);
                // one 256-B bulk op per row (fp32 reduce-add into dQ, or a
                // store of the per-(query, block) partial when deterministic);
                // the warp's 32 rows are staged 16 at a time. The bulk ops are
                // per-thread (a single issuing thread serialises them) and
                // each compiles to an elect/broadcast iteration, so fewer,
                // larger ops is what shortens this loop.
                const int64_t r_in = t * MQ + row;
#pragma unroll
                for (int rr = 0; rr < 2; ++rr) {
                    bulk_wait_read0();                       // the previous round's rows have been read
                    __syncwarp();
                    if ((lane >> 4) == rr) {
#pragma unroll
                        for (int i = 0; i < 64; i += 4)
                            sts128(srow + i * 4, make_uint4(__float_as_uint(v[i]), __float_as_uint(v[i + 1]),
                                                            __float_as_uint(v[i + 2]), __float_as_uint(v[i + 3])));
                        fence_proxy_async_smem();
                        if (qi >= 0) {
                            if (dq_part != nullptr)
                                bulk_store(dq_part + x.slab * part_stride + (x.fl_base + r_in) * D, srow, 256);
                            else
                                bulk_reduce_add_f32(dq_acc + (x.h * N + qi) * D, srow, 256);
                        }
                        bulk_commit();
                    }
                }
                if (warp == kEp0) TRB(g, 12);
            }
            // dK (scaled) and dV are zero when no query attends the block
            if (x.n_tiles == 0 && row < x.klen) {
                __nv_bfloat16* dk_row = dK + (x.h * N + x.kb0 + row) * D;
                __nv_bfloat16* dv_row = dV + (x.h * N + x.kb0 + row) * D;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    *reinterpret_cast<uint4*>(dk_row + 8 * c) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4*>(dv_row + 8 * c) = make_uint4(0, 0, 0, 0);
                }
            }
        }
        bulk_wait0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMma) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace bwdp

// host launcher (attn_bwd.cu): d = 64, block_size <= 256, sched = one zeroed int
int launch_bwd_pipe(const void* q, const void* k, const void* v, const void* dout, const float* lse, const float* Dd,
                    int64_t bh, int kv_group, int64_t N, int B, int width, const int32_t* counts, const int32_t* offsets,
                    const int32_t* flat, float scale, int* sched, float* dq_acc, float* dq_part,
                    int64_t part_stride, void* dk, void* dv, cudaStream_t s) {
    using namespace bwdp;
    static_assert(kSmem <= 232448, "backward smem budget");
    CUtensorMap tm_k, tm_v;
    if (!make_tmap_bf16(&tm_k, k, (uint64_t)(bh / kv_group * N), D, KT) ||
        !make_tmap_bf16(&tm_v, v, (uint64_t)(bh / kv_group * N), D, KT))
        return MOBA_ERR_CUDA;
    const int64_t n_items = bh * ceil_div(N, B) * ceil_div(B, KT);
    if (n_items >= (1ll << 31)) return MOBA_ERR_UNSUPPORTED;
    // heads per item group: the group's fp32 dQ accumulator rows <= 48 MB
    const int hg = (int)std::min<int64_t>(bh, std::max<int64_t>(1, (48ll << 20) / (N * D * 4)));
    cudaMemsetAsync(sched, 0, sizeof(int), s);
    auto kern = moba_bwd_pipe_kernel;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    const int grid = (int)std::min<int64_t>(n_items, kNumSMs);
    static long long* trace = nullptr;
    const char* trace_path = std::getenv("MOBA_BWD_TRACE");
    if (trace_path != nullptr && trace == nullptr) cudaMalloc(&trace, 256 * 16 * sizeof(long long));
    if (trace_path != nullptr) cudaMemsetAsync(trace, 0, 256 * 16 * sizeof(long long), s);
    kern<<<grid, kThreads, kSmem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)dout, tm_k, tm_v, lse, Dd, bh, hg,
                                       kv_group, N, B, width, counts, offsets, flat, scale, (int)n_items, sched, dq_acc, dq_part,
                                       part_stride, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv,
                                       trace_path != nullptr ? trace : nullptr,
                                       std::getenv("MOBA_BWD_TRACE_G0") ? std::atoi(std::getenv("MOBA_BWD_TRACE_G0")) : 0);
    int st = check_launch("moba_bwd_pipe_kernel");
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

}  // namespace moba
