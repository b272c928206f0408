// fs_order.cuh -- the queue's order from one fill to the next, hand-written
// (no library sort / select on the per-step path).
//
// lpm_order (local_policies.py:15-17) sorts the queue by (-match_len, arrival,
// rid) every fill.  The worker keeps its queue in (arrival, rid) label order,
// so a queue position is a dense label rank, and a stable sort by the key
// (kmax - mlen) over positions gives exactly lpm_order.  Between two fills
// most queued requests keep their match (incremental K1: the hint settles
// them), hence their key, so the new sorted order is
//
//   A  = the previous fill's sorted order restricted to the requests K1
//        settled this fill (still sorted by (key, label)), merged with
//   B  = everything else -- the positions K1 had to walk (hint gone, miss key
//        admitted) and the arrivals -- sorted by (key, position).
//
//   k_arrivals   arrivals join (state, per-client pending count, stale hints
//                dropped) and find their place in the old label order
//   k_upkeep     old queue minus last fill's admissions, arrivals merged in,
//                one pass (decoupled look-back over tiles)
//   (k_match_fast emits B in position order with the same look-back)
//   k_sort_b     B sorted by (key, position): one CTA in shared memory when
//                small, else a grid-wide stable LSD radix sort (cooperative)
//   k_merge_a    A in previous-sorted order -> final positions (rank in A +
//                B elements before it), scheduler slots gathered
//   k_scatter_b  B -> final positions (rank in B + A elements before it)
//
// With no usable previous order (first fill, hints off, a per-call tree edit)
// B is the whole queue and A is empty: the same kernels are a full sort.
#pragma once
#include <cooperative_groups.h>

#include "fs_kernels.cuh"

namespace cg = cooperative_groups;


// ---------------------------------------------------------------- queue upkeep
// Arrivals (label order): queued state, one more pending request for the
// client (Worker.enqueue -> on_request_enqueued), stale K1 hints dropped (a
// re-enqueued request's hint belongs to an older queue), and ins[k] = number
// of old queue entries with a smaller label.
__global__ void k_arrivals(const int32_t *__restrict__ ids, const int64_t *__restrict__ lab, int32_t nn,
                           const int32_t *__restrict__ oldq, int32_t no, const int64_t *__restrict__ rlabel,
                           int8_t *__restrict__ rstate, const int32_t *__restrict__ rclient,
                           int32_t *__restrict__ pend_cnt, int32_t *__restrict__ owner, int32_t *__restrict__ ins) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nn) return;
    const int32_t r = ids[k];
    rstate[r] = 1;
    atomicAdd(&pend_cnt[rclient[r]], 1);
    if (owner) owner[r] = -1;
    const int64_t l = lab[k];
    int32_t lo = 0, hi = no;
    // arrivals usually carry the largest labels: one probe settles them
    if (no > 0 && rlabel[oldq[no - 1]] < l) lo = hi = no;
    while (lo < hi) {
        const int32_t m = (lo + hi) >> 1;
        if (rlabel[oldq[m]] < l) lo = m + 1; else hi = m;
    }
    ins[k] = lo;
}

// first index in ins[lo, hi) with ins[i] > x (ins nondecreasing)
__device__ __forceinline__ int32_t upper_bound_i32(const int32_t *ins, int32_t lo, int32_t hi, int32_t x) {
    while (lo < hi) {
        const int32_t m = (lo + hi) >> 1;
        if (ins[m] <= x) lo = m + 1; else hi = m;
    }
    return lo;
}

// New label-ordered queue: the old entries still queued (state 1) and the
// arrivals, one tile of FS_OT_TILE old entries per block, striped (round u,
// thread t -> entry u*256 + t: coalesced loads and stores).  Launch
// max(1, tiles) blocks.
__global__ void __launch_bounds__(FS_OT_THREADS) k_upkeep(const int32_t *__restrict__ oldq, int32_t no,
                                                         const int8_t *__restrict__ rstate,
                                                         const int32_t *__restrict__ ins, int32_t nn,
                                                         const int32_t *__restrict__ newids,
                                                         int32_t *__restrict__ outq, unsigned long long *st,
                                                         uint32_t epoch, int32_t *ctr) {
    constexpr int NW = FS_OT_THREADS / 32;
    __shared__ uint32_t bal[FS_OT_ITEMS][NW];  // kept entries of each round and warp
    __shared__ int32_t rpre[FS_OT_ITEMS + 1];  // kept entries before each round
    __shared__ int64_t s_excl;
    __shared__ int32_t s_ka, s_kb;
    const int32_t tile = dyn_tile(ctr);
    const int32_t ntiles = max(1, (no + FS_OT_TILE - 1) / FS_OT_TILE);
    const int32_t base = tile * FS_OT_TILE;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int32_t v[FS_OT_ITEMS];
    uint32_t msk = 0;
#pragma unroll
    for (int u = 0; u < FS_OT_ITEMS; u++) {
        const int32_t i = base + u * FS_OT_THREADS + t;
        v[u] = i < no ? oldq[i] : -1;
        const bool kept = i < no && rstate[v[u]] == 1;
        if (kept) msk |= 1u << u;
        const unsigned bm = __ballot_sync(FS_FULL, kept);
        if (lane == 0) bal[u][warp] = bm;
    }
    __syncthreads();
    if (warp == 0) {
        int32_t tot = 0;
        for (int u = 0; u < FS_OT_ITEMS; u++) {
            if (lane == 0) rpre[u] = tot;
            for (int w = 0; w < NW; w++) tot += __popc(bal[u][w]);
        }
        const int64_t ex = warp_lookback(st, tile, epoch, tot, lane);
        if (lane != 0) goto up_done;
        rpre[FS_OT_ITEMS] = tot;
        s_excl = ex;
        // arrivals placed by this tile: ins in [base, base + TILE), the last
        // tile also takes ins == no
        const int32_t lo_x = base, hi_x = (tile == ntiles - 1) ? INT32_MAX : base + FS_OT_TILE;
        int32_t a2 = 0, b2 = nn;
        while (a2 < b2) { const int32_t m = (a2 + b2) >> 1; if (ins[m] < lo_x) a2 = m + 1; else b2 = m; }
        s_ka = a2;
        b2 = nn;
        int32_t c = a2;
        while (c < b2) { const int32_t m = (c + b2) >> 1; if (ins[m] < hi_x) c = m + 1; else b2 = m; }
        s_kb = c;
    }
up_done:
    __syncthreads();
    const int64_t excl = s_excl;
    const int32_t ka = s_ka, kb = s_kb, total = rpre[FS_OT_ITEMS];
    // kept entries of this tile before in-tile position x
    auto kept_before = [&](int32_t x) -> int32_t {
        if (x >= FS_OT_TILE) return total;
        const int32_t u = x / FS_OT_THREADS, tt = x % FS_OT_THREADS, w = tt >> 5, l = tt & 31;
        int32_t r = rpre[u];
        for (int k = 0; k < w; k++) r += __popc(bal[u][k]);
        return r + __popc(bal[u][w] & ((1u << l) - 1u));
    };
#pragma unroll
    for (int u = 0; u < FS_OT_ITEMS; u++) {
        if (msk & (1u << u)) {
            const int32_t i = base + u * FS_OT_THREADS + t;
            // arrivals with a smaller label: every ins[k] <= i
            const int32_t before = ka < kb ? upper_bound_i32(ins, ka, kb, i) : ka;
            outq[excl + kept_before(u * FS_OT_THREADS + t) + before] = v[u];
        }
    }
    for (int32_t k = ka + t; k < kb; k += FS_OT_THREADS) {
        const int32_t x = ins[k];
        const int32_t kbf = (x >= no) ? total : kept_before(x - base);
        outq[excl + kbf + k] = newids[k];
    }
}

// ---------------------------------------------------------------- sort of B
// B sorted by (key, queue position), one cooperative launch (grid = one CTA
// per SM).  Small B (the steady state: the positions K1 had to walk plus the
// arrivals, a few thousand) is sorted by CTA 0 alone in shared memory: a
// bitonic sort of the 64-bit (key << 32 | position) words, the other CTAs
// leave at once.  Large B (first fill, hints off, many invalidated hints):
// B in position order -- stable compaction of K1's per-position flags, or the
// identity -- then a stable LSD radix sort by key, 8-bit digits, every CTA
// owning a contiguous range; grid barriers between the phases.
#define FS_SB_THREADS 1024
#define FS_SB_CAP 8192
#define FS_SB_WARPS (FS_SB_THREADS / 32)

struct SortBArgs {
    const int32_t *jobs;   // B positions in any order (nullptr: B = 0..n-1)
    const int32_t *njobs;  // |B| on the device (nullptr: n)
    int32_t n;             // queue length
    const uint8_t *flag;   // flag[i]: position i is in B (with jobs)
    const uint32_t *keys;  // key of every queue position
    int32_t npass;         // 8-bit key digits
    int32_t cap;           // B up to this size is sorted by CTA 0 alone (<= FS_SB_CAP)
    uint32_t *bkey, *bkey2, *bkey3;  // out: bkey/bpos; scratch
    int32_t *bpos, *bpos2, *bpos3;
    int32_t *blk;          // [gridDim.x * 256] per-CTA counts
};

struct SortBSmem {
    union {
        unsigned long long w[FS_SB_CAP];  // small path
        struct {
            uint32_t wc[FS_SB_WARPS][FS_RS_BINS];  // (round << 16) | count per warp and digit
            int32_t h[FS_RS_BINS], base[FS_RS_BINS], run[FS_RS_BINS];
            int32_t red[FS_SB_WARPS];
            int64_t excl;
        } r;
    };
};

// block-wide exclusive scan of one int per thread (1024 threads)
__device__ inline int32_t block_excl_scan1024(int32_t v, int32_t *red, int32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FS_FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) red[warp] = x;
    __syncthreads();
    int32_t wb = 0, tot = 0;
    for (int k = 0; k < FS_SB_WARPS; k++) {
        const int32_t q = red[k];
        if (k < warp) wb += q;
        tot += q;
    }
    __syncthreads();
    *total = tot;
    return wb + x - v;
}

__global__ void __launch_bounds__(FS_SB_THREADS, 1) k_sort_b(SortBArgs a) {
    extern __shared__ __align__(16) unsigned char sb_raw[];
    SortBSmem &sm = *reinterpret_cast<SortBSmem *>(sb_raw);
    const int32_t nb = a.njobs ? *a.njobs : a.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (nb <= a.cap) {
        if (blockIdx.x != 0) return;
        int32_t P2 = 1;
        while (P2 < nb) P2 <<= 1;
        for (int32_t i = tid; i < P2; i += FS_SB_THREADS) {
            unsigned long long w = ~0ull;
            if (i < nb) {
                const int32_t pos = a.jobs ? a.jobs[i] : i;
                w = ((unsigned long long)a.keys[pos] << 32) | (uint32_t)pos;
            }
            sm.w[i] = w;
        }
        __syncthreads();
        for (int32_t k = 2; k <= P2; k <<= 1) {
            for (int32_t j = k >> 1; j > 0; j >>= 1) {
                for (int32_t i = tid; i < P2; i += FS_SB_THREADS) {
                    const int32_t l = i ^ j;
                    if (l > i) {
                        const unsigned long long x = sm.w[i], y = sm.w[l];
                        if (((i & k) == 0) == (x > y)) { sm.w[i] = y; sm.w[l] = x; }
                    }
                }
                __syncthreads();
            }
        }
        for (int32_t i = tid; i < nb; i += FS_SB_THREADS) {
            a.bkey[i] = (uint32_t)(sm.w[i] >> 32);
            a.bpos[i] = (int32_t)(sm.w[i] & 0xffffffffu);
        }
        return;
    }
    cg::grid_group g = cg::this_grid();
    const int32_t G = gridDim.x, b = blockIdx.x;
    const uint32_t *kin = nullptr;
    const int32_t *vin = nullptr;
    if (a.jobs) {
        // B in position order: stable compaction of the flags
        const int64_t lo = (int64_t)a.n * b / G, hi = (int64_t)a.n * (b + 1) / G;
        int32_t c = 0;
        for (int64_t i = lo + tid; i < hi; i += FS_SB_THREADS) c += a.flag[i];
        int32_t tot;
        (void)block_excl_scan1024(c, sm.r.red, &tot);
        if (tid == 0) a.blk[b] = tot;
        g.sync();
        int32_t pre = 0;
        for (int32_t k = tid; k < b; k += FS_SB_THREADS) pre += a.blk[k];
        int32_t ptot;
        (void)block_excl_scan1024(pre, sm.r.red, &ptot);
        int64_t o = ptot;
        for (int64_t i0 = lo; i0 < hi; i0 += FS_SB_THREADS) {
            const int64_t i = i0 + tid;
            const int32_t f = (i < hi) ? a.flag[i] : 0;
            int32_t t2;
            const int32_t ex = block_excl_scan1024(f, sm.r.red, &t2);
            if (f) { a.bpos3[o + ex] = (int32_t)i; a.bkey3[o + ex] = a.keys[i]; }
            o += t2;
        }
        g.sync();
        kin = a.bkey3;
        vin = a.bpos3;
    }
    const int64_t elo = (int64_t)nb * b / G, ehi = (int64_t)nb * (b + 1) / G;
    const unsigned lt = (1u << lane) - 1u;
    for (int32_t p = 0; p < a.npass; p++) {
        const int sh = 8 * p;
        const bool to_final = ((a.npass - 1 - p) % 2) == 0;
        uint32_t *ko = to_final ? a.bkey : a.bkey2;
        int32_t *vo = to_final ? a.bpos : a.bpos2;
        if (tid < FS_RS_BINS) { sm.r.h[tid] = 0; sm.r.run[tid] = 0; }
        for (int i = tid; i < FS_SB_WARPS * FS_RS_BINS; i += FS_SB_THREADS) (&sm.r.wc[0][0])[i] = 0xffff0000u;
        __syncthreads();
        for (int64_t e = elo + tid; e < ehi; e += FS_SB_THREADS) {
            const uint32_t k = kin ? kin[e] : a.keys[e];
            atomicAdd(&sm.r.h[(k >> sh) & 0xff], 1);
        }
        __syncthreads();
        if (tid < FS_RS_BINS) a.blk[(int64_t)b * FS_RS_BINS + tid] = sm.r.h[tid];
        g.sync();
        {
            // digit d: every CTA's count before this one plus all smaller digits
            int32_t tot = 0, pre = 0;
            if (tid < FS_RS_BINS) {
                for (int32_t k = 0; k < G; k++) {
                    const int32_t x = a.blk[(int64_t)k * FS_RS_BINS + tid];
                    tot += x;
                    if (k < b) pre += x;
                }
            }
            int32_t all;
            const int32_t ex = block_excl_scan1024(tid < FS_RS_BINS ? tot : 0, sm.r.red, &all);
            if (tid < FS_RS_BINS) sm.r.base[tid] = ex + pre;
        }
        __syncthreads();
        int32_t round = 0;
        for (int64_t e0 = elo; e0 < ehi; e0 += FS_SB_THREADS, round++) {
            const int64_t e = e0 + tid;
            const bool ok = e < ehi;
            uint32_t k = 0;
            int32_t v = 0;
            if (ok) {
                k = kin ? kin[e] : a.keys[e];
                v = vin ? vin[e] : (int32_t)e;
            }
            const uint32_t d = ok ? (k >> sh) & 0xff : 0x100u + lane;
            const unsigned peers = __match_any_sync(FS_FULL, d);
            const int32_t rk = __popc(peers & lt);
            const uint32_t tag = (uint32_t)(round & 0x7fff);
            if (ok && rk == 0) sm.r.wc[warp][d] = (tag << 16) | (uint32_t)__popc(peers);
            __syncthreads();
            if (ok) {
                int32_t pw = 0;
                for (int w = 0; w < warp; w++) {
                    const uint32_t x = sm.r.wc[w][d];
                    if ((x >> 16) == tag) pw += (int32_t)(x & 0xffff);
                }
                const int32_t dst = sm.r.base[d] + sm.r.run[d] + pw + rk;
                ko[dst] = k;
                vo[dst] = v;
            }
            __syncthreads();
            if (tid < FS_RS_BINS) {
                int32_t s2 = 0;
                for (int w = 0; w < FS_SB_WARPS; w++) {
                    const uint32_t x = sm.r.wc[w][tid];
                    if ((x >> 16) == tag) s2 += (int32_t)(x & 0xffff);
                }
                sm.r.run[tid] += s2;
            }
            __syncthreads();
        }
        g.sync();
        kin = ko;
        vin = vo;
    }
}

// ---------------------------------------------------------------- merge
// The scheduler's per-sorted-position slots for queue position qi.
struct SlotOut {
    const int32_t *queue, *cov, *next, *mlen, *tok0, *rclient, *rlen;
    const int64_t *s0;
    int32_t *s_req, *s_len, *s_mlen0, *s_tok0;
    int4 *slot;
    int64_t *s_src0;
};
// The previous fill's sorted slots: a settled request keeps its length, match,
// miss token and deepest chain (K1's outputs for it equal its hint, which is
// these), so k_merge_a reads them in order instead of gathering them.
struct PrevSlots {
    const int32_t *len, *mlen0, *tok0;
    const int64_t *src0;
};
__device__ __forceinline__ void emit_settled(const SlotOut &o, const PrevSlots &pv, int32_t p, int32_t j, int32_t r,
                                             int32_t qi) {
    o.s_req[p] = r;
    o.s_len[p] = pv.len[j];
    o.slot[p] = make_int4(o.rclient[r], o.cov[qi], o.next[qi], 0);
    o.s_mlen0[p] = pv.mlen0[j];
    o.s_tok0[p] = pv.tok0[j];
    o.s_src0[p] = pv.src0[j];
}
__device__ __forceinline__ void emit_slot(const SlotOut &o, int32_t p, int32_t qi) {
    const int32_t r = o.queue[qi];
    o.s_req[p] = r;
    o.s_len[p] = o.rlen[r];
    o.slot[p] = make_int4(o.rclient[r], o.cov[qi], o.next[qi], 0);
    o.s_mlen0[p] = o.mlen[qi];
    o.s_tok0[p] = o.tok0[qi];  // first token the step-start trie misses (K1)
    o.s_src0[p] = o.s0[qi];
}

__device__ __forceinline__ bool kq_less(uint32_t k1, int32_t q1, uint32_t k2, int32_t q2) {
    return k1 < k2 || (k1 == k2 && q1 < q2);
}

// A: the previous fill's sorted requests (p_req[0, np)) that K1 settled this
// fill -- settled[r] = (tag << 32) | queue position.  Each goes to its rank in
// A plus the number of B elements ordered before it; A's (key, position)
// pairs are written compactly for k_scatter_b.  Striped tiles (round u,
// thread t -> entry u*256 + t) keep every load and store coalesced; the B
// entries falling inside a tile's key range (a handful: B is sparse) are
// staged in shared memory once per tile.
#define FS_MA_BSTAGE 512
__global__ void __launch_bounds__(FS_OT_THREADS) k_merge_a(const int32_t *__restrict__ p_req, int32_t np,
                                                          const int64_t *__restrict__ settled, int64_t tag,
                                                          uint32_t kmax, PrevSlots pv,
                                                          const uint32_t *__restrict__ bkey,
                                                          const int32_t *__restrict__ bpos, SlotOut o,
                                                          unsigned long long *__restrict__ akq,
                                                          unsigned long long *st, uint32_t epoch, OrderCtl *oc) {
    __shared__ int32_t cnt[FS_OT_ITEMS][FS_OT_THREADS / 32];
    __shared__ unsigned long long sb[FS_MA_BSTAGE];
    __shared__ int32_t s_jmin, s_jmax, s_lo, s_m;
    __shared__ unsigned long long s_wmin, s_wmax;
    __shared__ int64_t s_excl;
    const int32_t tile = dyn_tile(&oc->tile[OT_MERGE_A]);
    const int32_t ntiles = (np + FS_OT_TILE - 1) / FS_OT_TILE;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int32_t base = tile * FS_OT_TILE;
    if (t == 0) { s_jmin = INT32_MAX; s_jmax = -1; }
    __syncthreads();
    int32_t qpos[FS_OT_ITEMS], rq[FS_OT_ITEMS];
    uint32_t key[FS_OT_ITEMS];
    uint32_t msk = 0;
#pragma unroll
    for (int u = 0; u < FS_OT_ITEMS; u++) {
        const int32_t j = base + u * FS_OT_THREADS + t;
        qpos[u] = -1;
        key[u] = 0;
        rq[u] = -1;
        if (j < np) {
            rq[u] = p_req[j];
            const int64_t s = settled[rq[u]];
            if ((s >> 32) == tag) {
                qpos[u] = (int32_t)(s & 0xffffffff);
                key[u] = kmax - (uint32_t)pv.mlen0[j];  // unchanged: the hint settled it
                msk |= 1u << u;
            }
        }
        const unsigned bal = __ballot_sync(FS_FULL, (msk >> u) & 1u);
        if (lane == 0) cnt[u][warp] = __popc(bal);
    }
    if (msk) {
        atomicMin(&s_jmin, base + (__ffs(msk) - 1) * FS_OT_THREADS + t);
        atomicMax(&s_jmax, base + (31 - __clz(msk)) * FS_OT_THREADS + t);
    }
    __syncthreads();
    if (warp == 0) {
        int32_t total = 0;
        for (int u = 0; u < FS_OT_ITEMS; u++)
            for (int w = 0; w < FS_OT_THREADS / 32; w++) total += cnt[u][w];
        const int64_t ex = warp_lookback(st, tile, epoch, total, lane);
        if (lane == 0) {
            s_excl = ex;
            if (tile == ntiles - 1) oc->na = (int32_t)(ex + total);
        }
    }
    // the tile's first and last kept entries (its smallest and largest keys)
    const int32_t jmin = s_jmin, jmax = s_jmax;
#pragma unroll
    for (int u = 0; u < FS_OT_ITEMS; u++) {
        const int32_t j = base + u * FS_OT_THREADS + t;
        if (j == jmin) s_wmin = ((unsigned long long)key[u] << 32) | (uint32_t)qpos[u];
        if (j == jmax) s_wmax = ((unsigned long long)key[u] << 32) | (uint32_t)qpos[u];
    }
    __syncthreads();
    const int32_t nb = oc->njobs;
    if (t == 0 && jmax >= 0) {
        // B entries before the tile's first kept entry, and those up to its last
        int32_t l = 0, h = nb;
        while (l < h) {
            const int32_t m = (l + h) >> 1;
            const unsigned long long w = ((unsigned long long)bkey[m] << 32) | (uint32_t)bpos[m];
            if (w < s_wmin) l = m + 1; else h = m;
        }
        const int32_t lo = l;
        h = nb;
        while (l < h) {
            const int32_t m = (l + h) >> 1;
            const unsigned long long w = ((unsigned long long)bkey[m] << 32) | (uint32_t)bpos[m];
            if (w < s_wmax) l = m + 1; else h = m;
        }
        s_lo = lo;
        s_m = l - lo;
    }
    __syncthreads();
    if (jmax < 0) return;  // nothing kept in this tile (its look-back word is published)
    const int32_t lo = s_lo, m = s_m;
    const bool staged = m <= FS_MA_BSTAGE;
    if (staged)
        for (int32_t i = t; i < m; i += FS_OT_THREADS)
            sb[i] = ((unsigned long long)bkey[lo + i] << 32) | (uint32_t)bpos[lo + i];
    __syncthreads();
    int32_t rbase = (int32_t)s_excl;
    const unsigned ltm = (1u << lane) - 1u;
#pragma unroll
    for (int u = 0; u < FS_OT_ITEMS; u++) {
        int32_t wpre = 0, rtot = 0;
        for (int w = 0; w < FS_OT_THREADS / 32; w++) {
            const int32_t c = cnt[u][w];
            if (w < warp) wpre += c;
            rtot += c;
        }
        const unsigned bal = __ballot_sync(FS_FULL, (msk >> u) & 1u);
        if ((msk >> u) & 1u) {
            const int32_t ra = rbase + wpre + __popc(bal & ltm);
            const unsigned long long me = ((unsigned long long)key[u] << 32) | (uint32_t)qpos[u];
            int32_t l = 0, h = m;  // B entries of the tile's range before this one
            if (staged) {
                while (l < h) { const int32_t mm = (l + h) >> 1; if (sb[mm] < me) l = mm + 1; else h = mm; }
            } else {
                while (l < h) {
                    const int32_t mm = (l + h) >> 1;
                    const unsigned long long w = ((unsigned long long)bkey[lo + mm] << 32) | (uint32_t)bpos[lo + mm];
                    if (w < me) l = mm + 1; else h = mm;
                }
            }
            akq[ra] = me;
            emit_settled(o, pv, ra + lo + l, base + u * FS_OT_THREADS + t, rq[u], qpos[u]);
        }
        rbase += rtot;
    }
}

// B (sorted by key, then position): rank in B plus the A elements before it.
__global__ void k_scatter_b(const uint32_t *__restrict__ bkey, const int32_t *__restrict__ bpos,
                            const int32_t *nbp, int32_t n, const unsigned long long *__restrict__ akq,
                            const OrderCtl *oc, SlotOut o) {
    // every S-th packed A key in shared memory: the search per B entry is a
    // shared-memory bisection plus one over S entries in global memory
    constexpr int SAMPLES = 2048;
    __shared__ unsigned long long smp[SAMPLES];
    const int32_t nb = nbp ? *nbp : n;
    const int32_t na = oc->na;
    if (nb == 0) return;
    const int32_t S = max(1, (na + SAMPLES - 1) / SAMPLES);
    const int32_t ns = na > 0 ? (na + S - 1) / S : 0;
    for (int32_t i = threadIdx.x; i < ns; i += blockDim.x) smp[i] = akq[(int64_t)i * S];
    __syncthreads();
    for (int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; kk < nb; kk += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = (int32_t)kk;
        const uint32_t key = bkey[k];
        const int32_t qi = bpos[k];
        const unsigned long long me = ((unsigned long long)key << 32) | (uint32_t)qi;
        int32_t l = 0, h = ns;  // samples below me
        while (l < h) { const int32_t m = (l + h) >> 1; if (smp[m] < me) l = m + 1; else h = m; }
        // A entries below me lie in [(l - 1) * S, l * S)
        int32_t lo = l > 0 ? (l - 1) * S + 1 : 0, hi = min(na, l * S);
        while (lo < hi) {
            const int32_t m = (lo + hi) >> 1;
            if (akq[m] < me) lo = m + 1; else hi = m;
        }
        emit_slot(o, k + lo, qi);
    }
}
