// fs_kernels.cuh -- kernels of the decision path.
//
//   K1  k_match      warp-per-request longest-prefix match of the whole queue
//                    against the device trie (chain-jumping walk), stamping
//                    last_access, emitting (mlen key, pinned coverage B, the
//                    token after B).
//   K2  (CUB radix sort of the 13-16-bit (L - mlen) key, stable => ties stay in
//        the (arrival, rid) label order the queue is kept in)
//   K3+K4 k_schedule one persistent CTA: deficit-gated first-admissible search
//                    with the closed-form refill and budget test, and each
//                    admission's radix insert / split / LRU evict / pin.
//   k_unpin_many     batch completion: warp per finished path.
//   k_op / k_dispatch single-CTA tree operations and D2LPM dispatch chains.
#pragma once
#include "fs_device.cuh"
#include "fs_scan.cuh"

#ifndef FS_SCHED_THREADS
#define FS_SCHED_THREADS 512  // 112 registers without spills (1024 threads capped them at 64)
#endif
#ifndef FS_DISPATCH_THREADS
#define FS_DISPATCH_THREADS 1024  // one batch of block_path_nodes covers an 8k-token path
#endif
#ifndef FS_DISP_STAGE
#define FS_DISP_STAGE 256
#endif
#ifndef FS_PRE_SEGS
#define FS_PRE_SEGS 32
#endif
#ifndef FS_ITEMS
#define FS_ITEMS 8
#endif
#define FS_CHUNK (FS_SCHED_THREADS * FS_ITEMS)
#define FS_NONE 0x7fffffff
#ifndef FS_FSLOTS
// admission filter slots (shared memory + global mirror): saturates at 1024
// admissions per fill (two keys each, half load), after which stale
// coverages are re-walked.  Kept small: the rest of the SM's 256 KB is L1
// for the admission chain (FS_SCHED_CARVEOUT).
#define FS_FSLOTS 4096
#endif
#define FS_MKEY_SLOTS FS_FSLOTS

// ---------------------------------------------------------------- K1
// Per-request match hints kept across fills (incremental K1).  Between two
// fills of a worker the trie changes only through that fill's admissions
// (when no per-call operation touched the tree since -- the host checks a
// structural version), so a queued request's previous match p[:m] is still
// the exact match when (i) its deepest node is still cached -- one pos lookup
// (pos_valid), because a cached depth of a chain implies its whole root path is
// cached -- and (ii) no admission of that fill had the request's miss key
// (m, p[m]): an insert can extend p's match only if it shares p[:m+1], which
// forces its own step-start match to stop at the same depth with the same
// token (k_schedule's miss-key argument).  Otherwise the walk resumes at m, or
// starts from the root when the hint is gone.
struct K1Hints {
    int32_t *owner;                   // worker the hint belongs to (-1: none)
    int32_t *m;                       // match length (also the L2 prefetch extent)
    int64_t *S0;                      // chain (arena row) of the deepest matched node
    int32_t *tok0;                    // token at m, -1 when fully matched
    const unsigned long long *mkeys;  // the last fill's admission filter (global mirror)
    int32_t wid;
    int32_t use;                      // hints are valid for this fill
};

__device__ __forceinline__ bool mkey_hit(const unsigned long long *keys, int32_t m, int32_t tok) {
    const unsigned long long k = ((unsigned long long)((uint32_t)m | 0x80000000u) << 32) | (uint32_t)tok;
    uint32_t i = fs_hmix(k) & (FS_MKEY_SLOTS - 1);
    while (true) {
        const unsigned long long x = keys[i];
        if (x == k) return true;
        if (x == FS_HEMPTY) return false;
        i = (i + 1) & (FS_MKEY_SLOTS - 1);
    }
}

template <int U, bool PIPE, bool JOBS = false>
__global__ void __launch_bounds__(256, PIPE ? 8 : 1) k_match(TrieView t, const int32_t *__restrict__ ids, int32_t n,
                                               const int64_t *__restrict__ roff, const int32_t *__restrict__ rlen,
                                               int64_t now, int stamp, int64_t sq, uint32_t kmax,
                                               uint32_t *__restrict__ out_key, int32_t *__restrict__ out_mlen,
                                               int32_t *__restrict__ out_cov, int32_t *__restrict__ out_next,
                                               int64_t *__restrict__ out_s0, int32_t *__restrict__ out_tok0,
                                               unsigned long long *__restrict__ alg_tokens,
                                               K1Hints hints, const int32_t *__restrict__ jobs = nullptr,
                                               const int32_t *__restrict__ njobs = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // jobs != nullptr: persistent warps take the queue positions k_match_fast
    // could not settle (jobs[0, *njobs)); otherwise warp i takes position i
    const int64_t nw = JOBS ? ((int64_t)gridDim.x * blockDim.x) >> 5 : 1;
    const int64_t nj = JOBS ? *njobs : (gw < n ? gw + 1 : 0);
    for (int64_t k = gw; k < nj; k += nw) {
    const int64_t i = JOBS ? jobs[k] : k;
    // ids == nullptr: roff/rlen are the i-th sequence's arena offset and length
    // (eviction-notice paths), not request-table columns
    const int32_t r = ids ? ids[i] : (int32_t)i;
    const int32_t len = rlen[r];
    const int32_t *rq = t.arena + roff[r];
    int32_t hy = -1, hm = -1, htok = -1;
    bool stream = true;
    if (hints.use && hints.owner[r] == hints.wid) {
        hm = hints.m[r];
        htok = hints.tok0[r];
        if (hm > 0) {
            const int64_t S0 = hints.S0[r];
            const int32_t c = t.pos[S0 + hm - 1];
            if (pos_valid(t, c, S0, hm - 1)) hy = c;
        }
        if (hy > 0) stream = htok >= 0 && mkey_hit(hints.mkeys, hm, htok);
    }
    if (stream && hints.m) {
        // The request tokens this match will read are known up to the previous
        // step's match length: hand them to the TMA engine as L2 bulk prefetches
        // (4 KB per lane) so the DRAM fetch overlaps the trie hops below.
        const int32_t b_lo = hy > 0 ? hm : 0;
        const int32_t want = min(len, hints.m[r] + 32);
        const int32_t nb = (max(0, want - (b_lo & ~1023)) * 4 + 4095) >> 12;
        if (lane < nb) {
            const int32_t b0 = (b_lo & ~1023) + (lane << 10);
            const uint32_t bytes = (uint32_t)(((min(want, b0 + 1024) - b0) * 4 + 15) & ~15);
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(rq + b0), "r"(bytes),
                         "l"(l2_evict_first()) : "memory");
        }
    }
    WalkOut w;
    int32_t read_from = 0;
    if (hy > 0) {
        // the previous match still holds: coverage from the deep end; the walk
        // continues only if an admission of the last fill shared the miss key
        const int32_t cov0 = warp_cov_from_deepest(t, hy, hm, lane);
        if (!stream || hm < t.end[hy]) {
            w.mlen = hm; w.last = hy; w.plen = 0; w.nseg = 0; w.cov = cov0; w.unpinned = hm - cov0;
            read_from = hm + 1;  // nothing to read
        } else {
            WalkStart st;
            st.node = hy; st.idx = hm; st.nseg = 0; st.last = hy; st.cov = cov0; st.pinrun = cov0 == hm;
            auto none = [](int64_t, int32_t, int32_t, int32_t) {};
            w = warp_walk_from<8>(t, rq, len, lane, true, st, none);
            read_from = hm;
        }
    } else {
        w = warp_walk<U, PIPE>(t, rq, len, lane, nullptr, true);
    }
    if (lane == 0) {
        // match_prefix stamps every matched node (radix.py:86-90): lazily, at the deepest
        if (stamp && w.last > 0) stamp_node(t, w.last, now, sq);
        if (out_key) out_key[i] = kmax - (uint32_t)w.mlen;
        if (out_mlen) out_mlen[i] = w.mlen;
        if (out_cov) out_cov[i] = w.cov;
        if (out_next) out_next[i] = w.cov < len ? rq[w.cov] : -1;
        const int64_t s0 = w.last > 0 ? t.src[w.last] : -1;
        if (out_s0) out_s0[i] = s0;  // admission-walk hint
        const int32_t tok0 = (w.mlen == hm && hy > 0) ? htok : (w.mlen < len ? rq[w.mlen] : -1);
        if (out_tok0) out_tok0[i] = tok0;  // first token the step-start trie misses
        if (hints.owner) {
            hints.owner[r] = hints.wid;
            hints.S0[r] = s0;
            hints.tok0[r] = tok0;
        }
        if (hints.m) hints.m[r] = w.mlen;
        // request tokens this match read: [read_from, min(mlen+1, len)) (SURVEY 8d,
        // minus what the hint already established); the counters are spread over
        // 64 slot pairs (summed by the host)
        if (alg_tokens) {
            unsigned long long *slot = alg_tokens + 2 * (blockIdx.x & 63);
            atomicAdd(slot, (unsigned long long)max(0, min(w.mlen + 1, len) - read_from));
            atomicAdd(slot + 1, (unsigned long long)w.nseg);  // source chains crossed
        }
    }
    }
}

// ---------------------------------------------------------------- K1, TMA-fed streaming scan
// The full re-match (no usable hints: first fill, FS_OPT_K1_FULL, a per-call
// tree edit) streams every queued request's matched prefix from HBM -- the
// metric's "prefix-match GB/s".  Here the request row is staged through a
// per-warp shared-memory ring by the TMA engine (cp.async.bulk into shared
// memory, one mbarrier per stage, complete_tx): K1M_NST chunks of K1M_CH
// tokens in flight per warp, issued ahead of the compare, so the DRAM stream
// does not wait on each 512-byte compare step as the register loop does.  The
// extent fetched is the previous fill's match length (+32), so nothing past the
// match is streamed.  The trie side (other requests' rows, hot in L2/L1) stays
// on __ldg.  Same walk and outputs as k_match (warp_walk_from with coverage).
#ifndef K1M_CH
#define K1M_CH 512      // tokens per chunk (2 KB)
#endif
#ifndef K1M_NST
#define K1M_NST 4       // chunks in flight per warp
#endif
#define K1M_WARPS 8     // warps per CTA
#ifndef K1M_L2PF
#define K1M_L2PF 1      // bulk L2 prefetch of the whole extent at the row's start
#endif

struct K1Ring {
    int32_t *buf;        // K1M_NST * K1M_CH tokens (shared)
    uint64_t *bar;       // K1M_NST mbarriers (shared)
    const int32_t *row;  // request row (global, 16-B aligned)
    int32_t E;           // tokens staged: [0, E)
    int32_t nch;         // chunks of [0, E)
    int32_t issued;      // chunks issued so far
    int32_t landed;      // chunks known to have landed (waited for, in order)
    uint32_t phase;      // parity bit per stage
    uint64_t pol;        // L2 evict-first policy
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// lane 0: put chunk c of the row in flight into stage c % K1M_NST
__device__ __forceinline__ void k1r_issue(K1Ring &R, int32_t c) {
    const int st = c % K1M_NST;
    const int32_t lo = c * K1M_CH, hi = min(R.E, lo + K1M_CH);
    const uint32_t bytes = (uint32_t)(((hi - lo) * 4 + 15) & ~15);
    const uint32_t b = smem_addr(R.bar + st);
    // the stage's previous contents were read through the generic proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_addr(R.buf + st * K1M_CH)), "l"(R.row + lo), "r"(bytes), "r"(b), "l"(R.pol)
                 : "memory");
}

// Warp-uniform: chunks [landed, c_hi] have landed.  Chunks below c_lo are
// consumed (positions are read in nondecreasing order), so their stages may be
// refilled: chunks up to c_lo + K1M_NST - 1 are put in flight.
__device__ __forceinline__ void k1r_need(K1Ring &R, int32_t c_lo, int32_t c_hi, int lane) {
    c_hi = min(c_hi, R.nch - 1);
    while (true) {
        // chunk k refills the stage of chunk k - K1M_NST: that one must have
        // landed and be consumed
        const int32_t want = min(R.nch, min(c_lo, R.landed) + K1M_NST);
        if (R.issued < want) {
            __syncwarp();  // every lane is done with the stages being refilled
            if (lane == 0)
                for (int32_t k = R.issued; k < want; k++) k1r_issue(R, k);
            R.issued = want;
        }
        if (R.landed > c_hi) break;
        const int st = R.landed % K1M_NST;
        const uint32_t b = smem_addr(R.bar + st), par = (R.phase >> st) & 1u;
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(b), "r"(par) : "memory");
        R.phase ^= 1u << st;
        R.landed++;
    }
}

// is position p's chunk still in its stage?
__device__ __forceinline__ bool k1r_resident(const K1Ring &R, int32_t p) {
    return p < R.E && p / K1M_CH + K1M_NST >= R.issued;
}
__device__ __forceinline__ const int32_t *k1r_ptr(const K1Ring &R, int32_t p) {
    return R.buf + (p / K1M_CH % K1M_NST) * K1M_CH + p % K1M_CH;
}

// warp-uniform p: request token p (its staged chunk, else global memory)
__device__ __forceinline__ int32_t k1r_tok(K1Ring &R, int32_t p, int lane) {
    if (p < R.E) {
        const int32_t c = p / K1M_CH;
        if (c >= R.landed) {  // ahead of the stream: wait for it
            k1r_need(R, c, c, lane);
            return *k1r_ptr(R, p);
        }
        if (c + K1M_NST >= R.issued) return *k1r_ptr(R, p);  // landed, stage not refilled
    }
    return __ldg(R.row + p);
}

// drain: wait for every chunk issued for this row (stage parity stays in step)
__device__ __forceinline__ void k1r_drain(K1Ring &R, int lane) {
    while (R.landed < R.issued) {
        const int st = R.landed % K1M_NST;
        const uint32_t b = smem_addr(R.bar + st), par = (R.phase >> st) & 1u;
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(b), "r"(par) : "memory");
        R.phase ^= 1u << st;
        R.landed++;
    }
    __syncwarp();
}

// LCP of the chain row a[i0, n) with the request tokens [i0, n), chunk by
// chunk: one ring check per staged chunk, then 512 tokens per step (lane l
// compares 4 x 4 tokens, 16-B aligned: both rows are co-aligned arena rows
// read at the same depth), four independent trie-side loads in flight per
// lane.  Returns the first mismatch (or n).
__device__ __forceinline__ int k1r_first_diff(const int4 &x, const int4 &y, int32_t p, int32_t n) {
    int f = 4;
    if (x.w != y.w && p + 3 < n) f = 3;
    if (x.z != y.z && p + 2 < n) f = 2;
    if (x.y != y.y && p + 1 < n) f = 1;
    if (x.x != y.x && p < n) f = 0;
    return f;
}
__device__ inline int32_t k1r_lcp(K1Ring &R, const int32_t *__restrict__ a, int32_t i0, int32_t n, int lane) {
    if (i0 >= n) return n;
    // scalar head up to the next 16-B boundary
    const int32_t h = min(n, (i0 + 3) & ~3);
    if (h > i0) {
        if (i0 < R.E) k1r_need(R, i0 / K1M_CH, (min(h, R.E) - 1) / K1M_CH, lane);
        const int32_t p = i0 + lane;
        bool bad = false;
        if (p < h) bad = __ldg(a + p) != (k1r_resident(R, p) ? *k1r_ptr(R, p) : __ldg(R.row + p));
        const unsigned m = __ballot_sync(FS_FULL, bad);
        if (m) return i0 + __ffs(m) - 1;
    }
    int32_t k = h;
    while (k < n) {
        const bool staged = k < R.E;
        int32_t seg_end = n;
        const int32_t *bb = R.row;  // bb[p]: request token p
        if (staged) {
            const int32_t c = k / K1M_CH;
            k1r_need(R, c, c, lane);
            seg_end = min(n, (c + 1) * K1M_CH);
            bb = R.buf + (c % K1M_NST) * K1M_CH - c * K1M_CH;
        }
        for (; k < seg_end; k += 512) {
            int f[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int32_t p = k + 128 * u + 4 * lane;
                f[u] = 4;
                if (p < seg_end) {
                    const int4 av = __ldg(reinterpret_cast<const int4 *>(a + p));
                    const int4 bv = staged ? *reinterpret_cast<const int4 *>(bb + p)
                                           : __ldg(reinterpret_cast<const int4 *>(bb + p));
                    f[u] = k1r_first_diff(av, bv, p, n);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const unsigned m = __ballot_sync(FS_FULL, f[u] < 4);
                if (m) {
                    const int L = __ffs(m) - 1;
                    return min(n, k + 128 * u + 4 * L + __shfl_sync(FS_FULL, f[u], L));
                }
            }
        }
        k = seg_end;
    }
    return n;
}

__global__ void __launch_bounds__(32 * K1M_WARPS) k_match_tma(TrieView t, const int32_t *__restrict__ ids, int32_t n,
                                                           const int64_t *__restrict__ roff,
                                                           const int32_t *__restrict__ rlen, int64_t now, int64_t sq,
                                                           uint32_t kmax, uint32_t *__restrict__ out_key,
                                                           int32_t *__restrict__ out_mlen, int32_t *__restrict__ out_cov,
                                                           int32_t *__restrict__ out_next, int64_t *__restrict__ out_s0,
                                                           int32_t *__restrict__ out_tok0,
                                                           unsigned long long *__restrict__ alg_tokens, K1Hints hints) {
    extern __shared__ __align__(128) unsigned char k1m_sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    K1Ring R;
    R.buf = reinterpret_cast<int32_t *>(k1m_sm) + warp * K1M_NST * K1M_CH;
    R.bar = reinterpret_cast<uint64_t *>(k1m_sm + K1M_WARPS * K1M_NST * K1M_CH * 4) + warp * K1M_NST;
    R.phase = 0;
    R.pol = l2_evict_first();
    if (lane < K1M_NST) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(R.bar + lane)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t nw = (int64_t)gridDim.x * K1M_WARPS;
    for (int64_t i = (int64_t)blockIdx.x * K1M_WARPS + warp; i < n; i += nw) {
        const int32_t r = ids[i];
        const int32_t len = rlen[r];
        R.row = t.arena + roff[r];
        // staged extent: the previous match (+32) -- what this match will read
        R.E = hints.m ? min(len, hints.m[r] + 32) : len;
        R.E = min(len, (R.E + 3) & ~3);
        R.nch = (R.E + K1M_CH - 1) / K1M_CH;
        R.issued = 0;
        R.landed = 0;
#if K1M_L2PF
        {
            // the whole staged extent to L2 up front (4 KB per lane, as k_match):
            // the ring then refills from L2
            const int32_t nb = (R.E * 4 + 4095) >> 12;
            for (int32_t q = lane; q < nb; q += 32) {
                const int32_t b0 = q << 10;
                const uint32_t bytes = (uint32_t)(((min(R.E, b0 + 1024) - b0) * 4 + 15) & ~15);
                asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(R.row + b0), "r"(bytes),
                             "l"(R.pol) : "memory");
            }
        }
#endif
        if (lane == 0)
            for (int32_t k = 0; k < min(R.nch, K1M_NST); k++) k1r_issue(R, k);
        R.issued = min(R.nch, K1M_NST);
        // RadixTree._walk (radix.py:60-81) chain by chain, as warp_walk_from
        WalkOut o;
        o.mlen = 0; o.last = -1; o.plen = 0; o.nseg = 0; o.cov = 0; o.unpinned = 0;
        int32_t node = 0, idx = 0;
        bool pinrun = true;
        while (idx < len) {
            const int32_t c = h_find(t, node, k1r_tok(R, idx, lane));
            if (c < 0) break;
            const int64_t S = t.src[c];
            const int32_t bound = min(len, t.slen[c]);
            const int32_t D = k1r_lcp(R, t.arena + S, idx + 1, bound, lane);  // request == chain S on [idx, D)
            const int32_t y = chain_lookup(t, S, idx, D - 1);
            const int32_t e = t.end[y];
            const int32_t b = min(D, e);
            o.nseg++;
            if (pinrun) {
                o.cov = warp_seg_cov(t, S, idx, b, y, lane);
                pinrun = o.cov == b;
            }
            o.last = y;
            if (D < e) { o.plen = D - t.start[y]; idx = D; break; }
            idx = e;
            node = y;
        }
        o.mlen = idx;
        o.unpinned = o.mlen - o.cov;
        const int32_t tokcov = o.cov < len ? k1r_tok(R, o.cov, lane) : -1;
        const int32_t tokm = o.mlen < len ? k1r_tok(R, o.mlen, lane) : -1;
        k1r_drain(R, lane);
        if (lane == 0) {
            if (o.last > 0) stamp_node(t, o.last, now, sq);  // match_prefix stamps (radix.py:86-90), lazily
            out_key[i] = kmax - (uint32_t)o.mlen;
            out_mlen[i] = o.mlen;
            out_cov[i] = o.cov;
            out_next[i] = tokcov;
            const int64_t s0 = o.last > 0 ? t.src[o.last] : -1;
            out_s0[i] = s0;
            out_tok0[i] = tokm;
            if (hints.owner) {
                hints.owner[r] = hints.wid;
                hints.S0[r] = s0;
                hints.tok0[r] = tokm;
            }
            if (hints.m) hints.m[r] = o.mlen;
            if (alg_tokens) {
                unsigned long long *slot = alg_tokens + 2 * (blockIdx.x & 63);
                atomicAdd(slot, (unsigned long long)min(o.mlen + 1, len));
                atomicAdd(slot + 1, (unsigned long long)o.nseg);
            }
        }
    }
}

// Pinned coverage of the cached root path [0, d) ending in node y, by one
// thread: chain by chain from the deep end (refs never increase with depth);
// inside the chain where pinning stops, up the parent links to the deepest
// pinned node.  Same value as warp_cov_from_deepest.
__device__ inline int32_t thread_cov_from_deepest(const TrieView &t, int32_t y, int32_t d) {
    int32_t cur = y;
    while (d > 0 && cur > 0) {
        const int64_t S = t.src[cur];
        const int32_t c0 = t.ctop[cur];
        const int32_t X = t.cpar[cur];
        if (t.ref[t.pos[S + c0]] > 0) {
            int32_t n = cur;
            while (t.ref[n] == 0) n = t.parent[n];
            return min(t.end[n], d);
        }
        d = c0;
        cur = X;
    }
    return 0;
}

// The same, also returning the request's token at the coverage depth (the
// scheduler's filter key) from the trie side -- the path's tokens equal the
// request's up to d, so it is the first token of the node that starts there
// (L2-resident node fields instead of a DRAM read of the request row).
// tok_d: the request's token at depth d (-1 when d == len).
__device__ inline int32_t thread_cov_tok_from_deepest(const TrieView &t, int32_t y, int32_t d, int32_t tok_d,
                                                      int32_t *tok_cov) {
    int32_t cur = y, tok = tok_d;
    while (d > 0 && cur > 0) {
        const int64_t S = t.src[cur];
        const int32_t c0 = t.ctop[cur];
        const int32_t X = t.cpar[cur];
        const int32_t top = t.pos[S + c0];
        if (t.ref[top] > 0) {
            int32_t n = cur, prev = -1;
            while (t.ref[n] == 0) { prev = n; n = t.parent[n]; }
            const int32_t cv = min(t.end[n], d);
            *tok_cov = (prev >= 0 && cv < d) ? t.first[prev] : tok;
            return cv;
        }
        tok = t.first[top];  // the path's token at depth c0
        d = c0;
        cur = X;
    }
    *tok_cov = tok;
    return 0;
}

// K1 fast path, one thread per queued request: a request whose hint settles
// its match (K1Hints: deepest node still cached, miss key not admitted) gets
// every output here; the others are queued for the warp-per-request walk.
__global__ void __launch_bounds__(256) k_match_fast(TrieView t, const int32_t *__restrict__ ids, int32_t n,
                                                    const int64_t *__restrict__ roff,
                                                    const int32_t *__restrict__ rlen, int64_t now, int64_t sq,
                                                    uint32_t kmax, uint32_t *__restrict__ out_key,
                                                    int32_t *__restrict__ out_mlen, int32_t *__restrict__ out_cov,
                                                    int32_t *__restrict__ out_next, int64_t *__restrict__ out_s0,
                                                    int32_t *__restrict__ out_tok0, K1Hints hints,
                                                    int32_t *__restrict__ jobs, OrderCtl *oc,
                                                    uint8_t *__restrict__ slow_flag,
                                                    int64_t *__restrict__ smark, int64_t stag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // the block's deepest nodes already stamped: many queued requests share
    // their deepest node, and concurrent stores to one line serialize in L2
    __shared__ int32_t stamped[128];
    if (threadIdx.x < 128) stamped[threadIdx.x] = -1;
    __syncthreads();
    bool slow = true;
    if (i < n) {
        const int32_t r = ids[i];
        if (hints.use && hints.owner[r] == hints.wid) {
            const int32_t hm = hints.m[r];
            const int32_t htok = hints.tok0[r];
            const int64_t S0 = hints.S0[r];
            int32_t y = -1;
            bool settled = false;
            if (hm == 0) {
                settled = htok < 0 || !mkey_hit(hints.mkeys, 0, htok);
            } else {
                const int32_t c = t.pos[S0 + hm - 1];
                if (pos_valid(t, c, S0, hm - 1)) {
                    y = c;
                    settled = htok < 0 || hm < t.end[c] || !mkey_hit(hints.mkeys, hm, htok);
                }
            }
            if (settled) {
                slow = false;
                const int32_t len = rlen[r];
                int32_t tokc = htok;
                const int32_t cov = y > 0 ? thread_cov_tok_from_deepest(t, y, hm, htok, &tokc) : 0;
                if (y > 0) {
                    uint32_t h = ((uint32_t)y * 2654435761u) >> 25;  // 128 slots
                    bool mine = false;
                    for (int probe = 0; probe < 8; probe++) {
                        const int32_t old = atomicCAS(&stamped[h], -1, y);
                        if (old == -1) { mine = true; break; }
                        if (old == y) break;
                        h = (h + 1) & 127u;
                        if (probe == 7) mine = true;  // table crowded: stamp anyway (idempotent)
                    }
                    if (mine) stamp_node(t, y, now, sq);
                }
                out_key[i] = kmax - (uint32_t)hm;
                out_mlen[i] = hm;
                out_cov[i] = cov;
                // the token at the coverage; with no match (y < 0) the coverage
                // is 0 and the token is the request's first (its miss token)
                out_next[i] = cov < len ? (y > 0 ? tokc : htok) : -1;
                out_s0[i] = y > 0 ? S0 : -1;
                out_tok0[i] = htok;
                // the request keeps its key: K2 moves it with the previous order
                smark[r] = (stag << 32) | (int64_t)i;
            }
        }
    }
    // the unsettled positions: warp-aggregated append (any order; K2 sorts
    // them by (key, position)) and a per-position flag (K2's large path)
    if (i < n) slow_flag[i] = slow ? 1 : 0;
    const unsigned m = __ballot_sync(FS_FULL, i < n && slow);
    if (m) {
        const int lane = threadIdx.x & 31;
        int32_t base = 0;
        if (lane == __ffs(m) - 1) base = atomicAdd(&oc->njobs, __popc(m));
        base = __shfl_sync(FS_FULL, base, __ffs(m) - 1);
        if (i < n && slow) jobs[base + __popc(m & ((1u << lane) - 1))] = (int32_t)i;
    }
}

// Batch completion: unpin every finished path (worker.py:209-213), one warp
// per path.  The decrements commute; each node releases its edge from
// pinned_tokens when its count reaches zero (radix.py:180-185).
__global__ void k_unpin_many(TrieView t, const int32_t *__restrict__ nodes, int64_t n, int64_t *out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const int32_t nd = nodes[i];
    if (nd <= 0) return;
    warp_unpin_path(t, nd, lane);
    if (lane == 0 && t.sc->status == FS_ERR_UNDERFLOW) out[0] = FS_ERR_UNDERFLOW;
}

// ---------------------------------------------------------------- queue upkeep
// Stable merge of the label-ordered queue `a` with the label-ordered arrivals `b`.
__global__ void k_merge(const int32_t *__restrict__ a, int32_t na, const int32_t *__restrict__ b,
                        const int64_t *__restrict__ lb, int32_t nb, const int64_t *__restrict__ rlabel,
                        int32_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < na) {
        const int64_t la = rlabel[a[i]];
        int32_t lo = 0, hi = nb;
        while (lo < hi) { const int32_t m = (lo + hi) >> 1; if (lb[m] < la) lo = m + 1; else hi = m; }
        out[i + lo] = a[i];
    } else if (i < (int64_t)na + nb) {
        const int32_t k = (int32_t)(i - na);
        const int64_t l = lb[k];
        int32_t lo = 0, hi = na;
        while (lo < hi) { const int32_t m = (lo + hi) >> 1; if (rlabel[a[m]] < l) lo = m + 1; else hi = m; }
        out[k + lo] = b[k];
    }
}

// Gather per-sorted-position scheduler slots: {client, cov, next token, state}.
__global__ void k_gather(const int32_t *__restrict__ perm, const int32_t *__restrict__ queue, int32_t n,
                         const int32_t *__restrict__ cov, const int32_t *__restrict__ next,
                         const int32_t *__restrict__ mlen, const int64_t *__restrict__ s0,
                         const int32_t *__restrict__ rclient, const int32_t *__restrict__ rlen,
                         int32_t *__restrict__ s_req, int4 *__restrict__ slot, int32_t *__restrict__ s_len,
                         int32_t *__restrict__ s_mlen0, int64_t *__restrict__ s_src0,
                         const int32_t *__restrict__ tok0, int32_t *__restrict__ s_tok0) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int32_t qi = perm[p];
    const int32_t r = queue[qi];
    const int32_t len = rlen[r];
    const int32_t m0 = mlen[qi];
    s_req[p] = r;
    s_len[p] = len;
    slot[p] = make_int4(rclient[r], cov[qi], next[qi], 0);
    s_mlen0[p] = m0;
    s_tok0[p] = tok0[qi];  // first token the step-start trie misses (K1)
    s_src0[p] = s0[qi];
}

// ---------------------------------------------------------------- K3 + K4
struct FillArgs {
    TrieView t;
    int32_t n;
    const int32_t *s_req;
    int4 *slot;  // {client, cov(B), next token, state: >=0 pending w/ exact-epoch, -1 admitted}
    const int32_t *s_len;
    const int32_t *s_mlen0;  // K1 match length and last chain (admission-walk hint)
    const int32_t *s_tok0;   // token at s_mlen0 (-1 when fully matched): the miss key
    const int64_t *s_src0;
    const int64_t *roff;
    int64_t *q, *refills;
    const uint8_t *known;
    int32_t nclients;
    int32_t *pend_cnt;
    const int32_t *dl_client;  // on_outputs deltas to apply first
    const int64_t *dl_delta;
    int32_t ndl;
    int64_t M, R, gen_total, headroom0, w_e, quantum, now;
    int64_t sq_base;  // operation sequence number of admission e = sq_base + e
    int32_t lpm;
    Seg *segs;
    int32_t *adm_req, *adm_mlen, *adm_node;
    int64_t *adm_unp, *adm_pinb, *adm_rec_end;
    int32_t adm_cap;
    int8_t *rstate;
    int64_t *hdr;  // [n_adm, n_rec, status, epochs, refill_events, resumes, -, -, prof[8]]
    // grid sweep (see k_schedule): helper CTAs 1..nhelp, control block, filter mirror
    struct SweepCtl *ctl;
    unsigned long long *gkey;
    int32_t *gep;
    int32_t nhelp;
    int32_t local_chunks;  // chunks the leader scans before a grid sweep
    int32_t *rw_list;      // grid re-walk list (FS_CHUNK entries, -1 = skip)
    int32_t hbase;         // blockIdx of the first sweep helper (2 when CTA 1 is the evictor)
    // asynchronous cold eviction (FevCtl in fs_device.cuh): CTA 1 evicts
    int32_t fev, fev_cap, fev_tag;
    FevCtl *fev_ctl;
    void *fev_vrec;  // FEV_MAXC FevRec: the cold leaves in pop order
    int64_t *fev_need, *fev_rec_end;
    int32_t *fev_free;
};
#define FS_GRID_REWALK 96  // leader re-walk lists longer than this go to the helpers

// Control block of one fill's grid sweeps, written by the leader CTA and read
// by the helpers (release/acquire at gpu scope; reset by the host per fill).
struct SweepCtl {
    int32_t seq;       // sweep number; -1 releases the helpers
    int32_t from, until, any_mode, epoch, result, done, saturated;
    int32_t kind, nlist, pad2_;  // kind 0: sweep [from, until); 1: re-walk rw_list[0, nlist)
    int64_t slack, resumes, chunks, pad_;
    TrieScalars sc;    // the leader's trie scalars at the sweep
};


// (pinned coverage B, token at B) of every admission of this step -> latest
// admission epoch.  An admission e can raise a queued request's B only if
// both match (see block_find); open addressing in shared memory.

struct AdmFilter {
    unsigned long long key[FS_FSLOTS];
    int32_t ep[FS_FSLOTS];
    int32_t n;
    int32_t saturated;  // too many distinct keys: every stale B is re-walked
};

__device__ __forceinline__ unsigned long long adm_key(int32_t B, int32_t tok) {
    return ((unsigned long long)(uint32_t)B << 32) | (uint32_t)tok;
}

// Miss keys share the table, tagged by bit 63 (depths are < 2^31).
// Upper bound on any queued request's coverage during a fill: the trie at any
// point of the fill holds only strings that were in it at step start or are
// prefixes of requests admitted since, so B_p <= mlen_p <= max(mlen0_p,
// max_e LCP(p, e)).  LCP(p, e) > mlen0_p needs p[:mlen0_p+1] == e[:mlen0_p+1];
// that string was absent at step start while p[:mlen0_p] was present, so e's
// own step-start match ended at the same depth: mlen0_e == mlen0_p and
// tok0_e == tok0_p.  With no admission carrying p's miss key, B_p <= mlen0_p.
__device__ __forceinline__ unsigned long long miss_key(int32_t m0, int32_t tok) {
    return ((unsigned long long)((uint32_t)m0 | 0x80000000u) << 32) | (uint32_t)tok;
}

// Read-only view of the filter: the leader's shared-memory table, or its
// global mirror for the helper CTAs of a grid sweep.
struct FiltView {
    const unsigned long long *key;
    const int32_t *ep;
    int32_t saturated;
};

__device__ __forceinline__ FiltView filt_view(const AdmFilter *f) { return FiltView{f->key, f->ep, f->saturated}; }

// Returns the slot written (-1: saturated).  The global mirror (read by the
// helper CTAs' sweeps and the next fill's K1) is written by the caller, off
// the admission's critical warp (block_admit, after the insert).
__device__ inline int32_t adm_put_key(AdmFilter *f, unsigned long long k, int32_t e) {
    if (f->n * 2 >= FS_FSLOTS) { f->saturated = 1; return -1; }
    uint32_t i = fs_hmix(k) & (FS_FSLOTS - 1);
    while (f->key[i] != FS_HEMPTY && f->key[i] != k) i = (i + 1) & (FS_FSLOTS - 1);
    if (f->key[i] == FS_HEMPTY) { f->key[i] = k; f->n++; }
    f->ep[i] = e;
    return (int32_t)i;
}

__device__ inline void adm_put(AdmFilter *f, int32_t B, int32_t tok, int32_t m0, int32_t tok0, int32_t e,
                               int32_t *slots2) {
    // a request fully covered by pins extends nothing
    slots2[0] = tok >= 0 ? adm_put_key(f, adm_key(B, tok), e) : -1;
    slots2[1] = tok0 >= 0 ? adm_put_key(f, miss_key(m0, tok0), e) : -1;
}

// true when some admission in [since, now) had key k
__device__ __forceinline__ bool adm_maybe_key(const FiltView &f, unsigned long long k, int32_t since) {
    if (f.saturated) return true;
    uint32_t i = fs_hmix(k) & (FS_FSLOTS - 1);
    while (true) {
        const unsigned long long x = f.key[i];
        if (x == k) return f.ep[i] >= since;
        if (x == FS_HEMPTY) return false;
        i = (i + 1) & (FS_FSLOTS - 1);
    }
}

// true when some admission in [since, now) had the same (B, token)
__device__ __forceinline__ bool adm_maybe(const FiltView &f, int32_t B, int32_t tok, int32_t since) {
    if (tok < 0) return false;
    return adm_maybe_key(f, adm_key(B, tok), since);
}

// Can position p's exact coverage reach len - slack at all this fill?  False
// only when the miss-key bound (above) rules it out; slack never grows within
// a fill, so such a request needs no re-walk until its miss key is admitted.
__device__ __forceinline__ bool cov_may_reach(const FillArgs &a, const FiltView &f, int32_t p, int64_t slack) {
    const int32_t m0 = a.s_mlen0[p];
    if (a.s_len[p] - m0 <= slack) return true;
    const int32_t t0 = a.s_tok0[p];
    return t0 >= 0 && adm_maybe_key(f, miss_key(m0, t0), 0);
}

struct SchedSmem {
    InsertSmem ins;
    ChunkLRU lru;
    AdmFilter flt;
    int32_t wl[FS_CHUNK];
    int64_t red64[32];
    int32_t red32[32];
    int32_t wl_n, minA, minB;
    int32_t cursor, progress, epoch, npos, nadm, stop, j, cursor_seq;
    int32_t pre_j, pre_end;  // next-candidate prescan of the last admission (block_admit)
    Seg pseg[FS_PRE_SEGS];    // ... and the segments of that candidate's step-start match
    int32_t pseg_j, pseg_n;   // (queue position, count; -1: none)
    int64_t headroom, slack_at;
    int64_t resumes, refill_events;
    int64_t prof[16];  // cycles: [0] find, [1] walk, [2] evict, [3] admit tail; [4] chunks, [5] pops,
                       // [6] chains, [7] total, [8..10] pop argmin / edit / rescan, [11] setup
    FevLeader fev;
    int64_t prof2[8];  // cycles: [0] pin (warps 2..), [1] on_walk (thread 32), [2] order posts waiting for the evictor's setup
};

__device__ __forceinline__ int64_t sched_slack(const FillArgs &a, int64_t headroom) {
    const int64_t pinned = a.t.sc->pinned;
    int64_t s = a.M - a.gen_total - headroom - a.R - pinned;  // worker.py:104-107
    const int64_t cap = a.t.sc->capacity;
    if (cap > 0 && cap - pinned < s) s = cap - pinned;        // worker.py:108-109
    return s;
}

__device__ inline int32_t block_min_i32(int32_t v, int32_t *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_down_sync(FS_FULL, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? red[lane] : FS_NONE;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_down_sync(FS_FULL, v, o));
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

__device__ inline int64_t block_sum_i64(int64_t v, int64_t *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FS_FULL, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FS_FULL, v, o);
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

__device__ inline int64_t block_min_i64(int64_t v, int64_t *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, (int64_t)__shfl_down_sync(FS_FULL, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? red[lane] : INT64_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = min(v, (int64_t)__shfl_down_sync(FS_FULL, v, o));
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

// Exact pinned coverage B of a queued request (re-walk; only reached through
// the filter in block_find).  One warp.
__device__ inline void warp_resume(const FillArgs &a, int32_t p, int lane) {
    const TrieView &t = a.t;
    const int32_t r = a.s_req[p];
    const int32_t len = a.s_len[p];
    const int32_t *rq = t.arena + a.roff[r];
    const int32_t m0 = a.s_mlen0[p];
    const int64_t S0 = a.s_src0[p];
    int32_t cov;
    int32_t y = -1;
    if (m0 > 0) {
        const int32_t c = t.pos[S0 + m0 - 1];
        if (pos_valid(t, c, S0, m0 - 1)) y = c;
    }
    auto none = [](int64_t, int32_t, int32_t, int32_t) {};
    if (y < 0) {
        cov = warp_walk<8>(t, rq, len, lane, nullptr, true).cov;
    } else {
        // the step-start match still holds: coverage of its prefix from the
        // deep end, then continue past a node boundary (inserts of this step)
        cov = warp_cov_from_deepest(t, y, m0, lane);
        if (cov == m0 && m0 == t.end[y] && m0 < len) {
            WalkStart st;
            st.node = y; st.idx = m0; st.nseg = 0; st.last = y; st.cov = cov; st.pinrun = true;
            cov = warp_walk_from<8>(t, rq, len, lane, true, st, none).cov;
        }
    }
    if (lane == 0) {
        a.slot[p].y = cov;
        a.slot[p].z = cov < len ? rq[cov] : -1;
    }
}

// First sorted position p in [from, until) that is pending and, unless
// any_mode, passes the deficit gate (q > 0, skipped for LPM) and the budget
// test len - B <= slack with B exact.  B only grows inside a fill, and an
// admission `e` can raise B_p only if B_p == B_e and the request's token at
// B_p equals the admitted one's (LCP(r_p, r_e) > B_p forces both), so a stale
// B is re-walked only when such an admission happened since it was exact.
#define FS_FAST 256

// Warp-0 scan of [from, wend) in order; returns the first qualifying position
// or FS_NONE.  Same predicate and resume rule as the block-wide scan.
__device__ inline int32_t warp_find_window(const FillArgs &a, SchedSmem *sm, int32_t from, int32_t wend,
                                           bool any_mode, int64_t slack, int lane) {
    // 4 x 32 positions per round: all slot loads, then all counter / length
    // loads, then the in-order verdicts -- 2 memory round trips per 128
    // positions instead of 2 per 32
    constexpr int K = 4;
    const int32_t epoch = sm->epoch;
    for (int32_t base = from; base < wend; base += 32 * K) {
        int4 sv[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int32_t p = base + 32 * k + lane;
            sv[k] = p < wend ? a.slot[p] : make_int4(0, 0, 0, -1);
        }
        bool gate[K];
        int32_t need[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int32_t p = base + 32 * k + lane;
            gate[k] = sv[k].w >= 0 && (any_mode || a.lpm || a.q[sv[k].x] > 0);
            need[k] = gate[k] && !any_mode ? a.s_len[p] - sv[k].y : 0;
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int32_t p = base + 32 * k + lane;
            bool q = false, r = false;
            if (gate[k]) {
                if (any_mode || need[k] <= slack) {
                    q = true;
                } else if (sv[k].w < epoch) {
                    const FiltView fv = filt_view(&sm->flt);
                    if (!adm_maybe(fv, sv[k].y, sv[k].z, sv[k].w)) a.slot[p].w = epoch;
                    else if (cov_may_reach(a, fv, p, slack)) r = true;
                }
            }
            const unsigned mq = __ballot_sync(FS_FULL, q), mr = __ballot_sync(FS_FULL, r);
            if (mq | mr) {
                const int first = __ffs(mq | mr) - 1;
                if ((mq >> first) & 1u) return base + 32 * k + first;
                // a stale coverage must be re-walked first: hand the rest of the
                // search to the block, whose 32 warps re-walk in parallel
                return -(base + 32 * k + first) - 2;
            }
        }
    }
    return FS_NONE;
}

// One FS_CHUNK-position chunk [base, min(base+FS_CHUNK, until)) by the whole
// block: the first qualifying position, after re-walking the stale coverages
// that precede the chunk's first plain hit.  `sm` supplies the block's scratch
// (wl, red32, minB); the leader and the helper CTAs both run this.
__device__ int32_t grid_rewalk(const FillArgs &a, SchedSmem *sm, int32_t nlist, int64_t slack);

__device__ int32_t chunk_scan(const FillArgs &a, SchedSmem *sm, const FiltView &fv, int32_t base, int32_t until,
                              bool any_mode, int64_t slack, int32_t epoch, unsigned long long *resumes,
                              bool leader = false) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    if (tid == 0) { sm->wl_n = 0; sm->minB = FS_NONE; }
    __syncthreads();
    int32_t mine = FS_NONE;
#pragma unroll
    for (int u = 0; u < FS_ITEMS; u++) {
        const int32_t p = base + u * FS_SCHED_THREADS + tid;
        if (p >= until || mine != FS_NONE) continue;
        const int4 s = a.slot[p];
        if (s.w < 0) continue;
        if (any_mode) { mine = p; continue; }
        if (!a.lpm && a.q[s.x] <= 0) continue;
        const int32_t need = a.s_len[p] - s.y;
        if (need <= slack) { mine = p; continue; }
        if (s.w < epoch) {
            if (!adm_maybe(fv, s.y, s.z, s.w)) a.slot[p].w = epoch;  // B is still exact
            else if (cov_may_reach(a, fv, p, slack)) sm->wl[atomicAdd(&sm->wl_n, 1)] = p;
        }
    }
    const int32_t minA = block_min_i32(mine, sm->red32);
    if (leader && a.nhelp > 0 && sm->wl_n > FS_GRID_REWALK) {
        // many stale coverages before the first plain hit: the helper CTAs
        // re-walk them (a warp each) instead of the leader's 32 warps
        const int32_t nw = sm->wl_n;
        for (int32_t i = tid; i < nw; i += blockDim.x) a.rw_list[i] = sm->wl[i] < minA ? sm->wl[i] : -1;
        const int32_t mb = grid_rewalk(a, sm, nw, slack);
        __syncthreads();
        return min(minA, mb);
    }
    if (sm->wl_n > 0) {
        for (int32_t i = warp; i < sm->wl_n; i += nwarps) {
            const int32_t p = sm->wl[i];
            if (p >= minA) continue;
            warp_resume(a, p, lane);
            __syncwarp();
            if (lane == 0) {
                a.slot[p].w = epoch;
                if (a.s_len[p] - a.slot[p].y <= slack) atomicMin(&sm->minB, p);
                atomicAdd(resumes, 1ull);
            }
        }
        __syncthreads();
    }
    const int32_t best = min(minA, sm->minB);
    __syncthreads();
    return best;
}

// Leader side of a grid sweep: publish the search, wait for the helpers,
// return the first qualifying position in [from, until) (FS_NONE if none).
__device__ int32_t grid_sweep(const FillArgs &a, SchedSmem *sm, int32_t from, int32_t until, bool any_mode,
                              int64_t slack) {
    SweepCtl *c = a.ctl;
    __threadfence();  // this thread's trie / slot / counter writes, before the release
    __syncthreads();
    if (threadIdx.x == 0) {
        sm->cursor_seq++;
        c->kind = 0;
        c->from = from; c->until = until; c->any_mode = any_mode; c->epoch = sm->epoch;
        c->slack = slack; c->result = FS_NONE; c->done = 0; c->saturated = sm->flt.saturated;
        c->sc = *a.t.sc;
        __threadfence();
        st_release_i32(&c->seq, sm->cursor_seq);
        while (ld_acquire_i32(&c->done) < a.nhelp) __nanosleep(64);
        sm->minA = ld_acquire_i32(&c->result);
    }
    __syncthreads();
    (void)ld_acquire_i32(&c->done);  // every thread: drop L1 lines the helpers made stale
    const int32_t r = sm->minA;
    __syncthreads();
    return r;
}

// Leader side of a grid re-walk: the helpers' warps re-walk a.rw_list[0, n)
// (warp_resume: exact coverage), refresh those slots and return the first
// position that passes the budget test (FS_NONE if none).
__device__ int32_t grid_rewalk(const FillArgs &a, SchedSmem *sm, int32_t nlist, int64_t slack) {
    SweepCtl *c = a.ctl;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        sm->cursor_seq++;
        c->kind = 1; c->nlist = nlist; c->epoch = sm->epoch; c->slack = slack;
        c->result = FS_NONE; c->done = 0;
        c->sc = *a.t.sc;
        __threadfence();
        st_release_i32(&c->seq, sm->cursor_seq);
        while (ld_acquire_i32(&c->done) < a.nhelp) __nanosleep(64);
        sm->minA = ld_acquire_i32(&c->result);
    }
    __syncthreads();
    (void)ld_acquire_i32(&c->done);  // every thread: drop L1 lines the helpers made stale
    const int32_t r = sm->minA;
    __syncthreads();
    return r;
}

// Helper CTA: serve grid sweeps until the leader releases it.  Chunks are
// dealt round-robin; a helper stops at chunks past the best position found so
// far (the minimum over the grid is the sequential scan's first hit, because
// each position's verdict depends only on the state the leader published).
__device__ void helper_loop(const FillArgs &ap, SchedSmem *sm) {
    __shared__ FillArgs a;
    __shared__ TrieScalars sc;
    __shared__ int32_t seq_sh;
    SweepCtl *c = ap.ctl;
    const int tid = threadIdx.x;
    const int32_t h = blockIdx.x - ap.hbase;
    int32_t last = 0;
    if (tid == 0) { a = ap; a.t.sc = &sc; }
    while (true) {
        if (tid == 0) {
            int32_t v;
            while ((v = ld_acquire_i32(&c->seq)) == last) __nanosleep(128);
            seq_sh = v;
        }
        __syncthreads();
        const int32_t v = seq_sh;
        if (v < 0) return;
        last = v;
        (void)ld_acquire_i32(&c->seq);  // every thread: fresh view of the leader's writes
        if (tid < (int)(sizeof(TrieScalars) / 8))
            reinterpret_cast<int64_t *>(&sc)[tid] = reinterpret_cast<volatile int64_t *>(&c->sc)[tid];
        __syncthreads();
        const int32_t from = c->from, until = c->until, epoch = c->epoch;
        const bool any_mode = c->any_mode;
        const int64_t slack = c->slack;
        const FiltView fv{a.gkey, a.gep, c->saturated};
        int32_t best = FS_NONE;
        int64_t nch = 0;
        if (c->kind == 1) {
            // re-walk list: one warp per entry
            const int lane = tid & 31;
            const int32_t nlist = c->nlist;
            const int32_t gw = h * (int32_t)(blockDim.x >> 5) + (tid >> 5);
            const int32_t nw = a.nhelp * (int32_t)(blockDim.x >> 5);
            unsigned long long nres = 0;
            for (int32_t i = gw; i < nlist; i += nw) {
                const int32_t p = a.rw_list[i];
                if (p < 0) continue;
                warp_resume(a, p, lane);
                __syncwarp();
                if (lane == 0) {
                    a.slot[p].w = epoch;
                    if (a.s_len[p] - a.slot[p].y <= slack) atomicMin(&c->result, p);
                    nres++;
                }
            }
            if (lane == 0 && nres) atomicAdd((unsigned long long *)&c->resumes, nres);
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(&c->done, 1);
            continue;
        }
        for (int64_t base = from + (int64_t)h * FS_CHUNK; base < until; base += (int64_t)a.nhelp * FS_CHUNK) {
            if (tid == 0) sm->minA = *(volatile int32_t *)&c->result;
            __syncthreads();
            const bool skip = sm->minA <= base;
            __syncthreads();
            if (skip) break;
            nch++;
            best = chunk_scan(a, sm, fv, (int32_t)base, until, any_mode, slack, epoch,
                              (unsigned long long *)&c->resumes);
            if (best != FS_NONE) {
                if (tid == 0) atomicMin(&c->result, best);
                break;
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            atomicAdd((unsigned long long *)&c->chunks, (unsigned long long)nch);
            __threadfence();
            atomicAdd(&c->done, 1);
        }
    }
}


// CTA 1 under FEV (see FevCtl, fs_device.cuh).  Setup (whole CTA): collect
// the cold evictable leaves, sort them by the LRU key (last_access, seq)
// (radix.py:210-219) and lay their node fields out in that order; publish the
// cold supply.  Then warp 0 performs the leader's eviction needs in order:
// each pop is the smaller of the next sorted cold leaf and the top of a heap
// of parents that became leaves (radix.py:231-239) -- no index rescans -- and
// the detach (record, child-hash tombstone, parent child count and stamp,
// free slot; radix.py:206-208, 226-249) is issued with its loads overlapped
// (the records ahead are prefetched into L1; the hash probe is warp-wide).
#define FEV_MAXC 2048  // power of two (bitonic sort)
#define FEV_HEAP 640
#ifndef FS_FEV_CHECK
#define FS_FEV_CHECK 0
#endif
struct FevRec {
    int64_t src, la, lseq, seq;
    int32_t start, end, parent, first, node, pad_;
};
struct FevSmem {
    int64_t la[FEV_MAXC];
    int64_t sq[FEV_MAXC];
    int32_t id[FEV_MAXC];
    FevRec heap[FEV_HEAP];  // parents that became leaves, min-heap by (la, seq)
    int32_t hn, nc, bad, tr_i, tr_end;
    unsigned long long cold_tok;
};

__device__ __forceinline__ bool fev_less(int64_t a1, int64_t s1, int64_t a2, int64_t s2) {
    return a1 < a2 || (a1 == a2 && s1 < s2);
}
__device__ __forceinline__ void st_relaxed_i64(int64_t *p, int64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_relaxed_i64(const int64_t *p) {
    int64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ void fev_heap_push(FevSmem *e, const FevRec &r, FevCtl *ctl) {
    if (e->hn >= FEV_HEAP) { ctl->err = 1; return; }
    int32_t i = e->hn++;
    while (i > 0) {
        const int32_t p = (i - 1) >> 1;
        if (!fev_less(r.la, r.seq, e->heap[p].la, e->heap[p].seq)) break;
        e->heap[i] = e->heap[p];
        i = p;
    }
    e->heap[i] = r;
}
__device__ void fev_heap_pop(FevSmem *e) {
    const FevRec last = e->heap[--e->hn];
    int32_t i = 0;
    while (true) {
        int32_t c = 2 * i + 1;
        if (c >= e->hn) break;
        if (c + 1 < e->hn && fev_less(e->heap[c + 1].la, e->heap[c + 1].seq, e->heap[c].la, e->heap[c].seq)) c++;
        if (!fev_less(e->heap[c].la, e->heap[c].seq, last.la, last.seq)) break;
        e->heap[i] = e->heap[c];
        i = c;
    }
    if (e->hn > 0) e->heap[i] = last;
}

__device__ void evictor_loop(const FillArgs &ap, unsigned char *smraw) {
    static_assert(sizeof(FevSmem) <= sizeof(SchedSmem), "evictor state must fit the scheduler's shared memory");
    FevSmem *e = reinterpret_cast<FevSmem *>(smraw);
    const TrieView &t = ap.t;
    FevCtl *ctl = ap.fev_ctl;
    FevRec *vrec = reinterpret_cast<FevRec *>(ap.fev_vrec);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t hw0 = t.sc->hw;  // the global scalars are the step-start ones during the fill
    if (tid == 0) { e->hn = 0; e->nc = 0; e->bad = 0; e->cold_tok = 0; e->tr_i = -1; e->tr_end = 0; }
    __syncthreads();
    // cold evictable leaves: own stamp before this fill's K1 stamps (sq1); every
    // pre-fill stamp must be older than `now` so cold keys sort first
    const int64_t sq1 = ap.sq_base - 1;
    {
        unsigned long long c = 0;
        int b = 0;
        for (int32_t n = 1 + tid; n < hw0; n += blockDim.x) {
            if (!(t.flags[n] & FS_ALIVE) || t.lseq[n] >= sq1) continue;
            const int64_t la = t.la[n];
            if (la >= ap.now) b = 1;
            if (t.nchild[n] == 0 && t.ref[n] == 0) {
                c += (unsigned long long)(t.end[n] - t.start[n]);
                const int32_t k = atomicAdd(&e->nc, 1);
                if (k < FEV_MAXC) { e->la[k] = la; e->sq[k] = t.seq[n]; e->id[k] = n; }
            }
        }
        if (c) atomicAdd(&e->cold_tok, c);
        if (b) e->bad = 1;
    }
    __syncthreads();
    const int32_t nc = e->nc;
    const bool ok = !e->bad && nc <= FEV_MAXC;
    if (ok) {
        // bitonic sort of the cold leaves by (la, seq), padded to a power of two
        int32_t P2 = 1;
        while (P2 < nc) P2 <<= 1;
        for (int32_t i = nc + tid; i < P2; i += blockDim.x) { e->la[i] = INT64_MAX; e->sq[i] = INT64_MAX; e->id[i] = -1; }
        __syncthreads();
        for (int32_t k = 2; k <= P2; k <<= 1) {
            for (int32_t j = k >> 1; j > 0; j >>= 1) {
                for (int32_t i = tid; i < P2; i += blockDim.x) {
                    const int32_t l = i ^ j;
                    if (l > i) {
                        const bool up = (i & k) == 0;
                        const bool gt = fev_less(e->la[l], e->sq[l], e->la[i], e->sq[i]);
                        if (gt == up) {
                            int64_t x = e->la[i]; e->la[i] = e->la[l]; e->la[l] = x;
                            x = e->sq[i]; e->sq[i] = e->sq[l]; e->sq[l] = x;
                            const int32_t y = e->id[i]; e->id[i] = e->id[l]; e->id[l] = y;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // node fields in pop order (one or two L1 lines per pop, prefetched ahead)
        for (int32_t i = tid; i < nc; i += blockDim.x) {
            const int32_t n = e->id[i];
            FevRec r;
            r.src = t.src[n]; r.la = e->la[i]; r.lseq = t.lseq[n]; r.seq = e->sq[i];
            r.start = t.start[n]; r.end = t.end[n]; r.parent = t.parent[n]; r.first = t.first[n];
            vrec[i] = r;
        }
    }
    __syncthreads();
    if (tid == 0) {
        ctl->C = ok ? (int64_t)e->cold_tok : -1;
        ctl->ok = ok;
        __threadfence();
        st_release_i32(&ctl->ready, 1);
    }
    if (warp != 0) return;
    // ---- pops (warp 0)
    const int64_t tag = (int64_t)ap.fev_tag << 40;
    const int64_t low = (1ll << 40) - 1;
    int32_t k = 0, i = 0, nfreed = 0, hhw = 0;
    int64_t freed_tot = 0, nrec = 0, tombs = 0, pops = 0;
    while (true) {
        int64_t v = 0;
        if (lane == 0) {
            while (true) {
                v = ld_relaxed_i64(ap.fev_need + k);
                if ((v & ~low) == tag) break;
                if (ld_acquire_i32(&ctl->stop)) {
                    v = ld_relaxed_i64(ap.fev_need + k);
                    if ((v & ~low) != tag) v = 0;
                    break;
                }
                __nanosleep(20);
            }
        }
        v = __shfl_sync(FS_FULL, v, 0);
        if (v == 0) break;
        const int64_t need = v & low;
        int64_t freed = 0;
        while (freed < need) {
            // the next pop: the sorted cold leaf or the heap's re-joined parent
            const bool hs = e->hn > 0, ss = i < nc;
            if (!hs && !ss) { if (lane == 0) ctl->err = 1; break; }
            const bool from_heap = hs && (!ss || fev_less(e->heap[0].la, e->heap[0].seq, e->la[i], e->sq[i]));
            if (lane >= 1 && lane <= 8 && i + lane < nc) pf_l1(vrec + i + lane);
            FevRec r = from_heap ? e->heap[0] : vrec[i];
            if (!from_heap) {
                r.node = e->id[i];
                if (e->tr_i == i) r.end = e->tr_end;  // truncated by an earlier order
            }
            const int32_t el = r.end - r.start;
            const int64_t rem = need - freed;
            pops++;
#if FS_FEV_CHECK
            if (lane == 0) {
                // the popped node must still be an unpinned live leaf with the
                // fields the setup read (debug: FEV is opt-in while this is open)
                const int32_t nc = atomicAdd(&t.nchild[r.node], 0), rf = atomicAdd(&t.ref[r.node], 0);
                const uint8_t fl = *(volatile uint8_t *)&t.flags[r.node];
                const int32_t pa = *(volatile int32_t *)&t.parent[r.node];
                const int32_t st = *(volatile int32_t *)&t.start[r.node], en = *(volatile int32_t *)&t.end[r.node];
                int code = 0;
                if (!(fl & FS_ALIVE)) code = 2;
                else if (nc != 0) code = 3;
                else if (rf != 0) code = 4;
                else if (pa != r.parent) code = 5;
                else if (st != r.start) code = 6;
                else if (en != r.end) code = 7;
                if (code && !ctl->err) { ctl->err = code; ctl->nc = r.node; ctl->heap_hw = from_heap ? 1 : 0; }
            }
#endif
            if (el <= rem) {
                // whole leaf: record, tombstone (parent, first), parent child
                // count and stamp, free the slot (radix.py:226-230, 206-208)
                const int32_t P = r.parent;
                const uint64_t key = fs_hkey(P, r.first);
                const uint32_t h0 = fs_hmix(key) & t.hmask;
                int32_t old = 0;
                uint8_t flP = 0;
                int32_t refP = 0;
                int64_t laP = 0, lsP = 0, sqP = 0, srcP = 0;
                int32_t stP = 0, enP = 0, paP = 0, fiP = 0;
                if (lane == 0) {
                    old = atomicSub(&t.nchild[P], 1);
                    // P's fields from L2, not this SM's L1: the setup scan cached
                    // every node's line, and the leader pins and stamps during the
                    // fill (a stale ref or stamp would make a pinned, freshly
                    // stamped parent look like a cold candidate)
                    flP = *(volatile uint8_t *)&t.flags[P]; refP = *(volatile int32_t *)&t.ref[P];
                    laP = *(volatile int64_t *)&t.la[P]; lsP = *(volatile int64_t *)&t.lseq[P];
                    sqP = t.seq[P];
                    srcP = t.src[P]; stP = *(volatile int32_t *)&t.start[P]; enP = *(volatile int32_t *)&t.end[P];
                    paP = *(volatile int32_t *)&t.parent[P]; fiP = *(volatile int32_t *)&t.first[P];
                }
                // warp-wide probe of the child hash: the key's slot before the first empty one
                for (uint32_t base = 0; base <= t.hmask; base += 32) {
                    const uint32_t hi = (h0 + base + lane) & t.hmask;
                    const unsigned long long x = t.hslot[hi].x;
                    const unsigned mk = __ballot_sync(FS_FULL, x == key), me = __ballot_sync(FS_FULL, x == FS_HEMPTY);
                    const unsigned first_hit = mk ? __ffs(mk) - 1 : 32, first_empty = me ? __ffs(me) - 1 : 32;
                    if (first_hit < first_empty) {
                        if ((unsigned)lane == first_hit) t.hslot[hi].x = FS_HTOMB;
                        tombs++;
                        break;
                    }
                    if (me) break;
                }
                if (lane == 0) {
                    if (nrec < t.rcap) { t.rsrc[nrec] = r.src; t.rlen[nrec] = r.end; t.rkeep[nrec] = r.end - el; }
                    nrec++;
                    t.flags[r.node] = 0;
                    t.parent[r.node] = -2;
                    ap.fev_free[nfreed++] = r.node;
                    int64_t la2 = laP, ls2 = lsP;
                    if (P > 0 && r.lseq > lsP) { t.la[P] = r.la; t.lseq[P] = r.lseq; la2 = r.la; ls2 = r.lseq; }
                    if (from_heap) fev_heap_pop(e);
                    if (P > 0 && (flP & FS_ALIVE) && old - 1 == 0 && refP == 0) {
                        // the parent became a leaf: it joins the candidates at its key
                        FevRec q;
                        q.src = srcP; q.la = la2; q.lseq = ls2; q.seq = sqP;
                        q.start = stP; q.end = enP; q.parent = paP; q.first = fiP; q.node = P; q.pad_ = 0;
                        fev_heap_push(e, q, ctl);
                        hhw = max(hhw, e->hn);
                    }
                }
                if (!from_heap) i++;
                freed += el;
            } else {
                // truncate the leaf's tail (radix.py:240-246); it stays the minimum
                if (lane == 0) {
                    if (nrec < t.rcap) { t.rsrc[nrec] = r.src; t.rlen[nrec] = r.end; t.rkeep[nrec] = (int32_t)(r.end - rem); }
                    nrec++;
                    t.end[r.node] = r.end - (int32_t)rem;
                    if (from_heap) e->heap[0].end = r.end - (int32_t)rem;
                    else { e->tr_i = i; e->tr_end = r.end - (int32_t)rem; }
                }
                freed += rem;
            }
            __syncwarp();
        }
        if (lane == 0) {
            freed_tot += freed;
            if (freed != need) ctl->err = 1;
            ap.fev_rec_end[k] = nrec;
            __threadfence();
            st_release_i32(&ctl->done, k + 1);
        }
        k++;
        __syncwarp();
    }
    if (lane == 0) {
        ctl->freed = freed_tot;
        ctl->nrec = nrec;
        ctl->nfreed = nfreed;
        ctl->tombs = tombs;
        ctl->pops = pops;
        ctl->nc = nc;
        ctl->heap_hw = hhw;
        __threadfence();
        st_release_i32(&ctl->finished, 1);
    }
}

__device__ int32_t block_find(const FillArgs &a, SchedSmem *sm, int32_t from, int32_t until, bool any_mode,
                              int64_t slack) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long cw0 = clock64();
    {
        // the next admissible request is usually right after the cursor: one
        // warp checks a short window before the whole block sweeps chunks
        const int32_t wend = min(until, from + FS_FAST);
        if (warp == 0) {
            const int32_t r = warp_find_window(a, sm, from, wend, any_mode, slack, lane);
            if (lane == 0) sm->minA = r;
        }
        __syncthreads();
        const int32_t r = sm->minA;
        __syncthreads();
        (void)cw0;
        if (r >= 0 && r != FS_NONE) return r;
        from = r == FS_NONE ? wend : -(r + 2);
    }
    // the leader scans the next FS_LOCAL_CHUNKS chunks itself (a hit is usually
    // close), then hands the rest of the queue to the helper CTAs
    const FiltView fv = filt_view(&sm->flt);
    const int32_t local_end = a.nhelp > 0 ? min(until, from + a.local_chunks * FS_CHUNK) : until;
    const int32_t grid_from = local_end;
    for (int32_t base = from; base < local_end; base += FS_CHUNK) {
        if (tid == 0) sm->prof[4]++;
        const int32_t best = chunk_scan(a, sm, fv, base, min(until, base + FS_CHUNK), any_mode, slack, sm->epoch,
                                        (unsigned long long *)&sm->resumes, true);
        if (best != FS_NONE) return best;
    }
    if (grid_from < until) {
        const long long cg = clock64();
        const int32_t r = grid_sweep(a, sm, grid_from, until, any_mode, slack);
        if (threadIdx.x == 0) { sm->prof[15]++; sm->prof[14] += clock64() - cg; }  // grid sweeps, cycles
        return r;
    }
    return FS_NONE;
}

// Closed-form DLPM refill (local_policies.py:94-106, 116-120): rounds repeat
// until some pending client is positive, i.e. k = min over pending c of
// floor(-q_c/Q)+1; every client_list member with q <= 0 receives
// min(k, floor(-q_c/Q)+1) quanta.
__device__ void block_refill(const FillArgs &a, SchedSmem *sm) {
    const int tid = threadIdx.x;
    int64_t k = INT64_MAX;
    for (int32_t c = tid; c < a.nclients; c += blockDim.x)
        if (a.pend_cnt[c] > 0) k = min(k, (-a.q[c]) / a.quantum + 1);
    k = block_min_i64(k, sm->red64);
    for (int32_t c = tid; c < a.nclients; c += blockDim.x) {
        const int64_t qc = a.q[c];
        if (a.known[c] && qc <= 0) {
            const int64_t m = min(k, (-qc) / a.quantum + 1);
            a.q[c] = qc + m * a.quantum;
            a.refills[c] += m;
        }
    }
    __syncthreads();
    int64_t cnt = 0;
    for (int32_t c = tid; c < a.nclients; c += blockDim.x) cnt += (a.pend_cnt[c] > 0 && a.q[c] > 0);
    cnt = block_sum_i64(cnt, sm->red64);
    if (tid == 0) { sm->npos = (int32_t)cnt; sm->refill_events++; }
    __syncthreads();
}

// Worker.try_admit (worker.py:112-135) minus host bookkeeping -- probe,
// insert, pin (radix.py:187-192) -- then the policy's charge
// (local_policies.py:124).
// Worker.try_admit (worker.py:112-135) minus host bookkeeping -- probe,
// insert, pin (radix.py:187-192) -- then the policy's charge
// (local_policies.py:124).  The scheduler state this admission changes (the
// charge, pending counts, filter keys, epoch, headroom, pinned tokens) is
// settled as soon as the walk is done, so warp 1 can already search the next
// window for the following candidate while warp 0 evicts and warps 2.. pin.
__device__ void block_admit(const FillArgs &a, SchedSmem *sm, int32_t j, int64_t slack) {
    const int tid = threadIdx.x;
    const TrieView &t = a.t;
    // (every thread reads the condition before thread 0's hand-over clears
    // fev.on: a thread reading it afterwards would skip fev_drain's barriers)
    const bool fev_full = sm->fev.on && t.sc->hw + 2 > t.ncap;
    __syncthreads();
    if (fev_full) {
        // FEV allocates fresh node slots only (the evictor's freed slots come
        // back at the hand-over): out of fresh slots, hand over now
        fev_drain(t, &sm->fev, true);
        block_chunk_build(t, &sm->lru);
        if (tid == 0) sm->ins.lru = &sm->lru;
        __syncthreads();
    }
    const int32_t r = a.s_req[j];
    const int32_t len = a.s_len[j];
    const int64_t off = a.roff[r];
    __shared__ int64_t pinb;
    __shared__ int64_t pre_slack;
    __shared__ int32_t pre_ok;
    __shared__ int32_t mirror[2];  // filter slots this admission wrote (global mirror update below)
    // thread 0's charge operands do not depend on the tree edit: load them now
    // so they arrive while warp 0 walks
    int32_t c_pre = 0, pend_pre = 0, tok0_pre = -1, m0_pre = 0, b_pre = -1, tokb_pre = -1;
    int64_t q_pre = 0;
    if (tid == 0) {
        pinb = t.sc->pinned;
        sm->pre_j = -1;
        mirror[0] = mirror[1] = -1;
    }
    if (tid == 32) {  // on_walk runs on thread 32 (warp 1, lane 0)
        const int4 sl = a.slot[j];
        c_pre = sl.x;
        b_pre = sl.y;      // the coverage the search saw, and the token there
        tokb_pre = sl.z;
        pend_pre = a.pend_cnt[c_pre];
        q_pre = a.q[c_pre];
        m0_pre = a.s_mlen0[j];
        tok0_pre = a.s_tok0[j];
    }
    __syncthreads();
    const long long ct0 = clock64();
    auto on_walk = [&](int) {
        // thread 32: everything the next search depends on
        const long long cw = clock64();
        struct Acc { long long c; int64_t *p; __device__ ~Acc() { p[1] += clock64() - c; } } acc{cw, sm->prof2};
        const InsertSmem &in = sm->ins;
        pre_ok = 0;
        sm->pseg_j = -1;  // consumed by this walk (on_side may set the next one)
        if (in.status != FS_OK) return;
        const int32_t mlen = in.mlen;
        const int32_t cov = in.cov;
        const int64_t need = len - cov;
        t.sc->pinned += need;  // pinned_tokens grows by len - cov (the pin itself runs below)
        if (need > slack || in.unpinned != (int64_t)(mlen - cov)) {
            a.hdr[2] = FS_ERR_INTERNAL;  // closed-form budget test disagrees with can_add
            sm->stop = 1;
            return;
        }
        // the token at the coverage: known when the coverage is the search's
        // (slot) value or the step-start match length (K1's miss token)
        const int32_t tokc = cov >= len ? -1
                           : cov == b_pre ? tokb_pre
                           : (cov == m0_pre && tok0_pre >= 0) ? tok0_pre
                           : t.arena[off + cov];
        sm->prof2[3] += clock64() - cw;
        adm_put(&sm->flt, cov, tokc, m0_pre, tok0_pre, sm->epoch, mirror);
        sm->epoch++;
        sm->prof2[4] += clock64() - cw;
        a.slot[j].w = -1;
        a.rstate[r] = 2;
        const int32_t c = c_pre;
        const int32_t pend = pend_pre - 1;
        const int64_t qn = a.lpm ? q_pre : q_pre - a.w_e * (int64_t)(len - mlen);
        a.pend_cnt[c] = pend;
        if (!a.lpm) a.q[c] = qn;
        const bool was = pend_pre > 0 && q_pre > 0;
        const bool now_pos = pend > 0 && qn > 0;
        sm->npos += (int)now_pos - (int)was;
        sm->headroom += a.R;
        sm->progress = 1;
        pre_slack = sched_slack(a, sm->headroom);
        pre_ok = !(!a.lpm && sm->npos == 0);  // the next search needs no refill
    };
    auto on_side = [&](int lane) {
        // warp 1: the next search's first window (no tree reads; stale
        // coverages are reported, not re-walked)
        if (!pre_ok) return;
        const long long cs = clock64();
        const int32_t from = j + 1, wend = min(a.n, from + FS_FAST);
        const int32_t rr = from < wend ? warp_find_window(a, sm, from, wend, false, pre_slack, lane) : FS_NONE;
        if (lane == 0) { sm->pre_j = rr; sm->pre_end = wend; }
        // that candidate's matched path as source-chain segments, so its walk
        // starts without the chain hops.  Concurrent with warp 0's eviction,
        // which only detaches or truncates leaves: the ancestors of a node
        // are never touched, and a leaf touched here fails the walk's
        // pos_valid check of the hint, which then ignores these segments.
        int32_t ns = -1;
        if (rr >= 0 && rr != FS_NONE && a.s_mlen0[rr] > 0) {  // (negative: a stale coverage to re-walk)
            const int64_t S0 = a.s_src0[rr];
            const int32_t m0 = a.s_mlen0[rr];
            const int32_t y = t.pos[S0 + m0 - 1];
            if (pos_valid(t, y, S0, m0 - 1)) ns = warp_path_segments(t, y, m0, sm->pseg, lane, FS_PRE_SEGS);
#if FS_POP_PREFETCH
            if (ns > 0) {
                // warm L1 for that walk: the segments' end nodes' refs (the
                // coverage check) and the child slot of its next token
                if (lane < ns) {
                    const Seg g = sm->pseg[lane];
                    pf_l1(t.ref + t.pos[g.S + g.a]);
                    pf_l1(t.ref + t.pos[g.S + g.b - 1]);
                }
                if (lane == 0 && m0 == t.end[y]) {
                    const int32_t tok = a.s_tok0[rr];  // K1's token at m0 (-1: fully matched)
                    if (tok >= 0) pf_l1(t.hslot + (fs_hmix(fs_hkey(y, tok)) & t.hmask));
                }
            }
#endif
        }
        if (lane == 0) { sm->pseg_j = ns >= 0 ? rr : -1; sm->pseg_n = ns; sm->prof[12] += clock64() - cs; }
    };
    const bool have_pseg = sm->pseg_j == j;
    block_insert(t, off, len, a.now, a.sq_base + sm->epoch, -1, a.segs, &sm->ins, a.s_src0[j], a.s_mlen0[j], true,
                 on_walk, on_side, nullptr, have_pseg ? sm->pseg : nullptr, have_pseg ? sm->pseg_n : -1,
                 a.s_tok0[j]);
    if (tid == 0) {
        const InsertSmem &in = sm->ins;
        if (in.status != FS_OK) {
            a.hdr[2] = in.status;
            sm->stop = 1;
            sm->pre_j = -1;
        } else {
            const int32_t e = sm->nadm;
            if (e < a.adm_cap) {
                a.adm_req[e] = r;
                a.adm_mlen[e] = in.mlen;
                a.adm_unp[e] = in.unpinned;
                a.adm_pinb[e] = pinb;
                a.adm_node[e] = in.deepest;
                // under FEV the records of this admission are still being
                // written: keep the order count, resolved at the end of the fill
                a.adm_rec_end[e] = sm->fev.on ? -(int64_t)sm->fev.posted - 1 : t.sc->nrec;
            }
            sm->nadm = e + 1;
            if (t.sc->status != FS_OK) { a.hdr[2] = t.sc->status; sm->stop = 1; }
        }
        // the filter's global mirror (helpers' sweeps, next fill's K1 hints)
        for (int u = 0; u < 2; u++) {
            const int32_t i = mirror[u];
            if (i >= 0 && a.gkey) { a.gkey[i] = sm->flt.key[i]; a.gep[i] = sm->flt.ep[i]; }
        }
        sm->prof[3] += clock64() - ct0;
        sm->prof[6] += sm->ins.nseg;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(FS_SCHED_THREADS, 1) k_schedule(FillArgs ap) {
    extern __shared__ __align__(16) unsigned char fs_smraw[];
    SchedSmem &sm = *reinterpret_cast<SchedSmem *>(fs_smraw);
    // CTAs 1..nhelp (cooperative launch, co-resident) only serve the leader's
    // grid sweeps of the queue; CTA 0 runs the fill
    if (ap.fev && blockIdx.x == 1) { evictor_loop(ap, fs_smraw); return; }
    if (blockIdx.x > 0) { helper_loop(ap, &sm); return; }
    // the trie's scalars (used/pinned/seq/free stack/records) live in shared
    // memory for the whole step: every serial edit touches several of them
    __shared__ FillArgs a_sh;
    __shared__ TrieScalars sc_sh;
    const int tid = threadIdx.x;
    if (tid == 0) {
        a_sh = ap;
        sc_sh = *ap.t.sc;
        a_sh.t.sc = &sc_sh;
    }
    __syncthreads();
    const FillArgs &a = a_sh;
    // on_outputs deltas accumulated since the last fill (local_policies.py:130-133)
    if (tid == 0) {
        for (int32_t i = 0; i < a.ndl; i++) a.q[a.dl_client[i]] += a.dl_delta[i];
        a.t.sc->nrec = 0;
        a.hdr[2] = FS_OK;
        sm.cursor = 0; sm.progress = 0; sm.epoch = 0; sm.nadm = 0; sm.stop = 0;
        sm.headroom = a.headroom0; sm.resumes = 0; sm.refill_events = 0; sm.cursor_seq = 0;
        sm.pre_j = -1; sm.pre_end = 0; sm.pseg_j = -1; sm.pseg_n = -1;
        for (int i = 0; i < 16; i++) sm.prof[i] = 0;
        for (int i = 0; i < 8; i++) sm.prof2[i] = 0;
        for (int i = 0; i < 4; i++) sm.lru.prof[i] = 0;
        sm.ins.prof = sm.prof;
        sm.ins.prof2 = sm.prof2;
        sm.ins.lru = a.fev ? nullptr : &sm.lru;  // FEV: the evictor CTA owns the index
        sm.ins.lru_spare = &sm.lru;
        sm.ins.ev.pops = 0;
        sm.ins.fev = a.fev ? &sm.fev : nullptr;
        sm.ins.fev_switch = 0; sm.ins.fev_wait = 0;
        FevLeader &f = sm.fev;
        f.ctl = a.fev_ctl; f.need = a.fev_need; f.rec_end = a.fev_rec_end; f.free_list = a.fev_free;
        f.on = a.fev; f.posted = 0; f.cap_orders = a.fev_cap; f.ready_seen = 0; f.used_any = 0; f.stamped = 0;
        f.cum = 0; f.C = 0; f.tag = (int64_t)a.fev_tag << 40;
        f.nfree_saved = a.t.sc->nfree;
        if (a.fev) a.t.sc->nfree = 0;  // fresh slots only while the evictor frees concurrently
    }
    const long long t_start = clock64();
    // pend_cnt (pending requests per client) is maintained across fills:
    // +1 per arrival (k_enqueue_state), -1 per admission (block_admit)
    for (int32_t i = tid; i < FS_FSLOTS; i += blockDim.x) {
        sm.flt.key[i] = FS_HEMPTY;
        if (a.gkey) a.gkey[i] = FS_HEMPTY;
    }
    if (tid == 0) { sm.flt.n = 0; sm.flt.saturated = 0; }
    __syncthreads();
    if (!a.fev) block_chunk_build(a.t, &sm.lru);
    __syncthreads();
    {
        int64_t cnt = 0;
        for (int32_t c = tid; c < a.nclients; c += blockDim.x) cnt += (a.pend_cnt[c] > 0 && a.q[c] > 0);
        cnt = block_sum_i64(cnt, sm.red64);
        if (tid == 0) sm.npos = (int32_t)cnt;
    }
    __syncthreads();
    if (tid == 0) sm.prof[11] = clock64() - t_start;  // setup: LRU index, filter, counters
    // Dlpm.fill pass structure (local_policies.py:112-128): repeat passes over
    // the sorted snapshot until a whole pass admits nothing.
    while (true) {
        const bool ptrue = !a.lpm && sm.npos == 0;
        const int64_t slack = sched_slack(a, sm.headroom);
        const int32_t cur = sm.cursor;
        const int32_t pre = sm.pre_j;
        __syncthreads();
        const long long cf = clock64();
        int32_t j;
        if (pre >= 0 && pre != FS_NONE && !ptrue) {
            j = pre;  // the last admission's prescan already found it
        } else {
            // a clean prescan window needs no second look
            const int32_t from = (pre == FS_NONE && !ptrue) ? sm.pre_end : cur;
            j = from < a.n ? block_find(a, &sm, from, a.n, ptrue, slack) : FS_NONE;
        }
        if (tid == 0) { sm.prof[0] += clock64() - cf; sm.pre_j = -1; }
        if (j == FS_NONE) {
            if (sm.progress) {
                __syncthreads();
                if (tid == 0) { sm.cursor = 0; sm.progress = 0; }
                __syncthreads();
                continue;
            }
            break;
        }
        if (ptrue) {
            // no pending client holds credit: the visit of request j refills
            block_refill(a, &sm);
            const int64_t slack2 = sched_slack(a, sm.headroom);
            const int32_t jj = block_find(a, &sm, j, j + 1, false, slack2);
            if (jj != FS_NONE) block_admit(a, &sm, jj, slack2);
        } else {
            block_admit(a, &sm, j, slack);
        }
        if (tid == 0) sm.cursor = j + 1;
        __syncthreads();
        if (sm.stop) break;
    }
    __syncthreads();
    if (a.fev) {
        // stop the evictor (handing its state over if it is still on), then
        // resolve the admissions' record counts
        const bool fon = sm.fev.on;  // read by every thread before fev_drain clears it
        __syncthreads();
        if (fon) {
            fev_drain(a.t, &sm.fev, true);
        } else if (tid == 0) {
            st_release_i32(&a.fev_ctl->stop, 1);
            while (ld_acquire_i32(&a.fev_ctl->finished) == 0) __nanosleep(32);
        }
        __syncthreads();
        (void)ld_acquire_i32(&a.fev_ctl->finished);
        const int32_t na = min(sm.nadm, a.adm_cap);
        for (int32_t e = tid; e < na; e += blockDim.x) {
            const int64_t v = a.adm_rec_end[e];
            if (v < 0) {
                const int64_t k = -v - 1;
                a.adm_rec_end[e] = k > 0 ? a.fev_rec_end[k - 1] : 0;
            }
        }
        if (tid == 0) {
            sm.ins.ev.pops += ((volatile FevCtl *)a.fev_ctl)->pops;
            a.hdr[7] = sm.fev.posted | ((int64_t)((volatile FevCtl *)a.fev_ctl)->nc << 20) |
                       ((int64_t)((volatile FevCtl *)a.fev_ctl)->heap_hw << 40) |
                       ((int64_t)((volatile FevCtl *)a.fev_ctl)->ok << 60);
        }
        __syncthreads();
    }
    if (a.nhelp > 0) {
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            st_release_i32(&a.ctl->seq, -1);  // release the helpers
            sm.resumes += *(volatile int64_t *)&a.ctl->resumes;
            sm.prof[4] += *(volatile int64_t *)&a.ctl->chunks;
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.hdr[0] = sm.nadm;
        a.hdr[1] = a.t.sc->nrec;
        a.hdr[3] = sm.epoch;
        a.hdr[4] = sm.refill_events;
        a.hdr[5] = sm.resumes;
        a.hdr[6] = sm.flt.saturated;  // the next fill's K1 trusts the filter only when complete
        sm.prof[5] = sm.ins.ev.pops;
        sm.prof[7] = clock64() - t_start;
        for (int i = 0; i < 3; i++) sm.prof[8 + i] = sm.lru.prof[i];
        for (int i = 0; i < 16; i++) a.hdr[8 + i] = sm.prof[i];
        for (int i = 0; i < 8; i++) a.hdr[24 + i] = sm.prof2[i];
        *ap.t.sc = sc_sh;
    }
}

// Debug (FS_FILL_CHECK=1): after a fill, every admission's path -- from its
// deepest node up the parent links -- must be live nodes pinned at least once;
// and for every live node: a live parent, no more pins than the parent, its
// child-hash entry, a non-empty edge.  The first violation goes to hdr[2] as
// 200 + code (hdr[6] = the node).
__global__ void k_check_fill(TrieView t, const int32_t *adm_node, const int64_t *hdr_n, int32_t cap, int64_t *hdr) {
    const int64_t n = min((int64_t)cap, hdr_n[0]);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t y = adm_node[e];
        int guard = 0;
        while (y > 0 && guard++ < (1 << 20)) {
            int code = 0;
            if (!(t.flags[y] & FS_ALIVE)) code = 1;
            else if (t.ref[y] < 1) code = 2;
            if (code) {
                if (atomicCAS((unsigned long long *)&hdr[2], (unsigned long long)FS_OK,
                              (unsigned long long)(200 + code)) == FS_OK)
                    hdr[6] = y;
                return;
            }
            y = t.parent[y];
        }
    }
    const int32_t hw = t.sc->hw;
    for (int32_t y = 1 + blockIdx.x * blockDim.x + threadIdx.x; y < hw; y += gridDim.x * blockDim.x) {
        if (!(t.flags[y] & FS_ALIVE)) continue;
        const int32_t P = t.parent[y];
        int code = 0;
        if (P > 0 && !(t.flags[P] & FS_ALIVE)) code = 3;
        // every pin covers a whole root path: a node never holds more pins
        // than its parent (an unpin would underflow at the parent)
        else if (P > 0 && t.ref[P] < t.ref[y]) code = 4;
        else if (P >= 0 && h_find(t, P, t.first[y]) != y) code = 5;  // children[first] is this node
        else if (t.start[y] >= t.end[y] || t.ref[y] < 0) code = 6;
        if (code) {
            if (atomicCAS((unsigned long long *)&hdr[2], (unsigned long long)FS_OK, (unsigned long long)(200 + code)) ==
                FS_OK)
                hdr[6] = y;
            return;
        }
    }
}

// ---------------------------------------------------------------- VTC fill
// Vtc.fill (local_policies.py:170-189): repeatedly serve the least-served
// client -- clients in (counter, name) order, each offering its earliest
// queued request (arrival, rid); the first whose head passes can_add
// (worker.py:101-110, closed form len - B <= slack) is admitted (probe,
// insert, pin, radix.py:187-192) and charged its full input (cache-oblivious,
// local_policies.py:184-186); stop when no head fits.  VTC never calls
// match_prefix, so nothing is stamped besides the inserts.  One CTA: 16 warps
// test 16 clients' heads per round (exact pinned coverage by a read-only
// walk); the earliest passing one in client order is admitted.
#define VTC_MAXC 2048
struct VtcArgs {
    TrieView t;
    int32_t n;                 // queued requests (label order = (arrival, rid) order)
    const int32_t *queue;
    const int32_t *rclient, *rlen;
    const int64_t *roff;
    int64_t *q;                // per-client virtual counters
    const int32_t *rank;       // rank of the client's name (sorted() tie-break)
    int32_t nclients;
    int32_t *head;             // [nclients] scratch: queue position of each client's head (FS_NONE: none)
    const int32_t *dl_client;  // counter deltas to apply first (host-side on_outputs / lifts)
    const int64_t *dl_delta;
    int32_t ndl;
    int64_t M, R, gen_total, headroom0, w_e, now, sq_base;
    Seg *segs;
    int8_t *rstate;
    int32_t *adm_req, *adm_mlen, *adm_node;
    int64_t *adm_unp, *adm_pinb, *adm_rec_end;
    int32_t adm_cap;
    int64_t *hdr;
};
struct VtcSmem {
    InsertSmem ins;
    ChunkLRU lru;
    int64_t key[VTC_MAXC];   // counter of the client at sorted position i
    int32_t rk[VTC_MAXC];    // its name rank
    int32_t cl[VTC_MAXC];    // the client
    int32_t nact;            // active clients (with a queued head), sorted prefix of the arrays
    int32_t pass[16];        // this round's verdicts, by warp
    int32_t cov[16];
    int32_t red32[32];
    int64_t headroom;
    int32_t nadm, stop, best;
};

__device__ __forceinline__ bool vtc_less(int64_t k1, int32_t r1, int64_t k2, int32_t r2) {
    return k1 < k2 || (k1 == k2 && r1 < r2);
}

__global__ void __launch_bounds__(FS_SCHED_THREADS, 1) k_vtc(VtcArgs ap) {
    extern __shared__ __align__(16) unsigned char fs_smraw[];
    VtcSmem &sm = *reinterpret_cast<VtcSmem *>(fs_smraw);
    __shared__ VtcArgs a_sh;
    __shared__ TrieScalars sc_sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        a_sh = ap;
        sc_sh = *ap.t.sc;
        a_sh.t.sc = &sc_sh;
        for (int32_t i = 0; i < ap.ndl; i++) ap.q[ap.dl_client[i]] += ap.dl_delta[i];
        sc_sh.nrec = 0;
        sm.nadm = 0; sm.stop = 0; sm.nact = 0;
        sm.headroom = ap.headroom0;
        sm.ins.prof = nullptr; sm.ins.prof2 = nullptr; sm.ins.fev = nullptr;
        sm.ins.lru = &sm.lru; sm.ins.lru_spare = nullptr; sm.ins.ev.pops = 0;
        for (int i = 0; i < 4; i++) sm.lru.prof[i] = 0;
        ap.hdr[2] = FS_OK;
    }
    __syncthreads();
    const VtcArgs &a = a_sh;
    const TrieView &t = a.t;
    // every client's head: its first queued position (the queue is in (arrival, rid) order)
    for (int32_t c = tid; c < a.nclients; c += blockDim.x) a.head[c] = FS_NONE;
    __syncthreads();
    for (int32_t p = tid; p < a.n; p += blockDim.x) atomicMin(&a.head[a.rclient[a.queue[p]]], p);
    __syncthreads();
    block_chunk_build(t, &sm.lru);
    // active clients in (counter, name rank) order
    for (int32_t c = tid; c < a.nclients; c += blockDim.x) {
        if (a.head[c] != FS_NONE) {
            const int32_t k = atomicAdd(&sm.nact, 1);
            if (k < VTC_MAXC) { sm.key[k] = a.q[c]; sm.rk[k] = a.rank[c]; sm.cl[k] = c; }
        }
    }
    __syncthreads();
    if (sm.nact > VTC_MAXC) {
        if (tid == 0) { a.hdr[2] = FS_ERR_INVALID; a.hdr[0] = 0; a.hdr[1] = 0; }
        return;
    }
    {
        const int32_t na = sm.nact;
        int32_t P2 = 1;
        while (P2 < na) P2 <<= 1;
        for (int32_t i = na + tid; i < P2; i += blockDim.x) { sm.key[i] = INT64_MAX; sm.rk[i] = INT32_MAX; sm.cl[i] = -1; }
        __syncthreads();
        for (int32_t k = 2; k <= P2; k <<= 1)
            for (int32_t j = k >> 1; j > 0; j >>= 1) {
                for (int32_t i = tid; i < P2; i += blockDim.x) {
                    const int32_t l = i ^ j;
                    if (l > i) {
                        const bool up = (i & k) == 0;
                        if (vtc_less(sm.key[l], sm.rk[l], sm.key[i], sm.rk[i]) == up) {
                            const int64_t x = sm.key[i]; sm.key[i] = sm.key[l]; sm.key[l] = x;
                            int32_t y = sm.rk[i]; sm.rk[i] = sm.rk[l]; sm.rk[l] = y;
                            y = sm.cl[i]; sm.cl[i] = sm.cl[l]; sm.cl[l] = y;
                        }
                    }
                }
                __syncthreads();
            }
    }
    while (!sm.stop) {
        // the first client, in order, whose head passes can_add
        int64_t slack;
        {
            const int64_t pinned = t.sc->pinned;
            slack = a.M - a.gen_total - sm.headroom - a.R - pinned;  // worker.py:104-107
            const int64_t cap = t.sc->capacity;
            if (cap >= 0 && cap - pinned < slack) slack = cap - pinned;  // worker.py:108-109
        }
        int32_t found = -1;
        for (int32_t g = 0; g < sm.nact && found < 0; g += 16) {
            if (warp < 16) {
                const int32_t i = g + warp;
                int32_t ok = 0, cv = 0;
                if (i < sm.nact) {
                    const int32_t r = a.queue[a.head[sm.cl[i]]];
                    const int32_t len = a.rlen[r];
                    const WalkOut w = warp_walk<8>(t, t.arena + a.roff[r], len, lane, nullptr, true);
                    cv = w.cov;
                    ok = (int64_t)(len - w.cov) <= slack;
                }
                if (lane == 0) { sm.pass[warp] = ok; sm.cov[warp] = cv; }
            }
            __syncthreads();
            if (tid == 0) {
                sm.best = -1;
                for (int k = 0; k < 16 && g + k < sm.nact; k++)
                    if (sm.pass[k]) { sm.best = g + k; break; }
            }
            __syncthreads();
            found = sm.best;
            __syncthreads();
        }
        if (found < 0) break;
        // admit the head of client cl[found] (Worker.try_admit -> RadixTree.admit)
        const int32_t c = sm.cl[found];
        const int32_t hp = a.head[c];
        const int32_t r = a.queue[hp];
        const int32_t len = a.rlen[r];
        const int64_t off = a.roff[r];
        __shared__ int64_t pinb;
        if (tid == 0) pinb = t.sc->pinned;
        __syncthreads();
        auto on_walk = [&](int) {
            const InsertSmem &in = sm.ins;
            if (in.status != FS_OK) return;
            const int64_t need = len - in.cov;
            t.sc->pinned += need;
            if (need > slack || in.unpinned != (int64_t)(in.mlen - in.cov)) { a.hdr[2] = FS_ERR_INTERNAL; sm.stop = 1; }
        };
        block_insert(t, off, len, a.now, a.sq_base + sm.nadm, -1, a.segs, &sm.ins, -1, -1, true, on_walk, NoHook());
        if (tid == 0) {
            const InsertSmem &in = sm.ins;
            if (in.status != FS_OK) {
                a.hdr[2] = in.status;
                sm.stop = 1;
            } else {
                const int32_t e = sm.nadm;
                if (e < a.adm_cap) {
                    a.adm_req[e] = r; a.adm_mlen[e] = in.mlen; a.adm_unp[e] = in.unpinned;
                    a.adm_pinb[e] = pinb; a.adm_node[e] = in.deepest; a.adm_rec_end[e] = t.sc->nrec;
                }
                sm.nadm = e + 1;
                a.rstate[r] = 2;
                a.q[c] += a.w_e * (int64_t)len;  // the full input (local_policies.py:184-186)
                sm.headroom += a.R;
                if (t.sc->status != FS_OK) { a.hdr[2] = t.sc->status; sm.stop = 1; }
            }
        }
        __syncthreads();
        if (sm.stop) break;
        // the client's next head: its next queued position
        {
            int32_t mine = FS_NONE;
            for (int32_t p = hp + 1 + tid; p < a.n && mine == FS_NONE; p += blockDim.x)
                if (a.rclient[a.queue[p]] == c) mine = p;
            const int32_t nh = block_min_i32(mine, sm.red32);
            if (tid == 0) a.head[c] = nh;
        }
        __syncthreads();
        if (tid == 0) {
            // re-place the client: its counter only grew; drop it when its queue is empty
            int32_t i = found;
            if (a.head[c] == FS_NONE) {
                for (; i + 1 < sm.nact; i++) { sm.key[i] = sm.key[i + 1]; sm.rk[i] = sm.rk[i + 1]; sm.cl[i] = sm.cl[i + 1]; }
                sm.nact--;
            } else {
                const int64_t kk = a.q[c];
                const int32_t rr = sm.rk[i];
                while (i + 1 < sm.nact && vtc_less(sm.key[i + 1], sm.rk[i + 1], kk, rr)) {
                    sm.key[i] = sm.key[i + 1]; sm.rk[i] = sm.rk[i + 1]; sm.cl[i] = sm.cl[i + 1];
                    i++;
                }
                sm.key[i] = kk; sm.rk[i] = rr; sm.cl[i] = c;
            }
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid == 0) {
        a.hdr[0] = sm.nadm;
        a.hdr[1] = t.sc->nrec;
        a.hdr[3] = sm.nadm;
        for (int i = 4; i < 32; i++) a.hdr[i] = 0;
        a.hdr[13] = sm.ins.ev.pops;
        *ap.t.sc = sc_sh;
    }
}

// ---------------------------------------------------------------- per-call ops
enum { OP_INSERT = 1, OP_ADMIT, OP_PIN, OP_UNPIN, OP_EVICT, OP_LMW, OP_NOTIFY };

struct OpArgs {
    TrieView t;
    int32_t op;
    int64_t req_off;
    int32_t len;
    int64_t now;
    int32_t worker;
    int32_t node;
    int64_t needed;
    int32_t keep;
    int64_t notice;
    int64_t sq;  // operation sequence number for stamps
    Seg *segs;
    int32_t *found;
    int64_t *out;  // [status, mlen/new_len, deepest, mask, nrec]
};

__global__ void __launch_bounds__(256) k_op(OpArgs a) {
    __shared__ InsertSmem ins;
    __shared__ NotifySmem nsm;
    __shared__ int32_t s_nseg;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const TrieView &t = a.t;
    if (tid == 0) {
        t.sc->nrec = 0; t.sc->status = FS_OK; ins.prof = nullptr; ins.lru = nullptr; ins.ev.pops = 0; ins.fev = nullptr;
        for (int k = 0; k < 4; k++) nsm.prof[k] = 0;
    }
    __syncthreads();
    const int32_t *rq = t.arena + a.req_off;
    switch (a.op) {
        case OP_INSERT:
            block_insert(t, a.req_off, a.len, a.now, a.sq, a.worker, a.segs, &ins);
            if (tid == 0) { a.out[0] = ins.status; a.out[1] = ins.new_len; a.out[2] = ins.deepest; }
            break;
        case OP_ADMIT:
            // probe (radix.py:189) -> insert -> pin; the probe's mlen equals the
            // insert walk's (nothing changes between them)
            block_insert(t, a.req_off, a.len, a.now, a.sq, -1, a.segs, &ins);
            if (ins.status == FS_OK) block_pin_path(t, a.segs, ins.nseg, +1);
            __syncthreads();
            if (tid == 0) { a.out[0] = ins.status; a.out[1] = ins.mlen; a.out[2] = ins.deepest; }
            break;
        case OP_PIN:
        case OP_UNPIN:
            // _chain from the deepest node (radix.py:164-172) == the nodes of its root path
            block_path_of(t, a.node, a.segs, &s_nseg);
            block_pin_path(t, a.segs, s_nseg, a.op == OP_PIN ? +1 : -1);
            __syncthreads();
            if (tid == 0) a.out[0] = t.sc->status;
            break;
        case OP_EVICT:
            block_evict(t, a.needed, &ins.ev);
            if (tid == 0) a.out[0] = t.sc->status;
            break;
        case OP_LMW:
            if (warp == 0) {
                const WalkOut w = warp_walk(t, rq, a.len, lane, nullptr, false);
                if (lane == 0) {
                    // deepest = partial or last full node (radix.py:104); stamps the path
                    const int32_t deepest = w.mlen > 0 ? w.last : -1;
                    if (deepest > 0) stamp_node(t, deepest, a.now, a.sq);
                    a.out[0] = FS_OK;
                    a.out[1] = deepest > 0 ? w.mlen : 0;
                    a.out[3] = (deepest > 0 && t.wmask) ? (int64_t)t.wmask[deepest] : 0;
                }
            }
            break;
        case OP_NOTIFY:
            block_evict_notify(t, a.req_off, a.len, a.worker, a.keep, a.notice, a.segs, a.found, &nsm);
            if (tid == 0) a.out[0] = t.sc->status;
            break;
    }
    __syncthreads();
    if (tid == 0) a.out[4] = t.sc->nrec;
}

// A round's eviction notices applied in order (evict_notify, radix.py:254-302).
__global__ void __launch_bounds__(256) k_notify_many(TrieView t, int32_t n, const int64_t *__restrict__ src,
                                                     const int32_t *__restrict__ len, const int32_t *__restrict__ worker,
                                                     const int32_t *__restrict__ keep, const int64_t *__restrict__ when,
                                                     const int32_t *__restrict__ m0, const int64_t *__restrict__ s0,
                                                     Seg *segs, int32_t *found, int64_t *out) {
    __shared__ NotifySmem nsm;
    if (threadIdx.x == 0) {
        t.sc->nrec = 0; t.sc->status = FS_OK;
        for (int k = 0; k < 4; k++) nsm.prof[k] = 0;
    }
    __syncthreads();
    for (int32_t i = 0; i < n; i++) {
        block_evict_notify(t, src[i], len[i], worker[i], keep[i], when[i], segs, found, &nsm, s0[i], m0[i],
                           i + 1 < n ? s0[i + 1] : -1, i + 1 < n ? m0[i + 1] : -1);
        __syncthreads();
        if (t.sc->status != FS_OK) break;
    }
    if (threadIdx.x == 0) {
        out[0] = t.sc->status;
        for (int k = 0; k < 4; k++) out[1 + k] = nsm.prof[k];  // walk, collect, edit, repoint cycles
    }
}

// ---------------------------------------------------------------- D2LPM
// Batch-start match of one arrival against the routing index (no stamping):
// match length, chain of the deepest matched node and the path's source-chain
// segments.  One fixed-size record per arrival, so ranks can each match a
// slice of an arrival batch and all-gather the records (fs_dispatch_prematch).
struct PreRec {
    int32_t m0;    // match length
    int32_t nseg;  // segments, -1: more than FS_PRE_SEGS (rebuilt from the chain links)
    int64_t s0;    // chain (arena row) of the deepest matched node, -1: none
    Seg segs[FS_PRE_SEGS];
};
static_assert(sizeof(PreRec) == 16 + 16 * FS_PRE_SEGS, "PreRec is exchanged as raw bytes");

struct DispArgs {
    TrieView t;
    int32_t n, D;
    int32_t select_only;  // fs_dispatch_select: mask comes in out_mask[0]
    const int32_t *ids, *clients;
    const int64_t *nows;
    const int64_t *roff;
    const int32_t *rlen;
    int64_t *q;  // [client * D + w]
    uint8_t *qset;
    int64_t *qsize;
    int64_t quantum, w_e;
    int64_t sq_base;  // arrival i stamps with sq_base + 2i (match) and sq_base + 2i + 1 (insert)
    const int32_t *dl_idx;  // pending host-side updates (see k_dispatch)
    const int64_t *dl_q;
    const int32_t *dl_w;
    int32_t ndl;
    Seg *segs;
    const struct PreRec *pre;  // batch-start match of every arrival (k_dispatch_prematch, no stamp)
    int32_t *out_w, *out_mlen;
    uint64_t *out_mask;
    int64_t *out_rounds;
    int64_t *hdr;
    int32_t policy;  // 0: D2lpm (global_policies.py:88-132); 1: ThresholdRouter (135-161)
    double theta;
};

// ThresholdRouter.select (global_policies.py:149-155) + _min_queue (57-58):
// locality when the matched fraction reaches theta (the same IEEE double
// division as Python's `match_len / input_len`), else the least loaded worker.
__device__ inline int threshold_select(const DispArgs &a, int32_t mlen, int32_t len, uint64_t mask) {
    const bool local = mask != 0ull && len > 0 && (double)mlen / (double)len >= a.theta;
    int best = -1;
    for (int w2 = 0; w2 < a.D; w2++) {
        if (local && !((mask >> w2) & 1ull)) continue;
        if (best < 0 || a.qsize[w2] < a.qsize[best]) best = w2;
    }
    return best;
}

// D2lpm.select_worker (global_policies.py:107-114) + Dispatcher._min_queue
// (57-58).  The refill loop adds Q_w to every worker per round: k rounds in
// closed form.  Returns the worker; *rounds = refill rounds.
__device__ inline int d2_select(const DispArgs &a, int32_t c, uint64_t mask, int64_t *rounds) {
    int64_t *qr = a.q + (int64_t)c * a.D;
    uint8_t *qs = a.qset + (int64_t)c * a.D;
    bool any = false;
    for (int w2 = 0; w2 < a.D; w2++) any |= qr[w2] > 0;
    *rounds = 0;
    if (!any) {
        int64_t k = INT64_MAX;
        for (int w2 = 0; w2 < a.D; w2++) k = min(k, (-qr[w2]) / a.quantum + 1);
        for (int w2 = 0; w2 < a.D; w2++) { qr[w2] += k * a.quantum; qs[w2] = 1; }
        *rounds = k;
    }
    int best = -1;
    for (int pass = 0; pass < 2 && best < 0; pass++)
        for (int w2 = 0; w2 < a.D; w2++) {
            if (!(qr[w2] > 0)) continue;
            if (pass == 0 && !((mask >> w2) & 1ull)) continue;
            if (best < 0 || a.qsize[w2] < a.qsize[best]) best = w2;
        }
    return best;
}

// Batch-start longest match of every arrival of a dispatch chain, a warp each,
// in parallel (no stamps): match length, chain of the deepest matched node and
// the segments of the matched path.  Inside the chain the index only gains
// nodes (inserts and splits keep every node's source chain), so these
// segments still describe [0, m0) when the arrival's turn comes.
__global__ void __launch_bounds__(256) k_dispatch_prematch(TrieView t, const int32_t *__restrict__ ids, int32_t n,
                                                           const int64_t *__restrict__ roff,
                                                           const int32_t *__restrict__ rlen, PreRec *out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const int32_t r = ids[i];
    Seg *my = out[i].segs;
    int64_t lastS = -1;
    auto store = [&](int64_t S, int32_t a, int32_t b, int32_t k) {
        if (lane == 0 && k < FS_PRE_SEGS) { my[k].S = S; my[k].a = a; my[k].b = b; }
        lastS = S;
    };
    const WalkOut w = warp_walk_cb<8, decltype(store), true>(t, t.arena + roff[r], rlen[r], lane, false, store);
    if (lane == 0) {
        out[i].m0 = w.mlen;
        out[i].s0 = w.mlen > 0 ? lastS : -1;
        out[i].nseg = w.nseg <= FS_PRE_SEGS ? w.nseg : -1;
    }
}

// Dispatcher.dispatch for a chain of arrivals (global_policies.py:40-46,
// 116-124): every arrival's match sees the inserts of the ones before it.
__global__ void __launch_bounds__(FS_DISPATCH_THREADS, 1) k_dispatch(DispArgs a) {
    __shared__ InsertSmem ins;
    __shared__ int32_t s_w;
    __shared__ int32_t s_mlen;
    __shared__ uint64_t s_mask;
    // cycle profile: [0] lmw walk + select, [1] insert walk, [2] evict, [12] leaf + stamp +
    // repoint, [14] worker tags, [15] total
    __shared__ int64_t prof[16];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const TrieView &t = a.t;
    if (tid == 0) {
        // pending host-side updates: q index >= 0 -> counter delta (on_finish /
        // explicit override); q index -1 -> queue_size[w] += delta
        for (int32_t i = 0; i < a.ndl; i++) {
            if (a.dl_idx[i] >= 0) { a.q[a.dl_idx[i]] += a.dl_q[i]; a.qset[a.dl_idx[i]] = 1; }
            else a.qsize[a.dl_w[i]] += a.dl_q[i];
        }
        t.sc->status = FS_OK;
        for (int i = 0; i < 16; i++) prof[i] = 0;
        ins.prof = prof;
        ins.lru = nullptr;
        ins.fev = nullptr;
        ins.ev.pops = 0;
    }
    __syncthreads();
    const long long t0 = clock64();
    if (a.select_only) {
        if (tid == 0 && a.n > 0) {
            int64_t rounds;
            a.out_w[0] = d2_select(a, a.clients[0], a.out_mask[0], &rounds);
            a.out_rounds[0] = rounds;
            a.hdr[0] = FS_OK;
        }
        return;
    }
    // the chain's per-arrival scalars, staged FS_DISP_STAGE at a time so each
    // arrival starts without a dependent ids -> (len, off) round trip
    __shared__ int32_t s_len[FS_DISP_STAGE], s_m0[FS_DISP_STAGE], s_cl[FS_DISP_STAGE];
    __shared__ int64_t s_off[FS_DISP_STAGE], s_now[FS_DISP_STAGE], s_s0[FS_DISP_STAGE];
    for (int32_t i = 0; i < a.n; i++) {
        const int32_t k = i % FS_DISP_STAGE;
        if (k == 0) {
            __syncthreads();
            for (int32_t j = tid; j < FS_DISP_STAGE && i + j < a.n; j += blockDim.x) {
                const int32_t r = a.ids[i + j];
                s_len[j] = a.rlen[r]; s_off[j] = a.roff[r]; s_now[j] = a.nows[i + j];
                s_s0[j] = a.pre[i + j].s0; s_m0[j] = a.pre[i + j].m0; s_cl[j] = a.clients[i + j];
            }
            __syncthreads();
        }
        const int32_t len = s_len[k];
        const int64_t off = s_off[k];
        const int64_t now = s_now[k];
        const int64_t hs0 = s_s0[k];
        const int32_t hm0 = s_m0[k];
        const long long cw = clock64();
        WalkOut w{};
#if FS_POP_PREFETCH
        if (tid == 32 && k + 1 < FS_DISP_STAGE && i + 1 < a.n && s_m0[k + 1] > 0) {
            // warp 1 idles during this walk: warm L1 for the next arrival's
            // hinted walk (deepest node, its token at the hint depth and the
            // child slot that token probes) -- hints only
            const int32_t m1 = s_m0[k + 1];
            const int32_t y2 = t.pos[s_s0[k + 1] + m1 - 1];
            if (y2 > 0 && y2 < t.sc->hw) {
                pf_l1(t.flags + y2); pf_l1(t.src + y2); pf_l1(t.start + y2); pf_l1(t.end + y2);
                pf_l1(t.wmask + y2); pf_l1(t.lseq + y2);
                if (m1 < s_len[k + 1]) {
                    const int32_t tk = t.arena[s_off[k + 1] + m1];
                    pf_l1(t.hslot + (fs_hmix(fs_hkey(y2, tk)) & t.hmask));
                }
            }
        }
#endif
        if (warp == 0) {
            // RadixTree.longest_match_workers (radix.py:101-110).  The index only
            // gains prefixes of this batch's earlier arrivals (no capacity, no
            // eviction inside a batch), so the batch-start match is still a
            // prefix of the current one: resume from it (warp_walk_hint).
            // (with its segments: block_insert below reuses this walk)
            w = warp_walk_hint<8, false, true>(t, t.arena + off, len, lane, a.segs, hs0, hm0,
                                                a.pre[i].segs, a.pre[i].nseg);
            if (lane == 0) {
                const int32_t deepest = w.mlen > 0 ? w.last : -1;
                if (deepest > 0) stamp_node(t, deepest, now, a.sq_base + 2 * (int64_t)i);
                const uint64_t mask = deepest > 0 ? t.wmask[deepest] : 0ull;
                int64_t rounds = 0;
                const int32_t cl = s_cl[k];
                const int32_t ml = deepest > 0 ? w.mlen : 0;
                int best;
                if (a.policy == 1) {
                    best = threshold_select(a, ml, len, mask);
                    a.qsize[best] += 1;  // Dispatcher.dispatch (global_policies.py:42)
                } else {
                    best = d2_select(a, cl, mask, &rounds);
                    int64_t *qr = a.q + (int64_t)cl * a.D;
                    a.qsize[best] += 1;
                    qr[best] -= a.w_e * (int64_t)len;  // after_dispatch: full input (global_policies.py:123)
                    a.qset[(int64_t)cl * a.D + best] = 1;
                }
                s_w = best; s_mlen = ml; s_mask = mask;
                a.out_rounds[i] = rounds;
            }
        }
        __syncthreads();
        if (tid == 0) prof[0] += clock64() - cw;
        block_insert(t, off, len, now, a.sq_base + 2 * (int64_t)i + 1, s_w, a.segs, &ins, hs0, hm0, false,
                     NoHook(), NoHook(), warp == 0 ? &w : nullptr);
        if (tid == 0) {
            a.out_w[i] = s_w;
            a.out_mlen[i] = s_mlen;
            a.out_mask[i] = s_mask;
        }
        __syncthreads();
    }
    if (tid == 0) {
        a.hdr[0] = t.sc->status;
        prof[15] = clock64() - t0;
        for (int i = 0; i < 16; i++) a.hdr[4 + i] = prof[i];
    }
}

// Dlpm.check_refill (local_policies.py:94-106) on an explicit queued set.
__global__ void k_check_refill(int64_t *q, int64_t *refills, const uint8_t *known, int32_t nclients,
                               const uint8_t *queued, int64_t quantum, int64_t *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    bool anyq = false;
    for (int32_t c = 0; c < nclients; c++) {
        if (queued[c]) {
            anyq = true;
            if (q[c] > 0) { out[0] = 0; return; }
        }
    }
    if (!anyq) { out[0] = 0; return; }
    for (int32_t c = 0; c < nclients; c++)
        if (known[c] && q[c] <= 0) { q[c] += quantum; refills[c] += 1; }
    out[0] = 1;
}
