// fs_device.cuh -- device-side data model and primitives of the B200-native
// DLPM / D^2LPM decision path (arXiv 2501.14312).
//
// Data model (HBM):
//   * token arena: every request's int32 tokens, uploaded once, 16-B aligned.
//   * radix trie (one per RadixTree, radix.py:48): SoA node table.  A node does
//     not own tokens: its root path is arena[src : src+end] -- a prefix of the
//     request that created it (its "source chain") -- and its edge is
//     arena[src+start : src+end].  Splits and partial evictions only move
//     start/end; no token is ever copied.
//   * position shadow pos[arena offset]: for every token position p of a
//     source chain S that is cached in this trie, pos[S+p] is the node covering
//     depth p.  A walk therefore compares a request against a whole source
//     chain in one contiguous, coalesced stream and finds the node it stops in
//     with one lookup -- the cost is per source chain crossed, not per node.
//     (The reference trees of configs 2/5 hold hundreds of split nodes along
//     one document chain.)
//   * children: one open-addressing hash (parent, first token) -> child, with
//     key and value packed in one 16-byte slot (one load per probe), linear
//     probing, backward-shift deletion.
//   * last_access is stored lazily: la[n] holds the latest stamp of a path
//     that *ended* at n, tagged with its operation sequence number; the
//     reference value is the most recent stamp in n's subtree (every stamp in
//     radix.py:86-90,107-109,158-159 covers a whole root path, last write
//     wins).  A detached leaf pushes its stamp up to its parent, so leaves --
//     the only nodes LRU eviction compares (radix.py:196-219) -- always hold
//     their exact value.
//   * ref counts stay exact per node; pin/unpin touch every node of a path,
//     enumerated block-parallel from the source-chain segments of the walk.
//
// Structural edits are made by one thread of one CTA (the reference is
// single-writer); compares are warp-wide, bulk per-position and
// per-path-node updates are block-parallel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FS_FULL 0xffffffffu
#define FS_HEMPTY 0xffffffffffffffffull
#define FS_HTOMB 0xfffffffffffffffeull  // deleted slot (real keys are < 2^63)

#define FS_OK 0
#define FS_ERR_INVALID 1
#define FS_ERR_CUDA 2
#define FS_ERR_CACHE_FULL 3
#define FS_ERR_TOKEN_RANGE 4
#define FS_ERR_NOMEM 5
#define FS_ERR_INTERNAL 6
#define FS_ERR_UNDERFLOW 7

#define FS_ALIVE 1u
#define FS_PROTECT 2u

struct TrieScalars {
    int64_t used;      // used_tokens   (radix.py:53)
    int64_t pinned;    // pinned_tokens (radix.py:54)
    int64_t next_seq;  // _seq          (radix.py:55)
    int64_t capacity;  // < 0: None
    int64_t nrec;      // eviction records emitted by the current op
    int32_t hw;        // node-table high-water mark
    int32_t nfree;     // free-stack depth
    int32_t status;    // sticky device error
    int32_t live;      // live nodes (incl. root)
    int32_t tombs;     // deleted child-hash slots
    int32_t pad_;
};

struct TrieView {
    const int32_t *arena;
    int32_t *pos;      // position shadow over the arena
    int64_t *src;
    int32_t *start, *end, *slen, *parent, *nchild, *ref, *first;
    int32_t *ctop;     // first depth of the node's source chain (its original leaf's start)
    int32_t *cpar;     // node above the chain's topmost node (same for the whole chain)
    int64_t *la, *seq;
    int64_t *lseq;     // operation sequence number of la[n] (last write wins)
    uint8_t *flags;
    uint64_t *wmask;   // nullptr unless track_workers
    int64_t *wtime;    // [node * nw + w]
    int32_t nw;
    ulonglong2 *hslot; // {key, child}
    uint32_t hmask;
    int32_t *freest;
    int32_t ncap;
    TrieScalars *sc;
    int64_t *rsrc;     // eviction-record sink
    int32_t *rlen, *rkeep;
    int64_t rcap;
};

// ---------------------------------------------------------------- hashing
__device__ __forceinline__ uint64_t fs_hkey(int32_t p, int32_t tok) {
    return ((uint64_t)(uint32_t)p << 32) | (uint32_t)tok;
}
__device__ __forceinline__ uint32_t fs_hmix(uint64_t k) {
    k ^= k >> 33; k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return (uint32_t)k;
}
// children.get(tok) (radix.py:71)
__device__ __forceinline__ int32_t h_find(const TrieView &t, int32_t p, int32_t tok) {
    const uint64_t key = fs_hkey(p, tok);
    uint32_t i = fs_hmix(key) & t.hmask;
    for (uint32_t probes = 0; probes <= t.hmask; probes++) {
        const ulonglong2 s = t.hslot[i];
        if (s.x == key) return (int32_t)s.y;
        if (s.x == FS_HEMPTY) return -1;
        i = (i + 1) & t.hmask;
    }
    return -1;
}
// children[tok] = child (update in place, else the first free or deleted slot)
__device__ inline void h_put(const TrieView &t, int32_t p, int32_t tok, int32_t child) {
    const uint64_t key = fs_hkey(p, tok);
    uint32_t i = fs_hmix(key) & t.hmask;
    int64_t tomb = -1;
    uint32_t probes = 0;
    while (true) {
        const uint64_t k = t.hslot[i].x;
        if (k == key) break;
        if (k == FS_HEMPTY || probes++ > t.hmask) {
            if (tomb >= 0) { i = (uint32_t)tomb; atomicSub(&t.sc->tombs, 1); }
            else if (k != FS_HEMPTY) { t.sc->status = FS_ERR_NOMEM; return; }  // table full
            break;
        }
        if (k == FS_HTOMB && tomb < 0) tomb = i;
        i = (i + 1) & t.hmask;
    }
    t.hslot[i] = make_ulonglong2(key, (unsigned long long)(uint32_t)child);
}
// del children[tok] -- tombstone (one store); the host rebuilds the table when
// tombstones pass a quarter of it (fs_lib.cu trie_maintain)
__device__ inline void h_del(const TrieView &t, int32_t p, int32_t tok) {
    const uint64_t key = fs_hkey(p, tok);
    uint32_t i = fs_hmix(key) & t.hmask;
    for (uint32_t probes = 0;; probes++) {
        const uint64_t k = t.hslot[i].x;
        if (k == key) break;
        if (k == FS_HEMPTY || probes > t.hmask) return;
        i = (i + 1) & t.hmask;
    }
    t.hslot[i].x = FS_HTOMB;
    t.sc->tombs++;
}

// ---------------------------------------------------------------- nodes
// RadixNode(...) with seq = self._seq; self._seq += 1  (radix.py:117-118, 153-154)
__device__ inline int32_t node_new(const TrieView &t, int64_t src, int32_t start, int32_t end, int32_t slen,
                                   int32_t parent, int32_t first_tok = -1) {
    int32_t n;
    if (t.sc->nfree > 0) n = t.freest[--t.sc->nfree];
    else if (t.sc->hw < t.ncap) n = t.sc->hw++;
    else { t.sc->status = FS_ERR_NOMEM; return -1; }
    t.src[n] = src; t.start[n] = start; t.end[n] = end; t.slen[n] = slen; t.parent[n] = parent;
    t.ctop[n] = start; t.cpar[n] = parent;  // a new leaf starts its own chain
    t.nchild[n] = 0; t.ref[n] = 0; t.la[n] = 0; t.lseq[n] = 0;
    t.seq[n] = t.sc->next_seq++;
    t.first[n] = first_tok >= 0 ? first_tok : t.arena[src + start];
    t.flags[n] = FS_ALIVE;
    if (t.wmask) t.wmask[n] = 0;
    t.sc->live++;
    return n;
}
__device__ inline void node_free(const TrieView &t, int32_t n) {
    t.flags[n] = 0;
    t.parent[n] = -2;
    t.freest[t.sc->nfree++] = n;
    t.sc->live--;
}
__device__ __forceinline__ int32_t elen(const TrieView &t, int32_t n) { return t.end[n] - t.start[n]; }

// last_access = now on every node of the root path ending at n (lazy: the
// stamp is kept at n with its operation sequence number; a node's reference
// value is the most recent stamp in its subtree).
__device__ __forceinline__ void stamp_node(const TrieView &t, int32_t n, int64_t now, int64_t sq) {
    if (t.lseq[n] != sq || t.la[n] != now) { t.la[n] = now; t.lseq[n] = sq; }
}

// RadixTree._split (radix.py:114-126): top gets a new seq, copies ref /
// last_access / workers; the bottom keeps its identity (and seq).  The caller
// re-points pos[] for the top's depth range [start, start+k) (block_repoint).
__device__ inline int32_t trie_split(const TrieView &t, int32_t node, int32_t k) {
    const int32_t P = t.parent[node];
    const int32_t top = node_new(t, t.src[node], t.start[node], t.start[node] + k, t.slen[node], P);
    if (top < 0) return -1;
    t.ctop[top] = t.ctop[node];
    t.cpar[top] = t.cpar[node];
    t.ref[top] = t.ref[node];
    t.la[top] = 0;  // lazy: the top's value is the latest stamp in its subtree (the bottom's)
    t.lseq[top] = 0;
    if (t.wmask) {
        t.wmask[top] = t.wmask[node];
        for (int w = 0; w < t.nw; w++) t.wtime[(int64_t)top * t.nw + w] = t.wtime[(int64_t)node * t.nw + w];
    }
    h_put(t, P, t.first[node], top);  // node.parent.children[top.edge[0]] = top
    t.start[node] += k;
    t.first[node] = t.arena[t.src[node] + t.start[node]];
    t.parent[node] = top;
    h_put(t, top, t.first[node], node);
    t.nchild[top] = 1;
    return top;
}

// RadixTree._detach (radix.py:206-208); the leaf's last_access moves to its
// parent so the parent's subtree maximum is unchanged.
__device__ inline void trie_detach(const TrieView &t, int32_t n) {
    const int32_t P = t.parent[n];
    h_del(t, P, t.first[n]);
    t.nchild[P]--;
    if (P > 0 && t.lseq[n] > t.lseq[P]) { t.la[P] = t.la[n]; t.lseq[P] = t.lseq[n]; }
    t.sc->used -= elen(t, n);
    node_free(t, n);
}

__device__ inline void push_record(const TrieView &t, int64_t src, int32_t len, int32_t keep) {
    const int64_t i = t.sc->nrec++;
    if (i < t.rcap) { t.rsrc[i] = src; t.rlen[i] = len; t.rkeep[i] = keep; }
}

// ---------------------------------------------------------------- compare
// LCP of a[0:n) and b[0:n) by one warp: 128 tokens per step, first mismatch
// by ballot + ffs (common_prefix_len, _speedups.pyx:11-22, at warp width).
// U loads per lane in flight: 4 for the many-warp match kernel (bounded
// over-read past the mismatch), 8 for the single-warp walks on the admission
// critical path (latency-bound).
// Request tokens are read once per match: keep them out of L1 so the trie's
// hot chains (compared by every warp of the SM) stay resident there.
// They are also marked evict-first in L2: K1 streams ~10 GB per step on
// config 5, which would otherwise flush the trie's node table, child hash and
// position shadow out of L2 before the latency-bound scheduler runs.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *p) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2_evict_first()));
    return v;
}

template <int U = 4>
__device__ __forceinline__ int32_t warp_lcp(const int32_t *__restrict__ a, const int32_t *__restrict__ b,
                                            int32_t n, int lane) {
    int32_t k = 0;
    while (k < n) {
        bool bad[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int32_t p = k + u * 32 + lane;
            bad[u] = (p < n) && (__ldg(a + p) != ld_stream(b + p));
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const unsigned m = __ballot_sync(FS_FULL, bad[u]);
            if (m) return min(n, k + u * 32 + __ffs(m) - 1);
        }
        k += 32 * U;
    }
    return n;
}

// Vectorized LCP for the many-warp match kernel (K1).  Both sequences are
// arena rows of 16-B aligned requests compared at the same depth, so they
// share their alignment mod 4 tokens: after a scalar head up to the next
// 16-B boundary, every lane compares 4 tokens with one 128-bit load per side
// (V loads per side in flight per lane, 128*V tokens per warp step).  Reads
// at most 3 tokens past n (inside the arena's row padding / next row).
template <int V = 2>
__device__ __forceinline__ int32_t warp_lcp_vec(const int32_t *__restrict__ a, const int32_t *__restrict__ b,
                                                int32_t n, int lane) {
    if (n <= 0) return 0;
    const uint64_t pol = l2_evict_first();
    const int32_t h = min(n, (int32_t)(((16u - ((uint32_t)(uintptr_t)b & 15u)) & 15u) >> 2));
    if ((((uintptr_t)a ^ (uintptr_t)b) & 15u) != 0) return warp_lcp<8>(a, b, n, lane);  // not co-aligned
    if (h > 0) {
        const unsigned m = __ballot_sync(FS_FULL, lane < h && __ldg(a + lane) != ld_stream(b + lane));
        if (m) return __ffs(m) - 1;
    }
    for (int32_t k = h; k < n; k += 128 * V) {
        int4 av[V], bv[V];
#pragma unroll
        for (int v = 0; v < V; v++) {
            const int32_t p = k + 128 * v + 4 * lane;
            if (p < n) {
                av[v] = __ldg(reinterpret_cast<const int4 *>(a + p));
                int4 x;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
                             : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(b + p), "l"(pol));
                bv[v] = x;
            } else {
                av[v] = make_int4(0, 0, 0, 0);
                bv[v] = av[v];
            }
        }
#pragma unroll
        for (int v = 0; v < V; v++) {
            const int32_t p = k + 128 * v + 4 * lane;
            int f = 4;
            if (av[v].w != bv[v].w && p + 3 < n) f = 3;
            if (av[v].z != bv[v].z && p + 2 < n) f = 2;
            if (av[v].y != bv[v].y && p + 1 < n) f = 1;
            if (av[v].x != bv[v].x && p < n) f = 0;
            const unsigned m = __ballot_sync(FS_FULL, f < 4);
            if (m) {
                const int L = __ffs(m) - 1;
                return min(n, k + 128 * v + 4 * L + __shfl_sync(FS_FULL, f, L));
            }
        }
    }
    return n;
}

// Is node y the cached node covering depth d of source chain S?
__device__ __forceinline__ bool pos_valid(const TrieView &t, int32_t y, int64_t S, int32_t d) {
    return y > 0 && y < t.sc->hw && (t.flags[y] & FS_ALIVE) && t.src[y] == S && t.start[y] <= d && d < t.end[y];
}

// Deepest cached node of chain S covering a depth in [lo, hi] (depth lo is
// known cached).  A chain is cached on a contiguous depth range (only its
// bottom can be evicted or truncated), so validity is monotone.
__device__ inline int32_t chain_lookup(const TrieView &t, int64_t S, int32_t lo, int32_t hi) {
    int32_t y = t.pos[S + hi];
    if (pos_valid(t, y, S, hi)) return y;
    while (lo < hi) {
        const int32_t mid = (lo + hi + 1) >> 1;
        if (pos_valid(t, t.pos[S + mid], S, mid)) lo = mid; else hi = mid - 1;
    }
    return t.pos[S + lo];
}

struct Seg {
    int64_t S;
    int32_t a, b;  // depths [a, b) of chain S on the path
};

struct WalkOut {
    int32_t mlen;      // match length
    int32_t last;      // deepest node the match reaches (partial or last full); -1 if none
    int32_t plen;      // if partial: tokens matched inside `last`; 0 when `last` is fully matched
    int32_t nseg;      // source-chain segments of the path
    int32_t cov;       // matched tokens inside pinned nodes (pinned coverage B)
    int64_t unpinned;  // probe()'s matched-unpinned count (radix.py:96-98)
};

// RadixTree._walk (radix.py:60-81) by one warp, chain by chain.  on_seg(S, a, b)
// is called warp-uniformly for every source-chain segment of the path, in
// order.  All lanes return the same WalkOut.  With want_cov, also computes the
// pinned coverage: ref counts never increase with depth along a root path, so
// it is one binary search per chain.
// Pinned coverage inside segment [a, b) of chain S whose deepest node is y:
// returns b if every node is pinned, else the first depth in an unpinned node
// (a node start) -- 32-ary search, one probe per lane per round.  Warp-uniform.
__device__ inline int32_t warp_seg_cov(const TrieView &t, int64_t S, int32_t a, int32_t b, int32_t y, int lane) {
    if (t.ref[y] > 0) return b;
    int32_t lo = a, hi = b;
    while (hi - lo > 32) {
        const int32_t step = (hi - lo + 31) / 32;
        const int32_t d = min(lo + lane * step, hi - 1);
        const unsigned m = __ballot_sync(FS_FULL, t.ref[t.pos[S + d]] == 0);
        if (m == 0) {
            lo = min(lo + 31 * step, hi - 1) + 1;
        } else {
            const int f = __ffs(m) - 1;
            const int32_t df = min(lo + f * step, hi - 1);
            if (f == 0) { hi = lo; break; }
            lo = min(lo + (f - 1) * step, hi - 1) + 1;
            hi = df;
        }
    }
    if (hi - lo > 0) {
        const int32_t d = lo + lane;
        const unsigned m = __ballot_sync(FS_FULL, d < hi && t.ref[t.pos[S + d]] == 0);
        hi = m ? lo + __ffs(m) - 1 : hi;
    }
    return hi;
}

// Walk state handed between the chain walk and its starts (root, or a
// validated earlier match).
struct WalkStart {
    int32_t node, idx, nseg, last, cov;
    bool pinrun;
};

template <int U = 4, typename SegFn, bool PIPE = false>
__device__ inline WalkOut warp_walk_from(const TrieView &t, const int32_t *__restrict__ rq, int32_t len, int lane,
                                         bool want_cov, WalkStart st, SegFn on_seg, int32_t tok_first = -1) {
    // tok_first >= 0: the request's token at st.idx, known to the caller (K1's
    // miss token) -- saves the first hop's request read
    WalkOut o;
    o.mlen = 0; o.last = st.last; o.plen = 0; o.nseg = st.nseg; o.cov = st.cov; o.unpinned = 0;
    int32_t node = st.node, idx = st.idx;
    bool pinrun = want_cov && st.pinrun;
    while (idx < len) {
        const int32_t c = h_find(t, node, (idx == st.idx && tok_first >= 0) ? tok_first : rq[idx]);
        if (c < 0) break;
        const int64_t S = t.src[c];
        const int32_t bound = min(len, t.slen[c]);
        const int32_t k = 1 + (PIPE ? warp_lcp_vec<U>(t.arena + S + idx + 1, rq + idx + 1, bound - idx - 1, lane)
                                    : warp_lcp<U>(t.arena + S + idx + 1, rq + idx + 1, bound - idx - 1, lane));
        const int32_t D = idx + k;  // request == chain S on [idx, D)
        const int32_t y = chain_lookup(t, S, idx, D - 1);
        const int32_t e = t.end[y];
        const int32_t b = min(D, e);
        on_seg(S, idx, b, o.nseg);
        o.nseg++;
        if (pinrun) {
            o.cov = warp_seg_cov(t, S, idx, b, y, lane);
            pinrun = o.cov == b;
        }
        o.last = y;
        if (D < e) { o.plen = D - t.start[y]; idx = D; break; }  // diverged inside y (or request ended)
        idx = e;
        node = y;
    }
    o.mlen = idx;
    if (want_cov) o.unpinned = o.mlen - o.cov;
    return o;
}

template <int U = 4, typename SegFn, bool PIPE = false>
__device__ inline WalkOut warp_walk_cb(const TrieView &t, const int32_t *__restrict__ rq, int32_t len, int lane,
                                       bool want_cov, SegFn on_seg) {
    WalkStart st;
    st.node = 0; st.idx = 0; st.nseg = 0; st.last = -1; st.cov = 0; st.pinrun = true;
    return warp_walk_from<U, SegFn, PIPE>(t, rq, len, lane, want_cov, st, on_seg);
}

// Source-chain segments of the cached root path [0, d) whose depth d-1 lies in
// node y: chain by chain through the per-chain constants (src, ctop, cpar) --
// one dependent load round per chain, no token compare.  Lane 0 writes segs in
// path order; returns the count (warp-uniform).
__device__ inline int32_t warp_path_segments(const TrieView &t, int32_t y, int32_t d, Seg *segs, int lane,
                                             int32_t cap = INT32_MAX) {
    // cap: at most cap segments, else -1 (segs partly written)
    int32_t ns = 0;
    if (lane == 0) {
        int32_t cur = y;
        while (d > 0 && cur > 0) {
            if (ns == cap) { ns = -1; break; }
            const int64_t S = t.src[cur];
            const int32_t c0 = t.ctop[cur];
            const int32_t X = t.cpar[cur];
            segs[ns].S = S; segs[ns].a = c0; segs[ns].b = d;
            ns++;
            d = c0;
            cur = X;
        }
        for (int32_t i = 0; i < ns / 2; i++) {  // (nothing to reverse when ns == -1)
            const Seg tmp = segs[i];
            segs[i] = segs[ns - 1 - i];
            segs[ns - 1 - i] = tmp;
        }
    }
    ns = __shfl_sync(FS_FULL, ns, 0);
    __syncwarp();
    return ns;
}

// Pinned coverage of the cached root path [0, d) ending in node y, searched
// from the deep end chain by chain (refs never increase with depth): no
// segment storage.  Warp-uniform.
__device__ inline int32_t warp_cov_from_deepest(const TrieView &t, int32_t y, int32_t d, int lane) {
    int32_t cur = y;
    while (d > 0 && cur > 0) {
        const int64_t S = t.src[cur];
        const int32_t c0 = t.ctop[cur];
        const int32_t X = t.cpar[cur];
        if (t.ref[t.pos[S + c0]] > 0) return warp_seg_cov(t, S, c0, d, t.pos[S + d - 1], lane);
        d = c0;
        cur = X;
    }
    return 0;
}

// The walk of a queued request given its match at the start of the schedule
// step (chain S0, length m0, from K1).  Chains never grow and a cached depth
// of a chain implies its whole root path is cached, so if depth m0-1 of S0 is
// still cached the first m0 tokens still match without re-reading them; the
// walk only continues from m0 when m0 ends at a node boundary (an insert of
// this step may have added a child there).  Otherwise: full walk.
// COV: compute the pinned coverage (local tries; the routing index has no
// pins).  SEGS: record the path's chain segments (callers that edit the path).
template <int U = 8, bool COV = true, bool SEGS = true>
__device__ inline WalkOut warp_walk_hint(const TrieView &t, const int32_t *__restrict__ rq, int32_t len, int lane,
                                         Seg *segs, int64_t S0, int32_t m0, const Seg *pre = nullptr,
                                         int32_t pre_n = -1, int32_t tok_m0 = -1) {
    // pre / pre_n (optional, pre_n <= 32): the segments of [0, m0) recorded by
    // a batch-start walk of this same path (k_dispatch_prematch)
    int32_t y = -1;
    if (m0 > 0) {
        const int32_t c = t.pos[S0 + m0 - 1];
        if (pos_valid(t, c, S0, m0 - 1)) y = c;
    }
    auto store = [&](int64_t S, int32_t a, int32_t b, int32_t i) {
        if (SEGS && lane == 0) { segs[i].S = S; segs[i].a = a; segs[i].b = b; }
    };
    if (y < 0) return warp_walk_cb<U>(t, rq, len, lane, COV, store);
    WalkStart st;
    if ((SEGS || COV) && pre && pre_n >= 0 && pre_n <= 32) {
        if (lane < pre_n) segs[lane] = pre[lane];
        __syncwarp();
        st.nseg = pre_n;
    } else {
        st.nseg = SEGS || COV ? warp_path_segments(t, y, m0, segs, lane) : 0;
    }
    st.cov = 0;
    st.pinrun = COV;
    if (COV && st.nseg > 0 && st.nseg <= 32) {
        // every segment's top and bottom pin state in one round per lane; pinned
        // segments form a prefix of the path (refs never increase with depth)
        bool top_p = false, bot_p = false;
        int32_t botn = -1;
        if (lane < st.nseg) {
            const Seg g = segs[lane];
            const int32_t topn = t.pos[g.S + g.a];
            botn = t.pos[g.S + g.b - 1];
            top_p = t.ref[topn] > 0;
            bot_p = t.ref[botn] > 0;
        }
        const unsigned valid = st.nseg == 32 ? FS_FULL : ((1u << st.nseg) - 1u);
        const unsigned mtop = __ballot_sync(FS_FULL, top_p) & valid;
        const unsigned mbot = __ballot_sync(FS_FULL, bot_p) & valid;
        const int32_t kstar = (~mtop & valid) ? __ffs(~mtop & valid) - 1 : st.nseg;  // first unpinned top
        if (kstar == 0) {
            st.cov = segs[0].a;
            st.pinrun = false;
        } else {
            const int32_t kk = kstar - 1;
            const Seg g = segs[kk];
            const int32_t bk = __shfl_sync(FS_FULL, botn, kk);
            st.cov = ((mbot >> kk) & 1u) ? g.b : warp_seg_cov(t, g.S, g.a, g.b, bk, lane);
            st.pinrun = kk == st.nseg - 1 && st.cov == g.b;
        }
    } else {
        for (int32_t s = 0; COV && s < st.nseg && st.pinrun; s++) {
            const Seg g = segs[s];
            const int32_t last = t.pos[g.S + g.b - 1];
            st.cov = warp_seg_cov(t, g.S, g.a, g.b, last, lane);
            st.pinrun = st.cov == g.b;
        }
    }
    if (m0 < t.end[y]) {
        // K1 stopped inside y: the request's token there differs from the chain
        // (or the request ended) -- still true
        WalkOut o;
        o.mlen = m0; o.last = y; o.plen = m0 - t.start[y]; o.nseg = st.nseg; o.cov = st.cov;
        o.unpinned = m0 - st.cov;
        return o;
    }
    st.node = y; st.idx = m0; st.last = y;
    return warp_walk_from<U>(t, rq, len, lane, COV, st, store, tok_m0);
}

// warp_walk_cb storing the segments (lane 0) when segs != nullptr.
template <int U = 4, bool PIPE = false>
__device__ inline WalkOut warp_walk(const TrieView &t, const int32_t *__restrict__ rq, int32_t len, int lane,
                                    Seg *segs, bool want_cov) {
    auto store = [&](int64_t S, int32_t a, int32_t b, int32_t i) {
        if (lane == 0 && segs) { segs[i].S = S; segs[i].a = a; segs[i].b = b; }
    };
    return warp_walk_cb<U, decltype(store), PIPE>(t, rq, len, lane, want_cov, store);
}

// unpin (radix.py:180-185) of the cached root path arena[src : src+plen] by one
// warp: every node on it loses one reference; nodes reaching zero release
// their edge from pinned_tokens.  Warps unpinning different paths commute.
__device__ inline void warp_unpin_path(const TrieView &t, int32_t deepest, int lane) {
    // The path's nodes are the ancestors of its deepest node (RadixTree._chain,
    // radix.py:164-172), grouped in source chains.  Per chain, lane 0 follows up
    // to 8 parent links (a chain usually holds a few nodes); a chain split into
    // more nodes (nested prefixes) is finished by the whole warp scanning the
    // chain's remaining depths for node starts, 8 depths per lane per round.
    long long acc = 0;
    bool under = false;
    auto unpin1 = [&](int32_t n) {
        const int32_t el = elen(t, n);
        const int32_t old = atomicSub(&t.ref[n], 1);
        if (old <= 0) under = true;
        else if (old == 1) acc -= el;
    };
    int32_t cur = deepest, d = t.end[deepest];
    while (d > 0 && cur > 0) {
        const int64_t S = t.src[cur];
        const int32_t c0 = t.ctop[cur];
        const int32_t X = t.cpar[cur];
        int32_t rest = -1;  // chain depths [c0, rest) still to visit
        if (lane == 0) {
            int32_t n = cur;
            for (int k = 0; k < 8; k++) {
                unpin1(n);
                const int32_t st = t.start[n];
                if (st <= c0) { n = -1; break; }
                n = t.parent[n];
            }
            rest = n < 0 ? -1 : t.end[n];  // n (not yet visited) ends where the visited part starts
        }
        rest = __shfl_sync(FS_FULL, rest, 0);
        if (rest > c0) {
            constexpr int K = 8;
            for (int32_t p0 = c0 + lane; p0 < rest; p0 += 32 * K) {
                int32_t nd[K], st[K];
#pragma unroll
                for (int k = 0; k < K; k++) nd[k] = p0 + 32 * k < rest ? t.pos[S + p0 + 32 * k] : -1;
#pragma unroll
                for (int k = 0; k < K; k++) st[k] = nd[k] >= 0 ? t.start[nd[k]] : -1;
#pragma unroll
                for (int k = 0; k < K; k++)
                    if (nd[k] >= 0 && st[k] == p0 + 32 * k) unpin1(nd[k]);
            }
        }
        d = c0;
        cur = X;
    }
    if (acc) atomicAdd((unsigned long long *)&t.sc->pinned, (unsigned long long)acc);
    if (under) t.sc->status = FS_ERR_UNDERFLOW;
}

// ---------------------------------------------------------------- path nodes
// Call fn(node) once for every node of the path described by segs (each node
// is visited at its first depth).  Block-parallel; segs must be visible.
// The path's depths are flattened across its segments and each thread takes
// K of them: all K pos loads, then all K (start, end) loads, then the callbacks
// fn(node, start, end) -- a constant number of memory round trips per
// K*blockDim depths whatever the number of segments (fn's stores would
// otherwise pin every load behind them).
//
// Hop variant (FS_PATH_HOP, default): thread i owns a window of W consecutive
// flattened depths and reports the nodes STARTING in it -- one pos load at the
// window start, then hops node to node (pos at end[n]) until the window is
// passed.  Paths of long nodes (config 5: 1024-token levels) cost one
// pos + (start, end) round trip per thread instead of K of each.
#ifndef FS_PATH_HOP
#define FS_PATH_HOP 1
#endif
template <typename F>
__device__ inline void block_path_nodes(const TrieView &t, const Seg *segs, int32_t nseg, F fn, int32_t first = 0) {
    // threads [first, blockDim) take part (the others may be busy elsewhere)
#if FS_PATH_HOP
    {
        const int32_t nt = (int32_t)blockDim.x - first;
        if ((int32_t)threadIdx.x < first) return;
        int32_t total = 0;
        for (int32_t s = 0; s < nseg; s++) total += segs[s].b - segs[s].a;
        const int32_t W = (total + nt - 1) / nt;
        int32_t g = ((int32_t)threadIdx.x - first) * W;
        const int32_t hi = min(total, g + W);
        int32_t s = 0, base = 0;
        while (g < hi) {
            while (g - base >= segs[s].b - segs[s].a) { base += segs[s].b - segs[s].a; s++; }
            const int32_t d = segs[s].a + (g - base);
            const int32_t n = t.pos[segs[s].S + d];
            const int32_t st = t.start[n], en = t.end[n];
            if (st == d) fn(n, st, en);  // else: a node started before the window
            // next node: its first depth, clamped to the segment end
            g = base + min(en, segs[s].b) - segs[s].a;
        }
        return;
    }
#endif
    constexpr int K = 8;
    const int32_t nt = (int32_t)blockDim.x - first;
    if ((int32_t)threadIdx.x < first) return;
    int32_t total = 0;
    for (int32_t s = 0; s < nseg; s++) total += segs[s].b - segs[s].a;
    for (int32_t g0 = (int32_t)threadIdx.x - first; g0 < total; g0 += K * nt) {
        int32_t nd[K], dd[K];
        int32_t s = 0, base = 0;  // segment of depth index g (g increases with k)
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int32_t g = g0 + k * nt;
            nd[k] = -1;
            dd[k] = -1;
            if (g < total) {
                while (g - base >= segs[s].b - segs[s].a) { base += segs[s].b - segs[s].a; s++; }
                const int32_t d = segs[s].a + (g - base);
                dd[k] = d;
                nd[k] = t.pos[segs[s].S + d];
            }
        }
        int32_t st[K], en[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            st[k] = nd[k] >= 0 ? t.start[nd[k]] : -1;
            en[k] = nd[k] >= 0 ? t.end[nd[k]] : -1;
        }
#pragma unroll
        for (int k = 0; k < K; k++)
            if (nd[k] >= 0 && st[k] == dd[k]) fn(nd[k], st[k], en[k]);
    }
}

// pos[S + d] = n for d in [a, b)
__device__ inline void block_repoint(const TrieView &t, int64_t S, int32_t a, int32_t b, int32_t n) {
    for (int32_t d = a + (int32_t)threadIdx.x; d < b; d += blockDim.x) t.pos[S + d] = n;
}

// pin / unpin of a whole path (radix.py:164-185): ref +-1 on every node;
// pinned_tokens follows the 0 <-> 1 transitions.
__device__ inline void block_pin_path(const TrieView &t, const Seg *segs, int32_t nseg, int delta) {
    long long acc = 0;
    bool under = false;
    block_path_nodes(t, segs, nseg, [&](int32_t n, int32_t st, int32_t en) {
        const int32_t old = atomicAdd(&t.ref[n], delta);
        if (delta > 0 && old == 0) acc += en - st;
        if (delta < 0) {
            if (old <= 0) under = true;
            else if (old == 1) acc -= en - st;
        }
    });
    if (acc) atomicAdd((unsigned long long *)&t.sc->pinned, (unsigned long long)acc);
    if (under) t.sc->status = FS_ERR_UNDERFLOW;
}

// pin of a freshly admitted path whose pinned-token gain is known (len - cov,
// SURVEY a7'): fire-and-forget increments.
__device__ inline void block_pin_path_known(const TrieView &t, const Seg *segs, int32_t nseg, int64_t gain) {
    block_path_nodes(t, segs, nseg, [&](int32_t n, int32_t, int32_t) { atomicAdd(&t.ref[n], 1); });
    if (threadIdx.x == 0 && gain) atomicAdd((unsigned long long *)&t.sc->pinned, (unsigned long long)gain);
}

// ---------------------------------------------------------------- eviction
// RadixTree.evict_lru (radix.py:210-250) by one CTA.  The reference's candidate
// set (unprotected ref==0 leaves, parents re-added as they become leaves) is
// exactly "every current evictable leaf", so each pop is a block-wide argmin
// of (last_access, seq) over the node table; thread 0 detaches or truncates
// the winner and appends the record.  Protect set = FS_PROTECT flag.
__device__ __forceinline__ int32_t ld_acquire_i32(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_i32(int32_t *p, int32_t v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- cold eviction
// Asynchronous cold eviction (FEV) for the scheduler (k_schedule).  Within one
// fill every stamp lands on a queued request's path: K1 stamps each queued
// request's match (match_prefix in lpm_order, radix.py:86-90) with the fill's
// operation sequence sq1, and admissions stamp their own (pinned) paths.  A
// node whose own stamp predates sq1 and that is an evictable leaf -- "cold" --
// is therefore on no path any walk of this fill can take, no admission ever
// pins it, and (when every cold stamp is older than the fill's `now`, checked
// up front) every cold key (last_access, seq) is smaller than every other
// candidate's: the LRU pops of the fill start with the cold leaves in key
// order, whatever the admissions do.  While the cumulative eviction need stays
// within the cold leaves' tokens, the pops are fully determined by the sequence
// of per-admission needs, and each need is known as soon as the admission's
// walk is done (a partial truncation frees exactly what is left to free).  So
// the leader CTA only posts each need; a dedicated CTA performs the pops
// (records, detaches, parent re-joins) in order, concurrently with the
// following admissions.  Past the cold supply the leader drains the evictor
// and evicts itself (the serial path).
struct FevCtl {  // global, zeroed by the host per fill
    int32_t ready, ok, posted, stop, done, finished, err, pad_;
    int64_t C;                                   // cold candidate tokens at fill start
    int64_t freed, nrec, nfreed, tombs, pops;    // evictor totals (valid once finished)
    int32_t nc, heap_hw;                         // cold leaves sorted, re-join heap high water
};
struct FevLeader {  // leader CTA, shared memory
    FevCtl *ctl;
    int64_t *need;      // [orders] tokens to free
    int64_t *rec_end;   // [orders] records emitted after each order (evictor)
    int32_t *free_list; // node slots the evictor freed
    int32_t on, posted, cap_orders, ready_seen, used_any, nfree_saved;
    int32_t stamped;      // an existing node was stamped since the last post (fence before the next)
    int64_t cum, C, tag;  // tag: the fill's order tag (bits 40..62 of each posted need)
};

struct EvictSmem {
    int64_t la[32];
    int64_t sq[32];
    int32_t nd[32];
    int64_t freed;
    int32_t best;
    int64_t pops;
};

__device__ inline void block_evict(const TrieView &t, int64_t needed, EvictSmem *sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    if (tid == 0) sm->freed = 0;
    __syncthreads();
    while (true) {
        if (sm->freed >= needed) break;
        int64_t bla = INT64_MAX, bsq = INT64_MAX;
        int32_t bn = -1;
        const int32_t hw = t.sc->hw;
        for (int32_t n = 1 + tid; n < hw; n += blockDim.x) {
            const uint8_t f = t.flags[n];
            if ((f & FS_ALIVE) && !(f & FS_PROTECT) && t.nchild[n] == 0 && t.ref[n] == 0) {
                const int64_t a = t.la[n], s = t.seq[n];
                if (a < bla || (a == bla && s < bsq)) { bla = a; bsq = s; bn = n; }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const int64_t oa = __shfl_down_sync(FS_FULL, bla, off);
            const int64_t os = __shfl_down_sync(FS_FULL, bsq, off);
            const int32_t on = __shfl_down_sync(FS_FULL, bn, off);
            if (on >= 0 && (bn < 0 || oa < bla || (oa == bla && os < bsq))) { bla = oa; bsq = os; bn = on; }
        }
        if (lane == 0) { sm->la[warp] = bla; sm->sq[warp] = bsq; sm->nd[warp] = bn; }
        __syncthreads();
        if (tid == 0) {
            int64_t ba = INT64_MAX, bs = INT64_MAX;
            int32_t b = -1;
            for (int w = 0; w < nwarps; w++) {
                const int32_t on = sm->nd[w];
                if (on >= 0 && (b < 0 || sm->la[w] < ba || (sm->la[w] == ba && sm->sq[w] < bs))) {
                    ba = sm->la[w]; bs = sm->sq[w]; b = on;
                }
            }
            sm->best = b;
            if (b >= 0) {
                sm->pops++;
                const int32_t plen = t.end[b];  // len(full_path): the node's root-path length
                const int64_t remaining = needed - sm->freed;
                const int32_t el = elen(t, b);
                if (el <= remaining) {
                    push_record(t, t.src[b], plen, plen - el);
                    trie_detach(t, b);
                    sm->freed += el;
                } else {
                    // partial-edge eviction: drop the tail (radix.py:240-246)
                    push_record(t, t.src[b], plen, (int32_t)(plen - remaining));
                    t.end[b] -= (int32_t)remaining;
                    t.sc->used -= remaining;
                    sm->freed += remaining;
                }
            }
        }
        __syncthreads();
        if (sm->best < 0) break;
    }
    __syncthreads();
}

// ---------------------------------------------------------------- chunked LRU
// Inside one schedule step the evictable-leaf set only loses members (pins,
// detaches) or gains parents exposed by detaches, and no candidate's
// (last_access, seq) key changes (the only stamps are on admission paths,
// which are pinned).  The scheduler therefore keeps, in shared memory, the
// minimum key of every CH-node chunk of the node table: a pop is a warp-wide
// argmin over the chunk minima plus the rescan of the one or two chunks the
// pop changed -- no block barrier per pop.
#define FS_NCH 1024
struct ChunkLRU {
    int64_t la[FS_NCH];
    int64_t sq[FS_NCH];
    int32_t nd[FS_NCH];
    // minima of 32-chunk groups: a pop's argmin reads one entry per lane
    int64_t gla[FS_NCH / 32];
    int64_t gsq[FS_NCH / 32];
    int32_t gnd[FS_NCH / 32];
    int32_t ch;   // nodes per chunk (multiple of 32)
    int32_t nch;  // chunks covering [0, hw0)
    int32_t hw0;  // node-table size at the start of the step (later nodes are pinned)
    int64_t prof[4];  // pop cycles: argmin, edit, chunk update
};

#ifndef FS_POP_PREFETCH
#define FS_POP_PREFETCH 1
#endif
__device__ __forceinline__ void pf_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ bool lru_candidate(const TrieView &t, int32_t n) {
    return (t.flags[n] & FS_ALIVE) && t.nchild[n] == 0 && t.ref[n] == 0;
}

// warp-wide argmin over (la, sq, nd) triples; every lane gets the result
__device__ __forceinline__ void warp_key_min(int64_t &bla, int64_t &bsq, int32_t &bn) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const int64_t oa = __shfl_xor_sync(FS_FULL, bla, off);
        const int64_t os = __shfl_xor_sync(FS_FULL, bsq, off);
        const int32_t on = __shfl_xor_sync(FS_FULL, bn, off);
        if (on >= 0 && (bn < 0 || oa < bla || (oa == bla && os < bsq))) { bla = oa; bsq = os; bn = on; }
    }
}

// Warm this SM's L1 with what the next LRU pop will read: the current index
// minimum b (node fields), the nodes of b's chunk (the rescan), b's parent and
// the child-hash slot of (parent, first token) -- a hint only (every value is
// re-read by the pop; stores of this CTA keep L1 coherent).  One warp.
__device__ inline void warp_prefetch_pop(const TrieView &t, const ChunkLRU *L, int lane) {
    const int32_t ngroups = (L->nch + 31) / 32;
    int64_t bla = INT64_MAX, bsq = INT64_MAX;
    int32_t bn = -1;
    if (lane < ngroups) { bla = L->gla[lane]; bsq = L->gsq[lane]; bn = L->gnd[lane]; }
    warp_key_min(bla, bsq, bn);
    const int32_t b = bn;
    if (b <= 0) return;
    const int32_t lo = (b / L->ch) * L->ch, hi = min(lo + L->ch, L->hw0);
    for (int32_t n = lo + lane; n < hi; n += 32) {
        pf_l1(t.flags + n); pf_l1(t.nchild + n); pf_l1(t.ref + n); pf_l1(t.la + n); pf_l1(t.seq + n);
    }
    if (lane == 0) {
        pf_l1(t.start + b); pf_l1(t.end + b); pf_l1(t.src + b); pf_l1(t.lseq + b);
        const int32_t P = t.parent[b];
        const int32_t f = t.first[b];
        if (P >= 0) {
            pf_l1(t.nchild + P); pf_l1(t.ref + P); pf_l1(t.flags + P);
            pf_l1(t.la + P); pf_l1(t.lseq + P); pf_l1(t.seq + P);
            pf_l1(t.hslot + (fs_hmix(fs_hkey(P, f)) & t.hmask));
        }
    }
}

// Recompute the minimum of chunk group g (one warp).
__device__ inline void warp_group_update(ChunkLRU *L, int32_t g, int lane) {
    const int32_t c = g * 32 + lane;
    int64_t bla = INT64_MAX, bsq = INT64_MAX;
    int32_t bn = -1;
    if (c < L->nch) { bla = L->la[c]; bsq = L->sq[c]; bn = L->nd[c]; }
    warp_key_min(bla, bsq, bn);
    if (lane == 0) { L->gla[g] = bla; L->gsq[g] = bsq; L->gnd[g] = bn; }
    __syncwarp();
}

// Recompute the minimum of chunk c (one warp), leaving out node `exclude`.
__device__ inline void warp_chunk_scan(const TrieView &t, ChunkLRU *L, int32_t c, int32_t exclude, int lane) {
    int64_t bla = INT64_MAX, bsq = INT64_MAX;
    int32_t bn = -1;
    const int32_t lo = c * L->ch, hi = min(lo + L->ch, L->hw0);
    for (int32_t n = max(lo, 1) + lane; n < hi; n += 32) {
        if (n != exclude && lru_candidate(t, n)) {
            const int64_t a = t.la[n], s = t.seq[n];
            if (a < bla || (a == bla && s < bsq)) { bla = a; bsq = s; bn = n; }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const int64_t oa = __shfl_down_sync(FS_FULL, bla, off);
        const int64_t os = __shfl_down_sync(FS_FULL, bsq, off);
        const int32_t on = __shfl_down_sync(FS_FULL, bn, off);
        if (on >= 0 && (bn < 0 || oa < bla || (oa == bla && os < bsq))) { bla = oa; bsq = os; bn = on; }
    }
    if (lane == 0) { L->la[c] = bla; L->sq[c] = bsq; L->nd[c] = bn; }
    __syncwarp();
}

__device__ inline void block_chunk_build(const TrieView &t, ChunkLRU *L) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (threadIdx.x == 0) {
        L->hw0 = t.sc->hw;
        int32_t ch = (L->hw0 + FS_NCH - 1) / FS_NCH;
        ch = max(32, (ch + 31) & ~31);
        L->ch = ch;
        L->nch = (L->hw0 + ch - 1) / ch;
    }
    __syncthreads();
    for (int32_t c = warp; c < L->nch; c += nwarps) warp_chunk_scan(t, L, c, -1, lane);
    __syncthreads();
    for (int32_t g = warp; g * 32 < L->nch; g += nwarps) warp_group_update(L, g, lane);
    __syncthreads();
}

__device__ __forceinline__ void warp_chunk_touch(const TrieView &t, ChunkLRU *L, int32_t n, int32_t exclude,
                                                 int lane) {
    if (n > 0 && n < L->hw0) {
        const int32_t c = n / L->ch;
        warp_chunk_scan(t, L, c, exclude, lane);
        warp_group_update(L, c / 32, lane);
    }
}

// RadixTree.evict_lru with protect set {protect} (radix.py:210-250), one warp.
// ASYNC: the FEV evictor CTA (parents' child counts are shared with the
// leader's concurrent inserts: atomic).
template <bool ASYNC = false>
__device__ inline void warp_chunk_evict(const TrieView &t, ChunkLRU *L, int64_t needed, int32_t protect,
                                        EvictSmem *sm, int lane) {
    // The protected node (the path's deepest, just stamped) is rarely the LRU
    // minimum: it is dropped from its chunk's minimum only if it comes up.
    int64_t freed = 0;
    const int32_t ngroups = (L->nch + 31) / 32;
    while (freed < needed) {
        const long long p0 = clock64();
        int64_t bla = INT64_MAX, bsq = INT64_MAX;
        int32_t bn = -1;
        if (lane < ngroups) { bla = L->gla[lane]; bsq = L->gsq[lane]; bn = L->gnd[lane]; }
        warp_key_min(bla, bsq, bn);
        const int32_t b = bn;
        if (b < 0) break;
        // one round for everything the pop needs to know about b
        const uint8_t flb = t.flags[b];
        const int32_t ncb = t.nchild[b], refb = t.ref[b], stb = t.start[b], enb = t.end[b], Pb = t.parent[b];
        // Chunk minima may also name a node an earlier admission of this fill
        // pinned (or gave a child): block_admit leaves the index as is, and a
        // stale minimum is rescanned here when it comes up.
        if (b == protect || !((flb & FS_ALIVE) && ncb == 0 && refb == 0)) {
            warp_chunk_touch(t, L, b, protect, lane);
            continue;
        }
        const int32_t el = enb - stb;
        const bool whole = el <= needed - freed;
        __syncwarp();
        const long long p1 = clock64();
        // b is its chunk's minimum; a detach removes it, a truncation keeps
        // its key.  Lanes 1..31 rescan b's chunk without b (and without its
        // parent, whose state lane 0 is changing) while lane 0 edits.
        int64_t cla = INT64_MAX, csq = INT64_MAX;
        int32_t cn = -1;
        if (whole) {
            const int32_t c = b / L->ch;
            const int32_t lo = c * L->ch, hi = min(lo + L->ch, L->hw0);
            if (lane > 0)
                for (int32_t n = max(lo, 1) + lane - 1; n < hi; n += 31) {
                    if (n != b && n != Pb && n != protect && lru_candidate(t, n)) {
                        const int64_t x = t.la[n], s = t.seq[n];
                        if (x < cla || (x == cla && s < csq)) { cla = x; csq = s; cn = n; }
                    }
                }
        }
        int32_t P = -1;
        bool pcand = false;
        int64_t pla = 0, pseq = 0;
        if (lane == 0) {
            sm->pops++;
            const int32_t plen = enb;
            const int64_t remaining = needed - freed;
            if (whole) {
                // push_record + trie_detach (radix.py:206-208, 226-230) with every
                // load issued before the first store: two dependent rounds
                P = Pb;
                const int64_t srcb = t.src[b];
                const int32_t firstb = t.first[b];
                const int64_t lab = t.la[b], lsb = t.lseq[b];
                const int32_t ncP = ASYNC ? 0 : t.nchild[P], refP = t.ref[P];
                const uint8_t flP = t.flags[P];
                const int64_t laP = t.la[P], lsP = t.lseq[P], sqP = t.seq[P];
                const uint64_t key = fs_hkey(P, firstb);
                uint32_t hi = fs_hmix(key) & t.hmask;
                ulonglong2 hs = t.hslot[hi];
                for (uint32_t probes = 0; hs.x != key && hs.x != FS_HEMPTY && probes <= t.hmask; probes++) {
                    hi = (hi + 1) & t.hmask;
                    hs = t.hslot[hi];
                }
                push_record(t, srcb, plen, plen - el);
                if (hs.x == key) { t.hslot[hi].x = FS_HTOMB; atomicAdd(&t.sc->tombs, 1); }
                int32_t ncP1;
                if (ASYNC) {
                    ncP1 = atomicSub(&t.nchild[P], 1) - 1;
                } else {
                    ncP1 = ncP - 1;
                    t.nchild[P] = ncP1;
                }
                int64_t newla = laP;
                if (P > 0 && lsb > lsP) { t.la[P] = lab; t.lseq[P] = lsb; newla = lab; }
                t.sc->used -= el;
                node_free(t, b);
                freed += el;
                pcand = (flP & FS_ALIVE) && ncP1 == 0 && refP == 0;
                pla = newla;
                pseq = sqP;
            } else {
                push_record(t, t.src[b], plen, (int32_t)(plen - remaining));
                t.end[b] -= (int32_t)remaining;
                t.sc->used -= remaining;
                freed += remaining;
            }
        }
        freed = __shfl_sync(FS_FULL, freed, 0);
        P = __shfl_sync(FS_FULL, P, 0);
        const long long p2 = clock64();
        if (whole) {
            warp_key_min(cla, csq, cn);
            const int32_t c = b / L->ch;
            int32_t cp = -1;
            if (lane == 0) {
                L->la[c] = cla; L->sq[c] = csq; L->nd[c] = cn;
                // the parent joins the candidates once it becomes a leaf
                // (radix.py:231-239): its chunk minimum can only drop
                if (P > 0 && P < L->hw0 && P != protect && pcand) {
                    cp = P / L->ch;
                    const int64_t pa = pla, ps = pseq;
                    if (L->nd[cp] < 0 || pa < L->la[cp] || (pa == L->la[cp] && ps < L->sq[cp])) {
                        L->la[cp] = pa; L->sq[cp] = ps; L->nd[cp] = P;
                    }
                }
            }
            cp = __shfl_sync(FS_FULL, cp, 0);
            __syncwarp();
            warp_group_update(L, c / 32, lane);
            if (cp >= 0 && cp / 32 != c / 32) warp_group_update(L, cp / 32, lane);
        }
        __syncwarp();
        if (lane == 0) { L->prof[0] += p1 - p0; L->prof[1] += p2 - p1; L->prof[2] += clock64() - p2; }
    }
    if (lane == 0) sm->freed = freed;
    __syncwarp();
}

// ---------------------------------------------------------------- insert
#ifndef FS_CEV
#define FS_CEV 1  // scheduler inserts evict on warp 2 concurrently (block_insert)
#endif
struct InsertSmem {
    EvictSmem ev;
    int32_t nseg, mlen, new_len, deepest, last, status, cov, split_top;
    int32_t leaf, leaf_tok;  // scheduler: the new leaf, allocated when the walk ends (-1: not yet)
    int64_t needed, unpinned;
    int64_t *prof;  // optional cycle counters: [1] walk, [2] evict, [5] evict pops
    int64_t *prof2; // scheduler only: [0] pin, [2] waits for the evictor's setup
    ChunkLRU *lru;  // scheduler: chunked LRU index (nullptr: block-wide scan)
    FevLeader *fev; // scheduler: asynchronous cold eviction (nullptr: off)
    ChunkLRU *lru_spare;  // ... the leader's own index, built when FEV hands over
    int32_t fev_switch, fev_wait;
};

// Leader side: wait until the evictor has performed every posted need; with
// `handover`, also stop it and take over its state (records, freed node
// slots, hash tombstones) so the rest of the fill evicts serially.  Block-wide.
__device__ inline void fev_drain(const TrieView &t, FevLeader *f, bool handover) {
    FevCtl *c = f->ctl;
    if (threadIdx.x == 0) {
        while (ld_acquire_i32(&c->done) < f->posted) __nanosleep(32);
        if (handover) {
            st_release_i32(&c->stop, 1);
            while (ld_acquire_i32(&c->finished) == 0) __nanosleep(32);
            volatile FevCtl *vc = c;
            if (vc->err) t.sc->status = 100 + vc->err;  // evictor check (FS_FEV_CHECK) / heap overflow
            else if (vc->freed != f->cum) t.sc->status = FS_ERR_INTERNAL;
            t.sc->nrec = vc->nrec;
            t.sc->tombs += (int32_t)vc->tombs;
            t.sc->live -= (int32_t)vc->nfreed;
            t.sc->nfree = f->nfree_saved;
            f->on = 0;
        }
    }
    __syncthreads();
    (void)ld_acquire_i32(&c->done);  // every thread: drop L1 lines the evictor made stale
    if (handover) {
        const int32_t nf = (int32_t)((volatile FevCtl *)c)->nfreed;
        const int32_t base = t.sc->nfree;
        for (int32_t i = threadIdx.x; i < nf; i += blockDim.x) t.freest[base + i] = f->free_list[i];
        __syncthreads();
        if (threadIdx.x == 0) t.sc->nfree = base + nf;
    }
    __syncthreads();
}

// RadixTree.insert (radix.py:128-162) by one CTA (warp 0 walks).  `segs` is a
// global scratch of >= len+2 entries; on return it holds the whole path
// (including the new leaf) so the caller can pin it.  Leaves in sm: mlen (the
// match before the new leaf == probe()'s), unpinned/cov of that walk, deepest
// path node, status (FS_ERR_CACHE_FULL after performing the evictions, like
// the reference).
struct NoHook {
    __device__ void operator()(int) const {}
};

// pin_path (scheduler admissions): ref + 1 on every node of the new path.  The
// pre-existing path nodes are pinned by warps 2.. while warp 0 evicts (they are
// internal nodes or the protected deepest node, never eviction candidates),
// the new leaf when it is created.  Hooks (pin_path only): once the walk's
// results are known, warp 1 runs on_walk (lane 0) then on_side, concurrently
// with warp 0's eviction and the other warps' pin.
template <typename OnWalk = NoHook, typename OnSide = NoHook>
__device__ inline void block_insert(const TrieView &t, int64_t req_off, int32_t len, int64_t now, int64_t sq,
                                    int32_t worker, Seg *segs, InsertSmem *sm, int64_t hint_S0 = -1,
                                    int32_t hint_m0 = -1, bool pin_path = false, OnWalk on_walk = OnWalk(),
                                    OnSide on_side = OnSide(), const WalkOut *pre = nullptr,
                                    const Seg *pre_segs = nullptr, int32_t pre_nseg = -1, int32_t hint_tok0 = -1) {
    // hint_tok0 (optional): the request's token at hint_m0 (-1: unknown / none)
    // pre (warp 0, optional): the caller's own walk of this path with segments
    // written to segs, against the current tree (the dispatch chain's
    // longest_match_workers walk) -- reused instead of walking again
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t *rq = t.arena + req_off;
    const long long c0 = clock64();
    if (warp == 0) {
        // the routing index (worker tags) has no pins: no coverage to compute
        const WalkOut w = pre ? *pre
                        : hint_m0 >= 0 ? (t.wmask ? warp_walk_hint<8, false, true>(t, rq, len, lane, segs, hint_S0, hint_m0,
                                                                                   pre_segs, pre_nseg, hint_tok0)
                                                  : warp_walk_hint<8, true, true>(t, rq, len, lane, segs, hint_S0, hint_m0,
                                                                                  pre_segs, pre_nseg, hint_tok0))
                                       : warp_walk<8>(t, rq, len, lane, segs, t.wmask == nullptr);
        if (lane == 0) {
            int32_t last = w.last >= 0 ? w.last : 0;
            sm->split_top = -1;
            if (w.plen > 0) {
                const int32_t top = trie_split(t, w.last, w.plen);
                sm->split_top = top;
                last = top;
            }
            sm->nseg = w.nseg; sm->mlen = w.mlen; sm->unpinned = w.unpinned; sm->cov = w.cov;
            sm->new_len = len - w.mlen;
            sm->last = last;
            sm->status = t.sc->status;
            sm->needed = 0;
            sm->fev_switch = 0;
            sm->fev_wait = 0;
            const int64_t cap = t.sc->capacity;
            if (cap >= 0 && t.sc->used + sm->new_len > cap) {
                const int64_t need = t.sc->used + sm->new_len - cap;
                FevLeader *f = sm->fev;
                bool posted = false;
                if (f && f->on) {
                    if (!f->ready_seen) {
                        const long long cr = clock64();
                        while (ld_acquire_i32(&f->ctl->ready) == 0) __nanosleep(32);
                        if (sm->prof2) sm->prof2[2] += clock64() - cr;
                        f->C = ((volatile FevCtl *)f->ctl)->ok ? ((volatile FevCtl *)f->ctl)->C : -1;
                        f->ready_seen = 1;
                    }
                    if (f->cum + need <= f->C && f->posted < f->cap_orders) {
                        // within the cold supply: the evictor performs it --
                        // one relaxed store, after a fence when this thread
                        // stamped an existing node since the last order (the
                        // evictor compares stamps when a detached leaf's parent
                        // re-joins the candidates)
                        if (f->stamped) { __threadfence(); f->stamped = 0; }
                        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(f->need + f->posted),
                                     "l"(f->tag | need) : "memory");
                        f->posted++;
                        f->cum += need;
                        f->used_any = 1;
                        t.sc->used -= need;
                        posted = true;
                    } else {
                        sm->fev_switch = 1;  // past the cold supply: hand over, evict serially
                    }
                }
                if (!posted) {
                    // only the path's deepest node can be a leaf: every other path
                    // node has its path child below it (radix.py:149 protect=path)
                    if (last > 0) t.flags[last] |= FS_PROTECT;
                    sm->needed = need;
                }
            }
            // a fully cached request stamps an existing node: the evictor may be
            // pushing a detached child's stamp into it -- let it finish first
            if (sm->fev && sm->fev->on && !sm->fev_switch && sm->new_len == 0 && w.mlen > 0) sm->fev_wait = 1;
            // scheduler without FEV: the new leaf's slot, fields, pin and stamp
            // are set now, so its eviction can run on warp 2 concurrently with
            // the leaf's hash entry, the path pin and the bookkeeping (see
            // below).  The leaf's seq does not depend on the eviction (which
            // allocates none); used_tokens counts it now (the capacity test
            // after the eviction adjusts).
            sm->leaf = -1;
            if (FS_CEV && pin_path && sm->lru && !sm->fev && sm->status == FS_OK && sm->new_len > 0) {
                const int32_t tk = (w.mlen == hint_m0 && hint_tok0 >= 0) ? hint_tok0 : rq[w.mlen];
                const int32_t leaf = node_new(t, req_off, w.mlen, len, len, last, tk);
                if (leaf < 0) {
                    sm->status = FS_ERR_NOMEM;
                } else {
                    t.ref[leaf] = 1;  // pinned from birth: never an eviction candidate
                    t.la[leaf] = now;
                    t.lseq[leaf] = sq;
                    t.sc->used += sm->new_len;
                    sm->leaf = leaf;
                    sm->leaf_tok = tk;
                }
            }
        }
    }
#if FS_POP_PREFETCH
    else if (warp == 2 && sm->lru) {
        // idle until the pin: warm L1 for this insert's first LRU pop while warp 0 walks
        warp_prefetch_pop(t, sm->lru, lane);
    } else if (warp == 3 && sm->lru && lane == 0) {
        // ... and for the new leaf: the node slot it will likely take, the
        // scalars, its first token (the walk's hint depth)
        pf_l1(t.sc);
        const int32_t nf = t.sc->nfree;
        if (nf > 0) pf_l1(t.freest + nf - 1);
        if (hint_m0 >= 0 && hint_m0 < len) pf_l1(rq + hint_m0);
    }
#endif
    __syncthreads();
    if (sm->fev_switch || sm->fev_wait) {
        const bool ho = sm->fev_switch;
        fev_drain(t, sm->fev, ho);
        if (ho) {
            block_chunk_build(t, sm->lru_spare);
            if (threadIdx.x == 0) sm->lru = sm->lru_spare;
        }
        if (threadIdx.x == 0) { sm->fev_switch = 0; sm->fev_wait = 0; }
        __syncthreads();
    }
    if (sm->split_top >= 0)
        block_repoint(t, t.src[sm->split_top], t.start[sm->split_top], t.end[sm->split_top], sm->split_top);
    const long long c1 = clock64();
    if (tid == 0 && sm->prof) sm->prof[1] += c1 - c0;
    int32_t nseg_path = sm->nseg;
    if (pin_path) {
        // The new leaf comes first: pinned from birth it is never an eviction
        // candidate, and its sequence number does not depend on the evictions
        // (they allocate none) -- only its node slot may differ, which nothing
        // observes.  used_tokens counts it now; the capacity test below adjusts.
        // Warp 0 creates the leaf while warp 1 settles the scheduler state
        // (on_walk needs only the walk) and warps 2.. pin the pre-existing
        // path; the leaf's positions follow once it exists (named barrier 1:
        // warps 0 and 2..).
        // sm->leaf >= 0: warp 2 evicts (below) while warp 0 links the leaf
        const bool cev = sm->leaf >= 0;
        if (warp == 0) {
            if (lane == 0) {
                int32_t deepest = sm->mlen > 0 ? sm->last : -1;
                if (cev) {
                    h_put(t, sm->last, sm->leaf_tok, sm->leaf);
                    atomicAdd(&t.nchild[sm->last], 1);  // the eviction warp may decrement it
                    deepest = sm->leaf;
                } else if (sm->status == FS_OK && sm->new_len > 0) {
                    const int32_t tk = (sm->mlen == hint_m0 && hint_tok0 >= 0) ? hint_tok0 : rq[sm->mlen];
                    const int32_t leaf = node_new(t, req_off, sm->mlen, len, len, sm->last, tk);
                    if (leaf < 0) {
                        sm->status = FS_ERR_NOMEM;
                    } else {
                        h_put(t, sm->last, tk, leaf);
                        if (sm->fev && sm->fev->on) atomicAdd(&t.nchild[sm->last], 1);  // the evictor may decrement it
                        else t.nchild[sm->last]++;
                        t.ref[leaf] = 1;
                        t.sc->used += sm->new_len;
                        // (sm->nseg stays: the other warps read it concurrently;
                        // the leaf is pinned from birth, not by the path pin)
                        deepest = leaf;
                        t.la[leaf] = now;  // stamp of the whole path (lazy): a fresh node needs no compare
                        t.lseq[leaf] = sq;
                    }
                } else if (sm->status == FS_OK && deepest > 0) {
                    stamp_node(t, deepest, now, sq);
                    if (sm->fev) sm->fev->stamped = 1;
                }
                sm->deepest = deepest;
                if (sm->prof) sm->prof[13] += clock64() - c1;
            }
            // named barrier 1 (warps 0 and 3..), reached from two code paths:
            // the non-.aligned form (bar.sync is .aligned, which requires every
            // thread to execute the same barrier instruction)
            __syncwarp();
            asm volatile("barrier.sync 1, %0;" ::"r"((int)blockDim.x - 64) : "memory");
        } else if (warp == 2) {
            // RadixTree.evict_lru for this insert (radix.py:149-151), concurrent
            // with warp 0's hash link and the pin: the path's nodes are internal
            // or the protected deepest one, the new leaf is pinned, the leaf's
            // parent's child count is updated atomically by both sides
            if (cev && sm->needed > 0) {
                const long long ce = clock64();
                warp_chunk_evict<true>(t, sm->lru, sm->needed, sm->last, &sm->ev, lane);
                if (lane == 0 && sm->prof) sm->prof[2] += clock64() - ce;
            }
        } else if (warp > 2) {
            // pin the pre-existing path, then point the new leaf's depths at it
            const long long cp = clock64();
            block_path_nodes(t, segs, nseg_path, [&](int32_t n, int32_t, int32_t) { atomicAdd(&t.ref[n], 1); }, 96);
            __syncwarp();
            asm volatile("barrier.sync 1, %0;" ::"r"((int)blockDim.x - 64) : "memory");
            if (sm->status == FS_OK && sm->new_len > 0 && sm->deepest > 0) {
                // 16-B stores (arena rows, hence their pos rows, are 16-B aligned):
                // a quarter of the store instructions next to warp 1's bookkeeping
                int32_t *row = t.pos + req_off;
                const int32_t v = sm->deepest;
                const int32_t a0 = sm->mlen, a4 = min(len, (a0 + 3) & ~3), b4 = len & ~3;
                const int32_t nt = (int32_t)blockDim.x - 96, me = (int32_t)tid - 96;
                if (me < a4 - a0) row[a0 + me] = v;
                for (int32_t q = a4 / 4 + me; q < b4 / 4; q += nt)
                    reinterpret_cast<int4 *>(row)[q] = make_int4(v, v, v, v);
                if (b4 >= a4 && me < len - b4) row[b4 + me] = v;
            }
            if (tid == 96 && sm->prof2) sm->prof2[0] += clock64() - cp;
        } else if (warp == 1) {
            if (lane == 0) on_walk(0);
            __syncwarp();
            on_side(lane);
        }
        if (cev || !(sm->needed > 0 && sm->lru)) __syncthreads();
        if (cev && sm->needed > 0) {
            if (tid == 0) {
                if (sm->last > 0) t.flags[sm->last] &= ~FS_PROTECT;
                if (t.sc->used > t.sc->capacity) sm->status = FS_ERR_CACHE_FULL;
            }
            __syncthreads();
        }
    }
    if (sm->needed > 0 && !(pin_path && sm->leaf >= 0)) {
        if (sm->lru) {
            if (warp == 0) warp_chunk_evict(t, sm->lru, sm->needed, sm->last, &sm->ev, lane);
            __syncthreads();
        } else {
            block_evict(t, sm->needed, &sm->ev);
        }
        if (tid == 0 && sm->prof) sm->prof[2] += clock64() - c1;
        if (tid == 0) {
            if (sm->last > 0) t.flags[sm->last] &= ~FS_PROTECT;
            if (t.sc->used + (pin_path ? 0 : sm->new_len) > t.sc->capacity) sm->status = FS_ERR_CACHE_FULL;
        }
        __syncthreads();
    }
    if (pin_path) {
        if (tid == 0 && sm->status != FS_OK && t.sc->status == FS_OK && sm->status != FS_ERR_CACHE_FULL)
            t.sc->status = sm->status;
        return;  // the leaf, its positions and the pins are done
    }
    if (tid == 0) {
        int32_t deepest = sm->mlen > 0 ? sm->last : -1;
        if (sm->status == FS_OK && sm->new_len > 0) {
            const int32_t leaf = node_new(t, req_off, sm->mlen, len, len, sm->last);
            if (leaf < 0) {
                sm->status = FS_ERR_NOMEM;
            } else {
                h_put(t, sm->last, rq[sm->mlen], leaf);
                t.nchild[sm->last]++;
                if (pin_path) t.ref[leaf] = 1;
                t.sc->used += sm->new_len;
                segs[sm->nseg].S = req_off; segs[sm->nseg].a = sm->mlen; segs[sm->nseg].b = len;
                sm->nseg++;
                deepest = leaf;
                t.la[leaf] = now;  // stamp of the whole path (lazy): a fresh node needs no compare
                t.lseq[leaf] = sq;
            }
        }
        if (sm->status == FS_OK && deepest > 0 && !(sm->new_len > 0))
            stamp_node(t, deepest, now, sq);  // the whole path (lazy); a new leaf was stamped at creation
        sm->deepest = deepest;
        if (sm->status != FS_OK && t.sc->status == FS_OK && sm->status != FS_ERR_CACHE_FULL) t.sc->status = sm->status;
    }
    __syncthreads();
    const long long c2 = clock64();
    if (sm->status == FS_OK && sm->new_len > 0 && sm->deepest > 0)
        block_repoint(t, req_off, sm->mlen, len, sm->deepest);
    __syncthreads();
    const long long c3 = clock64();
    (void)c3;
    if (sm->status == FS_OK && t.wmask && worker >= 0) {
        // n.workers[worker] = now on every path node (radix.py:160-161)
        block_path_nodes(t, segs, sm->nseg, [&](int32_t n, int32_t, int32_t) {
            t.wmask[n] |= (1ull << worker);
            t.wtime[(int64_t)n * t.nw + worker] = now;
        });
        __syncthreads();
        if (tid == 0 && sm->prof) sm->prof[14] += clock64() - c3;
    }
}

// Segments of an existing root path arena[src : src+plen] (every node on it is
// cached): the walk of the handle's own path.  Block-level (warp 0 walks).
__device__ inline void block_path_of(const TrieView &t, int32_t deepest, Seg *segs, int32_t *nseg_out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
        const int32_t ns = warp_path_segments(t, deepest, t.end[deepest], segs, lane);
        if (lane == 0) *nseg_out = ns;
    }
    __syncthreads();
}

// ---------------------------------------------------------------- evict_notify
// RadixTree.evict_notify + _prune_up (radix.py:254-302).  The nodes the
// reference touches are the path nodes intersecting depths [keep, mlen) of the
// walk of `pth`; they are collected in path order and edited by thread 0.
#define FS_NF_CAP 64
struct NotifySmem {
    int32_t nseg, mlen, nf, top, fast;
    long long prof[4];  // cycles: walk, collect, edit (thread 0), repoint
    // the collected nodes with what the edit needs (first FS_NF_CAP of them)
    int32_t fnode[FS_NF_CAP], fstart[FS_NF_CAP];
    uint64_t fmask[FS_NF_CAP];
    uint8_t fhit[FS_NF_CAP];
};

// hint_m0 >= 0: the path's match against the index at the start of the notice
// batch (chain hint_S0); notices only remove strings, so a still-valid hint is
// the exact match (warp_walk_hint validates it and re-walks otherwise).
__device__ inline void block_evict_notify(const TrieView &t, int64_t psrc, int32_t plen, int32_t worker,
                                          int32_t keep, int64_t notice, Seg *segs, int32_t *found,
                                          NotifySmem *sm, int64_t hint_S0 = -1, int32_t hint_m0 = -1,
                                          int64_t next_S0 = -1, int32_t next_m0 = -1) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long q0 = clock64();
#if FS_POP_PREFETCH
    if (tid == 32 && next_m0 > 0) {
        // warp 1 idles in the fast path: warm L1 for the next notice's deepest
        // node, its parent and the child slot its prune will probe (hints only)
        const int32_t y2 = t.pos[next_S0 + next_m0 - 1];
        if (y2 > 0 && y2 < t.sc->hw) {
            pf_l1(t.flags + y2); pf_l1(t.src + y2); pf_l1(t.start + y2); pf_l1(t.end + y2);
            pf_l1(t.nchild + y2); pf_l1(t.ref + y2); pf_l1(t.wmask + y2);
            if (worker >= 0 && worker < t.nw) pf_l1(t.wtime + (int64_t)y2 * t.nw + worker);
            const int32_t P2 = t.parent[y2], f2 = t.first[y2];
            if (P2 >= 0) {
                pf_l1(t.nchild + P2); pf_l1(t.wmask + P2); pf_l1(t.ref + P2); pf_l1(t.la + P2); pf_l1(t.lseq + P2);
                pf_l1(t.hslot + (fs_hmix(fs_hkey(P2, f2)) & t.hmask));
            }
        }
    }
#endif
    // Fast path (thread 0): the batch-start match still holds and cannot be
    // extended (it stops inside its deepest node, or covers the whole path), so
    // the walk's answer is known, and the nodes intersecting [keep, mlen) are
    // the deepest node's ancestors down to depth keep -- collected up the
    // parent links with what the edit needs, no segment list or depth scan.
    if (tid == 0) {
        sm->fast = 0;
        if (hint_m0 > 0) {
            const int32_t y = t.pos[hint_S0 + hint_m0 - 1];
            if (pos_valid(t, y, hint_S0, hint_m0 - 1) && (hint_m0 < t.end[y] || hint_m0 == plen)) {
                int32_t nf = 0;
                bool ok = true;
                for (int32_t n = y; n > 0 && keep < hint_m0; n = t.parent[n]) {
                    const int32_t st = t.start[n];
                    if (nf == FS_NF_CAP) { ok = false; break; }
                    const uint64_t wm = t.wmask[n];
                    const int64_t wt = worker >= 0 && worker < t.nw ? t.wtime[(int64_t)n * t.nw + worker] : 0;
                    sm->fnode[nf] = n; sm->fstart[nf] = st; sm->fmask[nf] = wm;
                    sm->fhit[nf] = worker >= 0 && worker < 64 && ((wm >> worker) & 1ull) && wt <= notice;
                    found[nf] = n;
                    nf++;
                    if (st <= keep) break;  // this node holds depth keep
                }
                if (ok) {
                    // ancestors were collected deepest first: path order is the reverse
                    for (int32_t i = 0; i < nf / 2; i++) {
                        const int32_t k = nf - 1 - i;
                        int32_t tn = sm->fnode[i]; sm->fnode[i] = sm->fnode[k]; sm->fnode[k] = tn;
                        int32_t ts = sm->fstart[i]; sm->fstart[i] = sm->fstart[k]; sm->fstart[k] = ts;
                        uint64_t tm = sm->fmask[i]; sm->fmask[i] = sm->fmask[k]; sm->fmask[k] = tm;
                        uint8_t th = sm->fhit[i]; sm->fhit[i] = sm->fhit[k]; sm->fhit[k] = th;
                    }
                    sm->nf = nf;
                    sm->mlen = hint_m0;
                    sm->fast = 1;
                }
            }
        }
    }
    __syncthreads();
    if (!sm->fast && warp == 0) {
        const WalkOut w = hint_m0 >= 0 ? warp_walk_hint<8, false, true>(t, t.arena + psrc, plen, lane, segs, hint_S0, hint_m0)
                                       : warp_walk<8>(t, t.arena + psrc, plen, lane, segs, false);
        if (lane == 0) { sm->nseg = w.nseg; sm->mlen = w.mlen; sm->nf = 0; }
    }
    __syncthreads();
    const long long q1 = clock64();
    const int32_t mlen = sm->mlen;
    if (!sm->fast && keep < mlen) {
        // nodes covering a depth in [keep, mlen): the node holding `keep` (visited
        // at depth keep) and every node starting inside the range; depths batched
        // K per thread (all pos loads, then all start loads)
        constexpr int K = 8;
        const int32_t nt_ = (int32_t)blockDim.x;
        for (int32_t s = 0; s < sm->nseg; s++) {
            const int64_t S = segs[s].S;
            const int32_t a = max(segs[s].a, keep), b = segs[s].b;
            for (int32_t d0 = a + tid; d0 < b; d0 += K * nt_) {
                int32_t nd[K], st[K];
#pragma unroll
                for (int k = 0; k < K; k++) nd[k] = d0 + k * nt_ < b ? t.pos[S + d0 + k * nt_] : -1;
#pragma unroll
                for (int k = 0; k < K; k++) st[k] = nd[k] >= 0 ? t.start[nd[k]] : -1;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int32_t d = d0 + k * nt_;
                    if (nd[k] >= 0 && (st[k] == d || d == keep)) {
                        // the tag test in parallel (loads issued before the
                        // append): the edit below only stores
                        const uint64_t wm = t.wmask[nd[k]];
                        const int64_t wt = worker >= 0 && worker < t.nw ? t.wtime[(int64_t)nd[k] * t.nw + worker] : 0;
                        const int32_t slot = atomicAdd(&sm->nf, 1);
                        found[slot] = nd[k];
                        if (slot < FS_NF_CAP) {
                            sm->fnode[slot] = nd[k];
                            sm->fstart[slot] = st[k];
                            sm->fmask[slot] = wm;
                            sm->fhit[slot] = worker >= 0 && worker < 64 && ((wm >> worker) & 1ull) && wt <= notice;
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    const long long q2 = clock64();
    if (tid == 0 && sm->nf <= FS_NF_CAP) {
        // the usual case: everything the edit reads was collected above
        const int32_t nf = sm->nf;
        sm->top = -1;
        for (int32_t i = 1; i < nf; i++) {  // path order == increasing start depth
            const int32_t xn = sm->fnode[i], xs = sm->fstart[i];
            const uint64_t xm = sm->fmask[i];
            const uint8_t xh = sm->fhit[i];
            int32_t j = i - 1;
            while (j >= 0 && sm->fstart[j] > xs) {
                sm->fnode[j + 1] = sm->fnode[j]; sm->fstart[j + 1] = sm->fstart[j];
                sm->fmask[j + 1] = sm->fmask[j]; sm->fhit[j + 1] = sm->fhit[j];
                j--;
            }
            sm->fnode[j + 1] = xn; sm->fstart[j + 1] = xs; sm->fmask[j + 1] = xm; sm->fhit[j + 1] = xh;
        }
        int32_t nt = 0;
        for (int32_t i = 0; i < nf; i++) {
            const int32_t nd = sm->fnode[i];
            if (sm->fstart[i] < keep) sm->top = trie_split(t, nd, keep - sm->fstart[i]);
            if (sm->fhit[i]) {
                t.wmask[nd] = sm->fmask[i] & ~(1ull << worker);
                found[nt++] = nd;
            }
        }
        for (int32_t i = 0; i < nt; i++) {
            int32_t n = found[i];
            while (n > 0 && t.nchild[n] == 0 && t.wmask[n] == 0 && t.ref[n] == 0) {
                const int32_t P = t.parent[n];
                if (P < 0) break;
                if (h_find(t, P, t.first[n]) == n) trie_detach(t, n); else break;
                n = P;
            }
        }
    } else if (tid == 0) {
        const int32_t nf = sm->nf;
        sm->top = -1;
        // path order == increasing start depth
        for (int32_t i = 1; i < nf; i++) {
            const int32_t x = found[i];
            int32_t j = i - 1;
            while (j >= 0 && t.start[found[j]] > t.start[x]) { found[j + 1] = found[j]; j--; }
            found[j + 1] = x;
        }
        int32_t nt = 0;
        for (int32_t i = 0; i < nf; i++) {
            const int32_t nd = found[i];
            const int32_t s = t.start[nd];
            if (s < keep) {
                // top survives with the tag; its positions are re-pointed by the block below
                sm->top = trie_split(t, nd, keep - s);
            }
            if (worker >= 0 && worker < 64 && ((t.wmask[nd] >> worker) & 1ull) &&
                t.wtime[(int64_t)nd * t.nw + worker] <= notice) {
                t.wmask[nd] &= ~(1ull << worker);
                found[nt++] = nd;  // touched (slot i already consumed)
            }
        }
        for (int32_t i = 0; i < nt; i++) {
            int32_t n = found[i];
            while (n > 0 && t.nchild[n] == 0 && t.wmask[n] == 0 && t.ref[n] == 0) {
                const int32_t P = t.parent[n];
                if (P < 0) break;
                if (h_find(t, P, t.first[n]) == n) trie_detach(t, n); else break;
                n = P;
            }
        }
    }
    __syncthreads();
    const long long q3 = clock64();
    if (sm->top >= 0) {
        const int32_t top = sm->top;
        block_repoint(t, t.src[top], t.start[top], t.end[top], top);
        __syncthreads();
    }
    if (tid == 0) {
        sm->prof[0] += q1 - q0; sm->prof[1] += q2 - q1; sm->prof[2] += q3 - q2; sm->prof[3] += clock64() - q3;
    }
}
