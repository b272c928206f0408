// fs_device.cuh -- device-side data model and primitives of the B200-native
// DLPM / D^2LPM decision path (arXiv 2501.14312).
//
// Data model (HBM):
//   * token arena: every request's int32 tokens, uploaded once, 16-B aligned.
//   * radix trie (one per RadixTree, radix.py:48): SoA node table.  A node does
//     not own tokens: its root path is arena[src : src+end] (a prefix of the
//     request that created it) and its edge is arena[src+start : src+end].
//     Splits and partial evictions only move start/end -- no token copies.
//   * children: one open-addressing hash (parent, first token) -> child,
//     linear probing with backward-shift deletion (no tombstones).
//
// All structural edits are done by a single thread of a single CTA (the
// reference is single-writer); token compares are warp-wide
// (32 lanes x 4 tokens per step, ballot + ffs for the first mismatch).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FS_FULL 0xffffffffu
#define FS_HEMPTY 0xffffffffffffffffull

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
};

struct TrieView {
    const int32_t *arena;
    int64_t *src;
    int32_t *start, *end, *parent, *nchild, *ref, *first;
    int64_t *la, *seq;
    uint8_t *flags;
    uint64_t *wmask;  // nullptr unless track_workers
    int64_t *wtime;   // [node * nw + w]
    int32_t nw;
    uint64_t *hkeys;
    int32_t *hvals;
    uint32_t hmask;
    int32_t *freest;
    int32_t ncap;
    TrieScalars *sc;
    int64_t *rsrc;  // eviction-record sink
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
    while (true) {
        const uint64_t k = t.hkeys[i];
        if (k == key) return t.hvals[i];
        if (k == FS_HEMPTY) return -1;
        i = (i + 1) & t.hmask;
    }
}
// children[tok] = child
__device__ inline void h_put(const TrieView &t, int32_t p, int32_t tok, int32_t child) {
    const uint64_t key = fs_hkey(p, tok);
    uint32_t i = fs_hmix(key) & t.hmask;
    while (true) {
        const uint64_t k = t.hkeys[i];
        if (k == key || k == FS_HEMPTY) { t.hkeys[i] = key; t.hvals[i] = child; return; }
        i = (i + 1) & t.hmask;
    }
}
// del children[tok] -- backward-shift deletion keeps probe chains intact
__device__ inline void h_del(const TrieView &t, int32_t p, int32_t tok) {
    const uint64_t key = fs_hkey(p, tok);
    uint32_t i = fs_hmix(key) & t.hmask;
    while (t.hkeys[i] != key) {
        if (t.hkeys[i] == FS_HEMPTY) return;
        i = (i + 1) & t.hmask;
    }
    uint32_t j = i;
    while (true) {
        j = (j + 1) & t.hmask;
        const uint64_t kj = t.hkeys[j];
        if (kj == FS_HEMPTY) break;
        const uint32_t h = fs_hmix(kj) & t.hmask;
        const bool stay = (i <= j) ? (i < h && h <= j) : (i < h || h <= j);
        if (stay) continue;
        t.hkeys[i] = kj; t.hvals[i] = t.hvals[j];
        i = j;
    }
    t.hkeys[i] = FS_HEMPTY;
}

// ---------------------------------------------------------------- nodes
// RadixNode(...) with seq = self._seq; self._seq += 1  (radix.py:117-118, 153-154)
__device__ inline int32_t node_new(const TrieView &t, int64_t src, int32_t start, int32_t end, int32_t parent) {
    int32_t n;
    if (t.sc->nfree > 0) n = t.freest[--t.sc->nfree];
    else if (t.sc->hw < t.ncap) n = t.sc->hw++;
    else { t.sc->status = FS_ERR_NOMEM; return -1; }
    t.src[n] = src; t.start[n] = start; t.end[n] = end; t.parent[n] = parent;
    t.nchild[n] = 0; t.ref[n] = 0; t.la[n] = 0;
    t.seq[n] = t.sc->next_seq++;
    t.first[n] = t.arena[src + start];
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

// RadixTree._split (radix.py:114-126): top gets a new seq, copies ref /
// last_access / workers; the bottom keeps its identity (and seq).
__device__ inline int32_t trie_split(const TrieView &t, int32_t node, int32_t k) {
    const int32_t P = t.parent[node];
    const int32_t top = node_new(t, t.src[node], t.start[node], t.start[node] + k, P);
    if (top < 0) return -1;
    t.ref[top] = t.ref[node];
    t.la[top] = t.la[node];
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

// RadixTree._detach (radix.py:206-208)
__device__ inline void trie_detach(const TrieView &t, int32_t n) {
    const int32_t P = t.parent[n];
    h_del(t, P, t.first[n]);
    t.nchild[P]--;
    t.sc->used -= elen(t, n);
    node_free(t, n);
}

__device__ inline void push_record(const TrieView &t, int64_t src, int32_t len, int32_t keep) {
    const int64_t i = t.sc->nrec++;
    if (i < t.rcap) { t.rsrc[i] = src; t.rlen[i] = len; t.rkeep[i] = keep; }
}

// pin / unpin via _chain (radix.py:164-185): deepest node up to the root
__device__ inline void pin_chain(const TrieView &t, int32_t n) {
    while (n > 0) {
        if (t.ref[n] == 0) t.sc->pinned += elen(t, n);
        t.ref[n]++;
        n = t.parent[n];
    }
}
__device__ inline void unpin_chain(const TrieView &t, int32_t n) {
    while (n > 0) {
        t.ref[n]--;
        if (t.ref[n] < 0) { t.sc->status = FS_ERR_UNDERFLOW; t.ref[n] = 0; return; }
        if (t.ref[n] == 0) t.sc->pinned -= elen(t, n);
        n = t.parent[n];
    }
}

// ---------------------------------------------------------------- compare
// LCP of a[0:n) and b[0:n) by one warp: 128 tokens per step, first mismatch
// by ballot + ffs (common_prefix_len, _speedups.pyx:11-22, at warp width).
// `a` is trie edge data (hot, read-only path), `b` the request stream (read
// once: streaming loads so it does not evict the trie from L1/L2).
__device__ __forceinline__ int32_t warp_lcp(const int32_t *__restrict__ a, const int32_t *__restrict__ b,
                                            int32_t n, int lane) {
    int32_t k = 0;
    while (k < n) {
        bool bad[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int32_t p = k + u * 32 + lane;
            bad[u] = (p < n) && (__ldg(a + p) != __ldcs(b + p));
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const unsigned m = __ballot_sync(FS_FULL, bad[u]);
            if (m) return min(n, k + u * 32 + __ffs(m) - 1);
        }
        k += 128;
    }
    return n;
}

struct WalkOut {
    int32_t mlen;       // match length
    int32_t last_full;  // deepest fully matched node, -1 if none
    int32_t partial;    // partially matched child, -1 if none
    int32_t plen;       // tokens matched inside partial
    int32_t cov;        // matched tokens inside pinned nodes (pinned coverage B)
    int32_t fnode;      // node holding depth `cov` (0 = root)
    int32_t npath;      // nodes written to `path` (full nodes + partial)
    int64_t unpinned;   // probe()'s matched-unpinned count (radix.py:96-98)
};

// RadixTree._walk (radix.py:60-81) by one warp, optionally stamping
// last_access = now on every full node and the partial node (radix.py:86-90).
// All lanes return the same WalkOut; lane 0 writes stamps / path entries.
__device__ inline WalkOut warp_walk(const TrieView &t, const int32_t *__restrict__ rq, int32_t len, int lane,
                                    bool stamp, int64_t now, int32_t *path) {
    WalkOut o;
    o.mlen = 0; o.last_full = -1; o.partial = -1; o.plen = 0; o.cov = 0; o.fnode = 0; o.npath = 0; o.unpinned = 0;
    int32_t node = 0, idx = 0;
    bool pinrun = true;
    while (idx < len) {
        const int32_t c = h_find(t, node, __ldcs(rq + idx));
        if (c < 0) break;
        const int32_t cs = t.start[c];
        const int32_t el = t.end[c] - cs;
        const int32_t n = min(el, len - idx);
        const int32_t k = 1 + warp_lcp(t.arena + t.src[c] + cs + 1, rq + idx + 1, n - 1, lane);
        const int32_t r = t.ref[c];
        if (pinrun) {
            if (r > 0) { o.cov = idx + k; o.fnode = c; } else pinrun = false;
        }
        if (r == 0) o.unpinned += k;
        if (lane == 0) {
            if (stamp && t.la[c] != now) t.la[c] = now;
            if (path) path[o.npath] = c;
        }
        o.npath++;
        idx += k;
        if (k < el) { o.partial = c; o.plen = k; break; }
        o.last_full = c;
        node = c;
    }
    o.mlen = idx;
    return o;
}

// ---------------------------------------------------------------- eviction
// RadixTree.evict_lru (radix.py:210-250) by one CTA.  The candidate set of the
// reference (unprotected ref==0 leaves, parents re-added as they become leaves)
// is exactly "every current evictable leaf", so each pop is a block-wide
// argmin of (last_access, seq) over the node table; thread 0 detaches or
// truncates the winner and appends the record.  Protect set = FS_PROTECT flag.
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

// ---------------------------------------------------------------- insert
struct InsertSmem {
    EvictSmem ev;
    int32_t np, mlen, new_len, deepest, last, status, cov, fnode;
    int64_t needed, unpinned;
    int64_t *prof;  // optional cycle counters: [1] walk, [2] evict, [5] evict pops
};

// RadixTree.insert (radix.py:128-162) by one CTA (warp 0 walks).  `path` is a
// global scratch of >= len+2 entries.  Leaves in sm: mlen (idx before the new
// leaf), unpinned/cov of the pre-insert walk (== probe()), deepest path node,
// status (FS_ERR_CACHE_FULL after performing the evictions, like the reference).
__device__ inline void block_insert(const TrieView &t, int64_t req_off, int32_t len, int64_t now,
                                    int32_t worker, int32_t *path, InsertSmem *sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t *rq = t.arena + req_off;
    const long long c0 = clock64();
    if (warp == 0) {
        const WalkOut w = warp_walk(t, rq, len, lane, false, 0, path);
        if (lane == 0) {
            int32_t np = w.npath;
            int32_t last = np ? path[np - 1] : 0;
            if (w.partial >= 0) {
                const int32_t top = trie_split(t, w.partial, w.plen);
                path[np - 1] = top;
                last = top;
            }
            sm->np = np; sm->mlen = w.mlen; sm->unpinned = w.unpinned; sm->cov = w.cov; sm->fnode = w.fnode;
            sm->new_len = len - w.mlen;
            sm->last = last;
            sm->status = t.sc->status;
            sm->needed = 0;
            const int64_t cap = t.sc->capacity;
            if (cap >= 0 && t.sc->used + sm->new_len > cap) {
                for (int32_t i = 0; i < np; i++) t.flags[path[i]] |= FS_PROTECT;
                sm->needed = t.sc->used + sm->new_len - cap;
            }
        }
    }
    __syncthreads();
    const long long c1 = clock64();
    if (tid == 0 && sm->prof) sm->prof[1] += c1 - c0;
    if (sm->needed > 0) {
        block_evict(t, sm->needed, &sm->ev);
        if (tid == 0 && sm->prof) sm->prof[2] += clock64() - c1;
        if (tid == 0) {
            for (int32_t i = 0; i < sm->np; i++) t.flags[path[i]] &= ~FS_PROTECT;
            if (t.sc->used + sm->new_len > t.sc->capacity) sm->status = FS_ERR_CACHE_FULL;
        }
        __syncthreads();
    }
    if (tid == 0) {
        int32_t np = sm->np;
        if (sm->status == FS_OK) {
            if (sm->new_len > 0) {
                const int32_t leaf = node_new(t, req_off, sm->mlen, len, sm->last);
                if (leaf < 0) {
                    sm->status = FS_ERR_NOMEM;
                } else {
                    h_put(t, sm->last, rq[sm->mlen], leaf);
                    t.nchild[sm->last]++;
                    t.sc->used += sm->new_len;
                    path[np++] = leaf;
                }
            }
            for (int32_t i = 0; i < np; i++) {
                const int32_t n = path[i];
                t.la[n] = now;
                if (t.wmask && worker >= 0) {
                    t.wmask[n] |= (1ull << worker);
                    t.wtime[(int64_t)n * t.nw + worker] = now;
                }
            }
        }
        sm->np = np;
        sm->deepest = np ? path[np - 1] : -1;
        if (sm->status != FS_OK && t.sc->status == FS_OK && sm->status != FS_ERR_CACHE_FULL) t.sc->status = sm->status;
    }
    __syncthreads();
}

// ---------------------------------------------------------------- evict_notify
// RadixTree.evict_notify + _prune_up (radix.py:254-302), single thread for the
// structure edits, warp for the compares.  `scratch` holds >= 2*(plen+2) ints.
__device__ inline void warp_evict_notify(const TrieView &t, const int32_t *pth, int32_t plen, int32_t worker,
                                         int32_t keep, int64_t notice, int32_t *scratch) {
    const int lane = threadIdx.x & 31;
    int32_t *fnode = scratch;
    int32_t *fstart = scratch + plen + 2;
    int32_t nf = 0;
    int32_t node = 0, idx = 0;
    while (idx < plen) {
        const int32_t c = h_find(t, node, pth[idx]);
        if (c < 0) break;
        const int32_t el = elen(t, c);
        const int32_t n = min(el, plen - idx);
        const int32_t k = 1 + warp_lcp(t.arena + t.src[c] + t.start[c] + 1, pth + idx + 1, n - 1, lane);
        if (k < el) {
            if (k > 0 && idx + k > keep) { fnode[nf] = c; fstart[nf] = idx; nf++; }
            break;
        }
        fnode[nf] = c; fstart[nf] = idx; nf++;
        idx += k;
        node = c;
    }
    __syncwarp();
    if (lane == 0) {
        int32_t nt = 0;
        int32_t *touched = fstart;  // reuse: entry i consumed before slot i is written
        for (int32_t i = 0; i < nf; i++) {
            const int32_t nd = fnode[i];
            const int32_t s = fstart[i];
            const int32_t e = s + elen(t, nd);
            if (e <= keep) continue;
            if (s < keep) trie_split(t, nd, keep - s);  // top survives with the tag
            if (worker >= 0 && worker < 64 && ((t.wmask[nd] >> worker) & 1ull) &&
                t.wtime[(int64_t)nd * t.nw + worker] <= notice) {
                t.wmask[nd] &= ~(1ull << worker);
                touched[nt++] = nd;
            }
        }
        for (int32_t i = 0; i < nt; i++) {
            int32_t n = touched[i];
            while (n > 0 && t.nchild[n] == 0 && t.wmask[n] == 0 && t.ref[n] == 0) {
                const int32_t P = t.parent[n];
                if (P < 0) break;
                if (h_find(t, P, t.first[n]) == n) trie_detach(t, n); else break;
                n = P;
            }
        }
    }
    __syncwarp();
}
