/*
 * fairsched_b200.h -- C ABI of the B200-native DLPM / D^2LPM decision path.
 *
 * One shared library (paper_2501_14312_b200/libfsb200.so) built for sm_100a.
 * Plain pointers and sizes only; no torch types cross this boundary.  Every
 * entry point returns an fs status code; on failure fs_last_error() returns a
 * thread-local message.  No exception crosses the ABI and there is no CPU
 * fallback: without a usable CUDA device every call fails with FS_ERR_CUDA.
 *
 * The reference (`fairsched`, arXiv 2501.14312) has no native FFI for this
 * path except `common_prefix_len` (pkg/src/fairsched/_speedups.pyx:11-22); its
 * plug points are Python protocols.  Each group below names the reference
 * interface it replaces (paths relative to /root/reference/pkg/src/fairsched).
 * INTEGRATION.md shows the ctypes binding the Python adapters use.
 *
 * Ownership: the library owns all device state behind opaque handles.  Host
 * buffers passed in are read (or written) before the call returns.
 * Threading: one handle is used by one thread at a time; calls are ordered on
 * the handle's CUDA stream and are synchronous unless stated otherwise.
 */
#ifndef FAIRSCHED_B200_H
#define FAIRSCHED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors of radix.py:19 / :183, local_policies.py:81-82,
 * global_policies.py:97-98 map onto these) */
#define FS_OK 0
#define FS_ERR_INVALID 1     /* bad argument (ValueError in the reference)          */
#define FS_ERR_CUDA 2        /* CUDA runtime / no device                            */
#define FS_ERR_CACHE_FULL 3  /* radix.py:150-151 CacheFull                          */
#define FS_ERR_TOKEN_RANGE 4 /* token id outside [0, 2^31) (requests.py:92)         */
#define FS_ERR_NOMEM 5       /* device allocation / table capacity                  */
#define FS_ERR_INTERNAL 6    /* device-side consistency check failed                */
#define FS_ERR_UNDERFLOW 7   /* radix.py:183 unpin below zero                       */

typedef struct fs_ctx fs_ctx;               /* one device: token arena + request pool */
typedef struct fs_trie fs_trie;             /* one RadixTree (local or global)        */
typedef struct fs_worker fs_worker;         /* one DLPM/LPM worker policy             */
typedef struct fs_dispatcher fs_dispatcher; /* one D2LPM dispatcher                   */

const char *fs_last_error(void);
int fs_version(void);
int fs_device_count(int *count);

/* ---- context / request pool ------------------------------------------------
 * Replaces the Python Request objects' token tuples (requests.py:22-32,
 * Trace.materialize requests.py:134-161): tokens are uploaded once per request
 * into a device arena and referenced by request id from then on.            */
int fs_ctx_create(int device, int64_t arena_tokens, int64_t max_requests, fs_ctx **out);
/* Page-lock a caller buffer (cudaHostRegister) so fs_requests_add uploads from
 * it by DMA; unregister before freeing it. */
int fs_host_register(void *ptr, int64_t bytes);
int fs_host_unregister(void *ptr);
int fs_ctx_destroy(fs_ctx *ctx);
int fs_ctx_sync(fs_ctx *ctx);
/* Append n requests.  tokens: concatenated ids, offsets[i]/lens[i] index them;
 * clients: dense client ids; labels: order key of (arrival, rid) used as the
 * LPM tie-break (local_policies.py:17).  Writes the new request ids.  When the
 * requests are back to back in `tokens` the block is copied in one transfer and
 * range-checked on the device (FS_ERR_TOKEN_RANGE leaves nothing appended). */
int fs_requests_add(fs_ctx *ctx, int64_t n, const int32_t *tokens, const int64_t *offsets,
                    const int32_t *lens, const int32_t *clients, const int64_t *labels,
                    int32_t *out_ids);
/* Trace.materialize / expand_tokens / _token_block (requests.py:89-102, 134-161)
 * on the device: append n requests whose tokens are generated in the arena.
 * Request i is the concatenation of segments [seg_first[i], seg_first[i+1]);
 * segment s is expand_tokens(ns, seg_len[s]) for namespace ns = seg_ns[s],
 * i.e. blocks sha256(f"{ns}#{b}") -> 8 big-endian words % 2^31.  Namespace k
 * is the UTF-8 string ns_bytes[ns_off[k] : ns_off[k]+ns_len[k]].  A "req:<rid>"
 * prefix is passed as the parent's leading segments (every segment starts at
 * block 0 of its namespace).  clients/labels as in fs_requests_add. */
int fs_requests_add_expanded(fs_ctx *ctx, int64_t n, const int64_t *seg_first, const int32_t *seg_ns,
                             const int32_t *seg_len, int64_t n_ns, const uint8_t *ns_bytes,
                             const int64_t *ns_off, const int32_t *ns_len, const int32_t *clients,
                             const int64_t *labels, int32_t *out_ids);
/* Relabel requests (the order-maintenance labels ran out of gaps). */
int fs_requests_set_labels(fs_ctx *ctx, int64_t n, const int32_t *ids, const int64_t *labels);
/* Set the client of requests first uploaded without one (a token sequence the
 * routing index saw before the worker enqueued it). */
int fs_requests_set_clients(fs_ctx *ctx, int64_t n, const int32_t *ids, const int32_t *clients);
int fs_requests_count(fs_ctx *ctx, int64_t *n);
int fs_request_info(fs_ctx *ctx, int32_t id, int64_t *arena_off, int32_t *len);
/* Read n arena tokens starting at arena offset off (paths of eviction records). */
int fs_arena_read(fs_ctx *ctx, int64_t off, int64_t n, int32_t *out);

/* ---- RadixTree  (radix.py:48-340) ------------------------------------------
 * capacity < 0 means None (global routing index).  n_workers bounds worker
 * tags when track_workers != 0 (<= 64).                                      */
int fs_trie_create(fs_ctx *ctx, int64_t capacity, int track_workers, int n_workers, fs_trie **out);
int fs_trie_destroy(fs_trie *t);
/* used_tokens, pinned_tokens (radix.py:53-54), next seq (radix.py:55), live nodes */
int fs_trie_stats(fs_trie *t, int64_t *used, int64_t *pinned, int64_t *next_seq, int64_t *nodes);

/* Batched longest-prefix match (K1).  stamp != 0: match_prefix semantics with
 * last_access = now on every matched node (radix.py:83-91); stamp == 0: probe
 * (radix.py:93-99).  out_cov[i] = matched tokens lying in pinned nodes, so
 * probe's unpinned count = out_mlen[i] - out_cov[i].  Either output may be NULL. */
int fs_trie_match(fs_trie *t, int64_t n, const int32_t *req_ids, int64_t now, int stamp,
                  int32_t *out_mlen, int32_t *out_cov);

/* Eviction records (radix.py:217-249): (arena offset of the full path, full
 * path length, keep_len).  Buffers may be NULL when rec_cap == 0; *n_rec
 * always receives the record count (records beyond rec_cap are dropped). */
typedef struct {
    int64_t rec_cap;
    int64_t *rec_src;
    int32_t *rec_len;
    int32_t *rec_keep;
    int64_t n_rec;
} fs_records;

/* Re-read records [first, first+n) of the trie's last operation (the device
 * sink keeps them until the next operation on this trie). */
int fs_trie_read_records(fs_trie *t, int64_t first, int64_t n, int64_t *src, int32_t *len, int32_t *keep);

/* RadixTree.insert (radix.py:128-162); worker < 0 means None.  *path_node is
 * the deepest node of the returned path (the handle pin/unpin use, radix.py:164-172),
 * -1 for an empty path.  Returns FS_ERR_CACHE_FULL after performing the evictions
 * exactly like the reference (records are still reported). */
int fs_trie_insert(fs_trie *t, int32_t req, int64_t now, int32_t worker, int32_t *new_len,
                   int32_t *path_node, fs_records *recs);
/* RadixTree.admit (radix.py:187-192): probe, insert, pin. */
int fs_trie_admit(fs_trie *t, int32_t req, int64_t now, int32_t *mlen, int32_t *path_node,
                  fs_records *recs);
int fs_trie_pin(fs_trie *t, int32_t path_node);   /* radix.py:174-178 */
int fs_trie_unpin(fs_trie *t, int32_t path_node); /* radix.py:180-185 */
/* unpin of a whole finishing batch in one launch (worker.py:209-213), in order */
int fs_trie_unpin_many(fs_trie *t, int64_t n, const int32_t *path_nodes);
/* fs_trie_unpin_many without waiting: the unpins are stream-ordered before the
 * next fill of this tree; their status (FS_ERR_UNDERFLOW) and device time are
 * reported by the next fs_worker_fill_end / fs_trie_last_ms / fs_trie_unpin_many. */
int fs_trie_unpin_many_async(fs_trie *t, int64_t n, const int32_t *nodes);
/* device time (CUDA events) of the last fs_trie_unpin_many */
int fs_trie_last_ms(fs_trie *t, float *ms);
/* RadixTree.evict_lru without a protect set (radix.py:210-250) */
int fs_trie_evict_lru(fs_trie *t, int64_t needed, fs_records *recs);
/* RadixTree.longest_match_workers (radix.py:101-110): mask bit w = worker w tagged */
int fs_trie_longest_match_workers(fs_trie *t, int32_t req, int64_t now, int32_t *mlen, uint64_t *mask);
/* RadixTree.evict_notify (radix.py:254-302); the path is arena[path_src : path_src+path_len] */
int fs_trie_evict_notify(fs_trie *t, int64_t path_src, int32_t path_len, int32_t worker,
                         int32_t keep_len, int64_t notice_time);
/* n notices applied in order in one launch (the all-gathered eviction notices of
 * a D2lpm round, global_policies.py:130-132 -> radix.py:254-302). */
int fs_trie_evict_notify_many(fs_trie *t, int64_t n, const int64_t *path_src, const int32_t *path_len,
                              const int32_t *worker, const int32_t *keep_len, const int64_t *notice_time);
/* SM cycles of the last fs_trie_evict_notify_many: walk, collect, edit, repoint */
int fs_trie_last_notify_profile(fs_trie *t, int64_t *prof4);
/* Node table export for RadixTree.dump / check (radix.py:306-340).  Writes up to
 * cap nodes (index 0 = root) and sets *n to the node-table size; dead slots have
 * parent == -2. wmask may be NULL. */
int fs_trie_export(fs_trie *t, int64_t cap, int64_t *n, int64_t *src, int32_t *start,
                   int32_t *end, int32_t *parent, int32_t *ref, int64_t *last_access,
                   uint64_t *wmask);

/* ---- DLPM / LPM / VTC worker  (local_policies.py:42-195 + worker.py:87-135) -
 * policy 0 = Dlpm (deficit gate, quantum refill), 1 = Lpm (gate always true),
 * 2 = Vtc (least-served client's earliest request first; counters charged the
 * full input, fs_worker_outputs adds w_q per output token; no match_prefix).
 * The worker owns the queue mirror (request ids), the per-client deficit
 * counters q, refill counts and client_list membership.                     */
int fs_worker_create(fs_ctx *ctx, fs_trie *tree, int policy, int64_t quantum, int64_t M,
                     int64_t output_reserve, int64_t w_e, int64_t w_q, int32_t max_clients,
                     fs_worker **out);
int fs_worker_destroy(fs_worker *w);
/* Worker.enqueue -> on_request_enqueued (worker.py:142-148, local_policies.py:88-92) */
int fs_worker_enqueue(fs_worker *w, int64_t n, const int32_t *req_ids);
/* Dlpm.on_outputs (local_policies.py:130-133): q[c] -= w_q * counts[i] */
int fs_worker_outputs(fs_worker *w, int64_t n, const int32_t *clients, const int64_t *counts);
/* Dlpm.check_refill (local_policies.py:94-106) for an explicit queued-client set */
int fs_worker_check_refill(fs_worker *w, int64_t n, const int32_t *queued_clients, int *refilled);
/* Host mirror of q / refill_counts / client_list membership (Dlpm.counters(),
 * local_policies.py:135-136).  Any pointer may be NULL. */
int fs_worker_counters(fs_worker *w, int32_t n, int64_t *q, int64_t *refills, uint8_t *known);
/* Vtc tie-break (local_policies.py:176: clients sorted by (counter, name)):
 * rank of each dense client id's name; by default the id order. */
int fs_worker_set_client_ranks(fs_worker *w, int32_t n, const int32_t *ranks);
int fs_worker_set_counter(fs_worker *w, int32_t client, int64_t q);
/* Grow the client tables (clients are dense ids assigned by the caller). */
int fs_worker_reserve_clients(fs_worker *w, int32_t max_clients);
/* Mark clients as members of Dlpm.client_list without enqueueing a request. */
int fs_worker_mark_known(fs_worker *w, int64_t n, const int32_t *clients);

/* One schedule step: Dlpm.fill / Lpm.fill (local_policies.py:108-128, 66-71).
 * Matches every queued request (K1, stamping last_access = now), sorts by
 * (-mlen, label) (K2), then runs the deficit-gated admission passes with the
 * closed-form refill and budget test and performs each admission's radix
 * insert / split / LRU evict / pin on device (K3+K4).
 * generated_total and headroom are Worker.generated_total and
 * Worker._reserved_headroom() at the call (worker.py:95-99). */
typedef struct {
    int64_t cap_adm;
    int32_t *adm_req;           /* admitted request ids, in admission order        */
    int32_t *adm_mlen;          /* match length at admission (probe, radix.py:189) */
    int64_t *adm_unpinned;      /* probe's matched-unpinned tokens (worker.py:102) */
    int64_t *adm_pinned_before; /* tree.pinned_tokens seen by can_add              */
    int32_t *adm_path_node;     /* pin handle                                      */
    int64_t *adm_rec_end;       /* records emitted up to and including this admission */
    fs_records recs;
    int64_t n_adm;              /* out */
    int64_t n_queued;           /* out: requests evaluated (scheduling decisions) */
    int64_t used, pinned;       /* out: tree stats after the fill */
    float device_ms;            /* out: device time of the fill (CUDA events)    */
} fs_fill_result;
int fs_worker_fill(fs_worker *w, int64_t now, int64_t generated_total, int64_t headroom,
                   fs_fill_result *res);
/* fs_worker_fill in two halves: _begin launches the fill and returns at once,
 * _end waits and fills res.  In between, context uploads (fs_requests_add*,
 * on their own stream) may run concurrently with the fill -- a serving loop
 * uploads the next arrivals while the scheduler decides; every other call on
 * this worker or its tree fails with FS_ERR_INVALID until _end. */
int fs_worker_fill_begin(fs_worker *w, int64_t now, int64_t generated_total, int64_t headroom);
int fs_worker_fill_end(fs_worker *w, fs_fill_result *res);
/* Timing breakdown of the last fill: [merge, match K1, sort K2, schedule K3/K4] ms */
int fs_worker_last_phases(fs_worker *w, float *ms4);
/* Device time around the last fill (serving-loop diagnostics, not a reference
 * interface): [0] ms from the fill's end to its results being staged in host
 * memory, [1] ms the GPU spent between the previous fill's staged results and
 * this fill's start (host work of the serving loop; -1 for a first fill). */
int fs_worker_last_gaps(fs_worker *w, float *ms2);
/* Counters of the last fill: [0] sum over queued j of min(mlen_j+1, len_j)
 * (request tokens K1 must read: the algorithmic bytes / 4), [1] requests
 * matched, [2] admission events, [3] refill events, [4] frontier resumes,
 * [5] kernel launches issued by the fill, [6] trie hops in K1, [8..15] scheduler-kernel SM cycles:
 * [8] candidate search, [9] admission walks, [10] LRU eviction, [11] admission
 * tail (pin, counters, records), [12] search chunks, [13] eviction pops,
 * [14] source chains in admission walks, [15] total, [16..18] eviction-pop
 * argmin / edit / index-update cycles.  Writes 24 entries. */
int fs_worker_last_stats(fs_worker *w, int64_t *stats24);
/* Scheduler cycle counters of the last fill (diagnostic): [0] path pin,
 * [1] post-walk scheduler bookkeeping, [2] waits for the asynchronous
 * evictor's setup, [3..7] reserved. */
int fs_worker_last_stats_ext(fs_worker *w, int64_t *ext8);
/* Worker options.  FS_OPT_K1_FULL (1): value != 0 makes every fill re-match
 * every queued request from the root instead of resuming from its previous
 * match (same decisions; the incremental match is the default). */
#define FS_OPT_K1_FULL 1
int fs_worker_set_option(fs_worker *w, int option, int64_t value);
/* Kernel launches issued by this library since load (all handles). */
int64_t fs_launch_count(void);
/* Queue length currently mirrored on device (worker.queue, worker.py:73) */
int fs_worker_queue_len(fs_worker *w, int64_t *n);

/* ---- D2LPM dispatcher  (global_policies.py:88-132) --------------------------
 * Owns the global routing index (a track_workers RadixTree), the per
 * (client, worker) counters q_{i,w} and queue sizes.  Workers are 0..D-1.   */
int fs_dispatcher_create(fs_ctx *ctx, int D, int64_t quantum, int64_t w_e, int64_t w_q,
                         int32_t max_clients, fs_dispatcher **out);
int fs_dispatcher_destroy(fs_dispatcher *d);
/* Routing policy of a dispatcher (default FS_DISPATCH_D2LPM).
 * FS_DISPATCH_THRESHOLD: ThresholdRouter (global_policies.py:135-161) on the
 * same tagged index -- locality when match_len / input_len >= theta (IEEE
 * double, like Python), else the least-loaded worker; no deficit counters
 * (fs_dispatch leaves q untouched, fs_dispatch_finish only decrements the
 * worker's queue size).  Errors: FS_ERR_INVALID for an unknown policy or
 * theta outside [0, 1] (global_policies.py:145-146). */
#define FS_DISPATCH_D2LPM 0
#define FS_DISPATCH_THRESHOLD 1
int fs_dispatcher_set_policy(fs_dispatcher *d, int32_t policy, double theta);
fs_trie *fs_dispatcher_tree(fs_dispatcher *d);
/* Dispatcher.dispatch for n arrivals in order (global_policies.py:40-46,
 * 107-124): longest_match_workers, SelectWorker with closed-form refill,
 * queue_size += 1, q -= w_e*input_len, global insert with worker tag.
 * Outputs per arrival: worker, match length, matched-worker mask, refill rounds. */
int fs_dispatch(fs_dispatcher *d, int64_t n, const int32_t *req_ids, const int32_t *clients,
                const int64_t *now, int32_t *out_worker, int32_t *out_mlen, uint64_t *out_mask,
                int64_t *out_rounds);
/* Multi-GPU dispatch: the batch-start matches of an arrival batch
 * against the routing index, split across ranks.  fs_dispatch_prematch writes
 * the records of n arrivals (one rank's slice) to device memory dev_out on the
 * dispatcher's device -- fs_prematch_record_bytes() bytes each -- and returns
 * when they are written; the ranks all-gather the slices (NCCL) and each
 * replica runs fs_dispatch_prematched with the records of the whole batch in
 * arrival order (dev_pre, device memory).  Same decisions as fs_dispatch,
 * which computes the records itself. */
int fs_prematch_record_bytes(void);
int fs_dispatch_prematch(fs_dispatcher *d, int64_t n, const int32_t *req_ids, void *dev_out);
int fs_dispatch_prematched(fs_dispatcher *d, int64_t n, const int32_t *req_ids, const int32_t *clients,
                           const int64_t *now, const void *dev_pre, int32_t *out_worker, int32_t *out_mlen,
                           uint64_t *out_mask, int64_t *out_rounds);
/* D2lpm.on_finish (global_policies.py:126-129) */
int fs_dispatch_finish(fs_dispatcher *d, int32_t client, int32_t worker, int64_t output_tokens);
/* n finish records in order (the all-gathered finishes of a round) */
int fs_dispatch_finish_many(fs_dispatcher *d, int64_t n, const int32_t *clients, const int32_t *workers,
                            const int64_t *output_tokens);
/* q_{i,w} row of one client (D values) and dict-key presence flags */
int fs_dispatch_counters(fs_dispatcher *d, int32_t client, int64_t *q_row, uint8_t *present);
int fs_dispatch_queue_sizes(fs_dispatcher *d, int64_t *sizes);
/* D2lpm.select_worker alone (global_policies.py:107-114): refill rounds and the
 * locality-first / min-queue choice for a given matched mask; no queue_size or
 * counter charge, no index update. */
int fs_dispatch_select(fs_dispatcher *d, int32_t client, uint64_t matched_mask, int32_t *worker,
                       int64_t *rounds);
/* Overwrite q_{i,w} / queue_size[w] (the Python dicts are mutable by callers). */
int fs_dispatch_set_counter(fs_dispatcher *d, int32_t client, int32_t worker, int64_t q);
int fs_dispatch_set_queue_size(fs_dispatcher *d, int32_t worker, int64_t size);
int fs_dispatcher_reserve_clients(fs_dispatcher *d, int32_t max_clients);
/* Device-side copy of the counters (tests compare it with the host mirror). */
/* SM-cycle profile of the last fs_dispatch chain: [0] match + select, [1] insert
 * walk, [2] evict, [12] leaf + stamp, [13] position repoint, [14] worker tags,
 * [15] total.  Writes 16 entries. */
int fs_dispatch_last_profile(fs_dispatcher *d, int64_t *prof16);
int fs_dispatch_device_counters(fs_dispatcher *d, int64_t n, int64_t *q, uint8_t *present, int64_t *qsize);
int fs_worker_device_counters(fs_worker *w, int32_t n, int64_t *q, int64_t *refills);

/* ---- post-run service-gap verifiers  (metrics.py:148-237) ----
 * Clients are indexed in sorted-name order (metrics.py:144-145).  Client c's
 * service events are ev_time[ev_off[c] .. ev_off[c+1]) (time-ordered), their
 * prefix sums ev_cum[ev_off[c] + c .. ev_off[c+1] + c] (n_c + 1 values, first
 * 0); its backlogged intervals (metrics.py:103-115) iv_lo/iv_hi[iv_off[c] ..
 * iv_off[c+1]).  Host buffers; the call runs on `device` and returns when the
 * results are written.
 * fs_verify_pairs: one result per client pair (f < g) at index f*C + g over the
 * windows of intersect_intervals x window_grid; mode 0 = |W_f - W_g|
 * (verify_service_bound_pairwise), mode 1 = max - min over the clients
 * backlogged through the window (verify_global_max_min).  out_valid = 0: the
 * pair has no window.  The caller takes the first maximum in pair order. */
int fs_verify_pairs(int device, int32_t C, const int64_t *ev_off, const int64_t *ev_time, const int64_t *ev_cum,
                    const int64_t *iv_off, const int64_t *iv_lo, const int64_t *iv_hi, int mode,
                    int64_t *out_gap, int64_t *out_t1, int64_t *out_t2, int32_t *out_valid);
/* fs_verify_vs_any (verify_service_bound_vs_nonbacklogged, metrics.py:177-197):
 * for each of nwin windows (client f, [t1, t2)) in the reference's order, the
 * worst W_g - W_f over g != f and the first g attaining it (INT64_MIN / -1
 * when C == 1). */
int fs_verify_vs_any(int device, int32_t C, const int64_t *ev_off, const int64_t *ev_time, const int64_t *ev_cum,
                     const int64_t *iv_off, const int64_t *iv_lo, const int64_t *iv_hi, int64_t nwin,
                     const int32_t *win_f, const int64_t *win_t1, const int64_t *win_t2, int64_t *out_gap,
                     int32_t *out_g);

#ifdef __cplusplus
}
#endif
#endif /* FAIRSCHED_B200_H */
