// fs_lib.cu -- host side of the C ABI (include/fairsched_b200.h).
//
// Owns device memory, streams, the queue mirror and host shadows of the few
// scalars the reference's caller reads between schedule steps (counters,
// used/pinned tokens).  All decision work runs in the kernels of
// fs_kernels.cuh; nothing here computes a scheduling decision.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fairsched_b200.h"
#include "fs_kernels.cuh"
#include "fs_order.cuh"
#include "fs_verify.cuh"
#include "fs_materialize.cuh"

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) return fail(FS_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define TRY(x)                   \
    do {                         \
        int rc_ = (x);           \
        if (rc_ != FS_OK) return rc_; \
    } while (0)

// Kernel launches issued by this library (the bench reports it as gpu_launches).
// CUB device-wide calls launch several kernels; their counts were taken from
// the ncu launch list (profiles/) for the code paths used here.
static std::atomic<int64_t> g_launches{0};
static inline void counted(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
extern "C" int64_t fs_launch_count(void) { return g_launches.load(); }

extern "C" const char *fs_last_error(void) { return g_err.c_str(); }
extern "C" int fs_version(void) { return 1; }
extern "C" int fs_device_count(int *count) {
    CK(cudaGetDeviceCount(count));
    return FS_OK;
}

// ---------------------------------------------------------------- buffers
template <typename T>
struct DBuf {
    T *p = nullptr;
    int64_t cap = 0;
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

template <typename T>
static int dgrow(DBuf<T> &b, int64_t n, cudaStream_t s, bool keep = false, int64_t keep_n = 0) {
    if (n <= b.cap) return FS_OK;
    int64_t nc = std::max<int64_t>(n, b.cap + b.cap / 2);
    nc = std::max<int64_t>(nc, 64);
    T *np = nullptr;
    CK(cudaMalloc(&np, sizeof(T) * nc));
    // FS_POISON=1 (debug): fresh allocations hold a non-zero pattern, so a read
    // of never-written memory shows up deterministically instead of depending
    // on what an earlier allocation left behind
    static const bool poison = [] { const char *e = getenv("FS_POISON"); return e && atoi(e) != 0; }();
    if (poison) CK(cudaMemsetAsync(np, 0xA5, sizeof(T) * nc, s));
    if (keep && b.p && keep_n > 0) CK(cudaMemcpyAsync(np, b.p, sizeof(T) * keep_n, cudaMemcpyDeviceToDevice, s));
    if (b.p) { CK(cudaStreamSynchronize(s)); cudaFree(b.p); }
    b.p = np;
    b.cap = nc;
    return FS_OK;
}

template <typename T>
struct HBuf {  // pinned host staging
    T *p = nullptr;
    int64_t cap = 0;
    void release() { if (p) cudaFreeHost(p); p = nullptr; cap = 0; }
};

template <typename T>
static int hgrow(HBuf<T> &b, int64_t n) {
    if (n <= b.cap) return FS_OK;
    int64_t nc = std::max<int64_t>(std::max<int64_t>(n, b.cap * 2), 64);
    T *np = nullptr;
    // portable + mapped: a fill's result staging is written by a kernel
    // directly (k_stage_results), from whichever device context runs it
    CK(cudaHostAlloc((void **)&np, sizeof(T) * nc, cudaHostAllocPortable | cudaHostAllocMapped));
    if (b.p) cudaFreeHost(b.p);
    b.p = np;
    b.cap = nc;
    return FS_OK;
}

// ---------------------------------------------------------------- uploads
// Request i: src[soff[i] : soff[i]+len[i]) -> arena[dst[i] ...], zero-padded to
// a 16-B row; any id outside [0, 2^31) sets *bad.
__global__ void k_scatter_rows(const int32_t *__restrict__ src, const int64_t *__restrict__ soff,
                               const int64_t *__restrict__ dst, const int32_t *__restrict__ len,
                               int32_t *__restrict__ arena, int32_t *bad) {
    const int64_t i = blockIdx.x;
    const int32_t n = len[i];
    const int32_t padded = (n + 3) & ~3;
    const int32_t *s = src + soff[i];
    int32_t *d = arena + dst[i];
    bool neg = false;
    for (int32_t k = threadIdx.x; k < padded; k += blockDim.x) {
        const int32_t v = k < n ? s[k] : 0;
        neg |= v < 0;
        d[k] = v;
    }
    if (__syncthreads_or(neg) && threadIdx.x == 0) *bad = 1;
}

// ---------------------------------------------------------------- context
struct fs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;   // fills and tree operations
    cudaStream_t ustream = nullptr;  // uploads (fs_requests_add*)
    DBuf<int32_t> arena;
    int64_t arena_used = 0;
    DBuf<int64_t> roff;
    DBuf<int32_t> rlen, rclient;
    DBuf<int64_t> rlabel;
    DBuf<int8_t> rstate;  // 0 none, 1 queued, 2 admitted
    DBuf<int32_t> rhint;  // last K1 match length per request (L2 prefetch extent, match hint)
    DBuf<int32_t> h_owner, h_tok0;  // match hints (K1Hints): owning worker, token at the match
    DBuf<int64_t> h_S0;             //   and the chain of its deepest node
    std::vector<int64_t> h_roff, h_rlabel;
    std::vector<int32_t> h_rlen, h_rclient;
    int32_t max_len = 1;
    HBuf<int32_t> stage_tok;
    HBuf<int64_t> stage64;
    HBuf<int32_t> stage32;
    // fs_requests_add_expanded scratch
    DBuf<int64_t> x_dst, x_nsoff;
    DBuf<int32_t> x_len, x_ns, x_nslen;
    DBuf<uint8_t> x_bytes;
    DBuf<int32_t> x_tok, x_flag;  // fs_requests_add contiguous fast path
};

static int ctx_use(fs_ctx *c) {
    CK(cudaSetDevice(c->device));
    return FS_OK;
}

extern "C" int fs_host_register(void *ptr, int64_t bytes) {
    if (!ptr || bytes <= 0) return fail(FS_ERR_INVALID, "bad host range");
    const cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) { cudaGetLastError(); return FS_OK; }  // idempotent
    CK(e);
    return FS_OK;
}

extern "C" int fs_host_unregister(void *ptr) {
    if (!ptr) return fail(FS_ERR_INVALID, "NULL");
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e == cudaErrorHostMemoryNotRegistered) { cudaGetLastError(); return FS_OK; }
    CK(e);
    return FS_OK;
}

extern "C" int fs_ctx_create(int device, int64_t arena_tokens, int64_t max_requests, fs_ctx **out) {
    if (!out) return fail(FS_ERR_INVALID, "out is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(FS_ERR_CUDA, "no CUDA device available (%s); the decision path has no CPU fallback",
                    e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
    if (device < 0 || device >= n) return fail(FS_ERR_INVALID, "device %d out of range [0,%d)", device, n);
    fs_ctx *c = new fs_ctx();
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    {
        // uploads have their own stream: they may run while a fill is in
        // flight (fs_worker_fill_begin), and at the highest priority so their
        // few blocks do not queue behind the fill's
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&c->ustream, cudaStreamNonBlocking, hi));
    }
    TRY(dgrow(c->arena, std::max<int64_t>(arena_tokens, 1024), c->stream));
    const int64_t mr = std::max<int64_t>(max_requests, 1024);
    TRY(dgrow(c->roff, mr, c->stream));
    TRY(dgrow(c->rlen, mr, c->stream));
    TRY(dgrow(c->rclient, mr, c->stream));
    TRY(dgrow(c->rlabel, mr, c->stream));
    TRY(dgrow(c->rstate, mr, c->stream));
    CK(cudaMemsetAsync(c->rstate.p, 0, mr, c->stream));
    *out = c;
    return FS_OK;
}

extern "C" int fs_ctx_destroy(fs_ctx *c) {
    if (!c) return FS_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    c->arena.release(); c->roff.release(); c->rlen.release(); c->rclient.release();
    c->rlabel.release(); c->rstate.release(); c->rhint.release();
    c->h_owner.release(); c->h_tok0.release(); c->h_S0.release();
    c->stage_tok.release(); c->stage64.release(); c->stage32.release();
    c->x_dst.release(); c->x_nsoff.release(); c->x_len.release(); c->x_ns.release(); c->x_nslen.release();
    c->x_bytes.release(); c->x_tok.release(); c->x_flag.release();
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->ustream);
    delete c;
    return FS_OK;
}

extern "C" int fs_ctx_sync(fs_ctx *c) {
    TRY(ctx_use(c));
    CK(cudaStreamSynchronize(c->ustream));
    CK(cudaStreamSynchronize(c->stream));
    return FS_OK;
}

// Uploads may overlap an in-flight fill that reads (and, for the match hints,
// writes) the per-request arrays and the arena: reallocating any of them
// waits for the whole device first.
static int quiesce_for_growth(fs_ctx *c, int64_t nr, int64_t arena_need) {
    const bool g = arena_need > c->arena.cap || nr > c->roff.cap || nr > c->rlen.cap || nr > c->rclient.cap ||
                   nr > c->rlabel.cap || nr > c->rstate.cap || nr > c->rhint.cap || nr > c->h_owner.cap;
    if (g) CK(cudaDeviceSynchronize());
    return FS_OK;
}

// Request-table rows for n requests already placed at place[i] in the arena.
static int append_request_meta(fs_ctx *c, int64_t n, const int64_t *place, const int32_t *lens,
                               const int32_t *clients, const int64_t *labels, int32_t *out_ids) {
    const int64_t base_id = (int64_t)c->h_roff.size();
    const int64_t nr = base_id + n;
    TRY(dgrow(c->roff, nr, c->ustream, true, base_id));
    TRY(dgrow(c->rlen, nr, c->ustream, true, base_id));
    TRY(dgrow(c->rclient, nr, c->ustream, true, base_id));
    TRY(dgrow(c->rlabel, nr, c->ustream, true, base_id));
    if (c->rstate.cap < nr) {
        const int64_t old = c->rstate.cap;
        TRY(dgrow(c->rstate, nr, c->ustream, true, base_id));
        CK(cudaMemsetAsync(c->rstate.p + old, 0, c->rstate.cap - old, c->ustream));
    }
    if (c->rhint.cap < nr) {
        const int64_t old = c->rhint.cap;
        TRY(dgrow(c->rhint, nr, c->ustream, true, old));
        CK(cudaMemsetAsync(c->rhint.p + old, 0, sizeof(int32_t) * (c->rhint.cap - old), c->ustream));
    }
    if (c->h_owner.cap < nr) {
        const int64_t old = c->h_owner.cap;
        TRY(dgrow(c->h_owner, nr, c->ustream, true, old));
        TRY(dgrow(c->h_tok0, c->h_owner.cap, c->ustream, true, old));
        TRY(dgrow(c->h_S0, c->h_owner.cap, c->ustream, true, old));
        CK(cudaMemsetAsync(c->h_owner.p + old, 0xff, sizeof(int32_t) * (c->h_owner.cap - old), c->ustream));
    }
    for (int64_t i = 0; i < n; i++) {
        c->h_roff.push_back(place[i]);
        c->h_rlen.push_back(lens[i]);
        c->h_rclient.push_back(clients ? clients[i] : 0);
        c->h_rlabel.push_back(labels ? labels[i] : base_id + i);
        c->max_len = std::max(c->max_len, lens[i]);
        if (out_ids) out_ids[i] = (int32_t)(base_id + i);
    }
    CK(cudaStreamSynchronize(c->ustream));  // staging buffer reuse
    CK(cudaMemcpyAsync(c->roff.p + base_id, c->h_roff.data() + base_id, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->ustream));
    CK(cudaMemcpyAsync(c->rlen.p + base_id, c->h_rlen.data() + base_id, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->ustream));
    CK(cudaMemcpyAsync(c->rclient.p + base_id, c->h_rclient.data() + base_id, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->ustream));
    CK(cudaMemcpyAsync(c->rlabel.p + base_id, c->h_rlabel.data() + base_id, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->ustream));
    CK(cudaStreamSynchronize(c->ustream));
    return FS_OK;
}

extern "C" int fs_requests_add(fs_ctx *c, int64_t n, const int32_t *tokens, const int64_t *offsets,
                               const int32_t *lens, const int32_t *clients, const int64_t *labels,
                               int32_t *out_ids) {
    if (!c || n < 0 || (n > 0 && (!tokens || !offsets || !lens))) return fail(FS_ERR_INVALID, "bad arguments");
    TRY(ctx_use(c));
    const int64_t base_id = (int64_t)c->h_roff.size();
    if (base_id + n > INT32_MAX) return fail(FS_ERR_NOMEM, "request id space exhausted");
    // 16-B aligned placement of every request in the arena
    int64_t total = 0;
    std::vector<int64_t> place(n);
    for (int64_t i = 0; i < n; i++) {
        if (lens[i] < 0) return fail(FS_ERR_INVALID, "negative length");
        place[i] = c->arena_used + total;
        total += (lens[i] + 3) & ~3LL;
    }
    TRY(quiesce_for_growth(c, base_id + n, c->arena_used + total + 4));
    bool contiguous = n > 0;
    for (int64_t i = 0; i + 1 < n && contiguous; i++) contiguous = offsets[i + 1] == offsets[i] + lens[i];
    static const bool hprof = getenv("FS_HOST_PROFILE") != nullptr;
    const auto a0 = std::chrono::steady_clock::now();
    if (contiguous) {
        // one H2D of the caller's token block (a DMA when the caller registered it,
        // fs_host_register), then a scatter kernel into the 16-B aligned arena
        // rows that also checks the id range -- no host pass over the tokens
        const int64_t src_total = offsets[n - 1] + lens[n - 1] - offsets[0];
        TRY(dgrow(c->arena, c->arena_used + total + 4, c->ustream, true, c->arena_used));
        // staging for the caller's block: reserved in 16 MB steps so a stream of
        // growing arrival batches does not reallocate (and synchronize) per call
        TRY(dgrow(c->x_tok, std::max<int64_t>(src_total + 4, std::min<int64_t>(c->arena.cap, 1 << 22)), c->ustream));
        TRY(dgrow(c->x_dst, n + 1, c->ustream)); TRY(dgrow(c->x_nsoff, n + 1, c->ustream));
        TRY(dgrow(c->x_len, n + 1, c->ustream)); TRY(dgrow(c->x_flag, 1, c->ustream));
        TRY(hgrow(c->stage64, 2 * n + 2)); TRY(hgrow(c->stage32, n + 2));
        for (int64_t i = 0; i < n; i++) {
            c->stage64.p[i] = place[i];
            c->stage64.p[n + i] = offsets[i] - offsets[0];
            c->stage32.p[i] = lens[i];
        }
        const auto ag = std::chrono::steady_clock::now();
        if (src_total) CK(cudaMemcpyAsync(c->x_tok.p, tokens + offsets[0], sizeof(int32_t) * src_total,
                                          cudaMemcpyHostToDevice, c->ustream));
        const auto ah = std::chrono::steady_clock::now();
        CK(cudaMemcpyAsync(c->x_dst.p, c->stage64.p, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->ustream));
        CK(cudaMemcpyAsync(c->x_nsoff.p, c->stage64.p + n, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->ustream));
        CK(cudaMemcpyAsync(c->x_len.p, c->stage32.p, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->ustream));
        CK(cudaMemsetAsync(c->x_flag.p, 0, sizeof(int32_t), c->ustream));
        const auto ac = std::chrono::steady_clock::now();
        if (hprof) CK(cudaStreamSynchronize(c->ustream));
        const auto ad = std::chrono::steady_clock::now();
        k_scatter_rows<<<(unsigned)n, 256, 0, c->ustream>>>(c->x_tok.p, c->x_nsoff.p, c->x_dst.p, c->x_len.p,
                                                           c->arena.p, c->x_flag.p);
        counted();
        CK(cudaGetLastError());
        int32_t bad = 0;
        CK(cudaMemcpyAsync(&bad, c->x_flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c->ustream));
        const auto aq = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(c->ustream));
        if (bad) return fail(FS_ERR_TOKEN_RANGE, "a token id is outside [0, 2^31)");  // nothing committed
        const auto a1 = std::chrono::steady_clock::now();
        TRY(append_request_meta(c, n, place.data(), lens, clients, labels, out_ids));
        c->arena_used += total;
        if (hprof) {
            const auto a2 = std::chrono::steady_clock::now();
            auto us = [](auto x, auto y) { return std::chrono::duration<double, std::micro>(y - x).count(); };
            fprintf(stderr, "requests_add: %lld rows, %lld tokens: copy+scatter %.0f us (grow %.0f, tok copy %.0f, rest %.0f, copy wait %.0f, kernel %.0f), meta %.0f us\n",
                    (long long)n, (long long)src_total, us(a0, a1), us(a0, ag), us(ag, ah), us(ah, ac), us(ac, ad), us(ad, a1), us(a1, a2));
        }
        return FS_OK;
    }
    for (int64_t i = 0; i < n; i++) {
        const int32_t *tk = tokens + offsets[i];
        for (int32_t k = 0; k < lens[i]; k++)
            if (tk[k] < 0) return fail(FS_ERR_TOKEN_RANGE, "token %d of request %lld is outside [0, 2^31)", tk[k], (long long)i);
    }
    TRY(dgrow(c->arena, c->arena_used + total + 4, c->ustream, true, c->arena_used));
    TRY(hgrow(c->stage_tok, total + 4));
    for (int64_t i = 0; i < n; i++) {
        int32_t *dst = c->stage_tok.p + (place[i] - c->arena_used);
        std::memcpy(dst, tokens + offsets[i], sizeof(int32_t) * lens[i]);
        for (int32_t k = lens[i]; k < ((lens[i] + 3) & ~3); k++) dst[k] = 0;
    }
    if (total) CK(cudaMemcpyAsync(c->arena.p + c->arena_used, c->stage_tok.p, sizeof(int32_t) * total,
                                  cudaMemcpyHostToDevice, c->ustream));
    TRY(append_request_meta(c, n, place.data(), lens, clients, labels, out_ids));
    c->arena_used += total;
    return FS_OK;
}

extern "C" int fs_requests_add_expanded(fs_ctx *c, int64_t n, const int64_t *seg_first, const int32_t *seg_ns,
                                        const int32_t *seg_len, int64_t n_ns, const uint8_t *ns_bytes,
                                        const int64_t *ns_off, const int32_t *ns_len, const int32_t *clients,
                                        const int64_t *labels, int32_t *out_ids) {
    if (!c || n < 0 || n_ns < 0 || (n > 0 && (!seg_first || !clients)) || (n_ns > 0 && (!ns_off || !ns_len)))
        return fail(FS_ERR_INVALID, "bad arguments");
    TRY(ctx_use(c));
    const int64_t base_id = (int64_t)c->h_roff.size();
    if (base_id + n > INT32_MAX) return fail(FS_ERR_NOMEM, "request id space exhausted");
    if (n == 0) return FS_OK;
    if (seg_first[0] != 0) return fail(FS_ERR_INVALID, "seg_first[0] must be 0");
    const int64_t nseg = seg_first[n];
    int64_t nbytes = 0;
    for (int64_t k = 0; k < n_ns; k++) {
        if (ns_len[k] < 0 || ns_off[k] < 0) return fail(FS_ERR_INVALID, "bad namespace %lld", (long long)k);
        nbytes = std::max<int64_t>(nbytes, ns_off[k] + ns_len[k]);
    }
    std::vector<int64_t> place(n), dst(std::max<int64_t>(nseg, 1));
    std::vector<int32_t> lens(n);
    int64_t total = 0;
    for (int64_t i = 0; i < n; i++) {
        if (seg_first[i + 1] < seg_first[i]) return fail(FS_ERR_INVALID, "seg_first not monotone");
        place[i] = c->arena_used + total;
        int64_t L = 0;
        for (int64_t s = seg_first[i]; s < seg_first[i + 1]; s++) {
            if (seg_len[s] < 0 || seg_ns[s] < 0 || seg_ns[s] >= n_ns)
                return fail(FS_ERR_INVALID, "bad segment %lld", (long long)s);
            dst[s] = place[i] + L;
            L += seg_len[s];
        }
        if (L > INT32_MAX) return fail(FS_ERR_INVALID, "request %lld longer than 2^31 tokens", (long long)i);
        lens[i] = (int32_t)L;
        total += (L + 3) & ~3LL;
    }
    TRY(quiesce_for_growth(c, (int64_t)c->h_roff.size() + n, c->arena_used + total + 4));
    TRY(dgrow(c->arena, c->arena_used + total + 4, c->ustream, true, c->arena_used));
    TRY(dgrow(c->x_dst, nseg + 1, c->ustream)); TRY(dgrow(c->x_len, nseg + 1, c->ustream));
    TRY(dgrow(c->x_ns, nseg + 1, c->ustream));
    TRY(dgrow(c->x_nsoff, n_ns + 1, c->ustream)); TRY(dgrow(c->x_nslen, n_ns + 1, c->ustream));
    TRY(dgrow(c->x_bytes, nbytes + 16, c->ustream));
    // pad tails of 16-B slots stay zero, like fs_requests_add
    CK(cudaMemsetAsync(c->arena.p + c->arena_used, 0, sizeof(int32_t) * total, c->ustream));
    if (nseg) {
        CK(cudaMemcpyAsync(c->x_dst.p, dst.data(), sizeof(int64_t) * nseg, cudaMemcpyHostToDevice, c->ustream));
        CK(cudaMemcpyAsync(c->x_len.p, seg_len, sizeof(int32_t) * nseg, cudaMemcpyHostToDevice, c->ustream));
        CK(cudaMemcpyAsync(c->x_ns.p, seg_ns, sizeof(int32_t) * nseg, cudaMemcpyHostToDevice, c->ustream));
    }
    if (n_ns) {
        CK(cudaMemcpyAsync(c->x_nsoff.p, ns_off, sizeof(int64_t) * n_ns, cudaMemcpyHostToDevice, c->ustream));
        CK(cudaMemcpyAsync(c->x_nslen.p, ns_len, sizeof(int32_t) * n_ns, cudaMemcpyHostToDevice, c->ustream));
    }
    if (nbytes) CK(cudaMemcpyAsync(c->x_bytes.p, ns_bytes, nbytes, cudaMemcpyHostToDevice, c->ustream));
    if (nseg) {
        ExpandArgs a;
        a.arena = c->arena.p; a.seg_dst = c->x_dst.p; a.seg_len = c->x_len.p; a.seg_ns = c->x_ns.p;
        a.ns_bytes = c->x_bytes.p; a.ns_off = c->x_nsoff.p; a.ns_len = c->x_nslen.p; a.nseg = nseg;
        const int64_t blocks = std::min<int64_t>((nseg + 7) / 8, 148LL * 16);
        k_expand<<<(int)std::max<int64_t>(blocks, 1), 256, 0, c->ustream>>>(a);
        counted();
        CK(cudaGetLastError());
    }
    TRY(append_request_meta(c, n, place.data(), lens.data(), clients, labels, out_ids));
    c->arena_used += total;
    return FS_OK;
}

extern "C" int fs_requests_set_labels(fs_ctx *c, int64_t n, const int32_t *ids, const int64_t *labels) {
    if (!c) return fail(FS_ERR_INVALID, "ctx is NULL");
    TRY(ctx_use(c));
    for (int64_t i = 0; i < n; i++) {
        if (ids[i] < 0 || ids[i] >= (int64_t)c->h_rlabel.size()) return fail(FS_ERR_INVALID, "bad request id");
        c->h_rlabel[ids[i]] = labels[i];
    }
    if (n <= 64) {
        for (int64_t i = 0; i < n; i++)
            CK(cudaMemcpyAsync(c->rlabel.p + ids[i], c->h_rlabel.data() + ids[i], sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    } else {
        CK(cudaMemcpyAsync(c->rlabel.p, c->h_rlabel.data(), sizeof(int64_t) * c->h_rlabel.size(), cudaMemcpyHostToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return FS_OK;
}

extern "C" int fs_requests_set_clients(fs_ctx *c, int64_t n, const int32_t *ids, const int32_t *clients) {
    if (!c || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    TRY(ctx_use(c));
    for (int64_t i = 0; i < n; i++) {
        if (ids[i] < 0 || ids[i] >= (int64_t)c->h_rclient.size()) return fail(FS_ERR_INVALID, "bad request id");
        if (clients[i] < 0) return fail(FS_ERR_INVALID, "bad client id");
        c->h_rclient[ids[i]] = clients[i];
        CK(cudaMemcpyAsync(c->rclient.p + ids[i], c->h_rclient.data() + ids[i], sizeof(int32_t),
                           cudaMemcpyHostToDevice, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    return FS_OK;
}

extern "C" int fs_requests_count(fs_ctx *c, int64_t *n) {
    if (!c || !n) return fail(FS_ERR_INVALID, "NULL");
    *n = (int64_t)c->h_roff.size();
    return FS_OK;
}

extern "C" int fs_request_info(fs_ctx *c, int32_t id, int64_t *off, int32_t *len) {
    if (!c || id < 0 || id >= (int64_t)c->h_roff.size()) return fail(FS_ERR_INVALID, "bad request id");
    if (off) *off = c->h_roff[id];
    if (len) *len = c->h_rlen[id];
    return FS_OK;
}

extern "C" int fs_arena_read(fs_ctx *c, int64_t off, int64_t n, int32_t *out) {
    if (!c || off < 0 || n < 0 || off + n > c->arena_used) return fail(FS_ERR_INVALID, "arena range");
    TRY(ctx_use(c));
    if (n) CK(cudaMemcpyAsync(out, c->arena.p + off, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FS_OK;
}

// ---------------------------------------------------------------- trie
struct fs_trie {
    fs_ctx *ctx = nullptr;
    DBuf<int64_t> chk;    // FS_FILL_CHECK outside fills (tree_check)
    HBuf<int64_t> h_chk;
    bool busy = false;  // a worker fill on this tree is in flight (fs_worker_fill_begin)
    cudaStream_t stream = nullptr;  // own stream (dispatcher index) or null = the context's
    int64_t capacity = -1;
    int track = 0, nw = 0;
    int32_t ncap = 0;
    uint32_t hsize = 0;
    DBuf<int64_t> src, la, seq, lseq;
    DBuf<int32_t> start, end, slen, parent, nchild, ref, first, freest, ctop, cpar;
    int64_t opseq = 0;   // sequence number of the last stamping operation
    int64_t version = 0; // bumped by every structural edit outside a worker fill (K1 hints)
    DBuf<uint8_t> flags;
    DBuf<uint64_t> wmask;
    DBuf<int64_t> wtime;
    DBuf<ulonglong2> hslot;
    DBuf<TrieScalars> sc;
    DBuf<int32_t> pos;   // position shadow over the context arena
    DBuf<Seg> segs;      // walk scratch: path segments
    DBuf<int32_t> found; // evict_notify scratch
    DBuf<int64_t> rsrc;
    DBuf<int32_t> rlen, rkeep;
    DBuf<int64_t> opout;
    DBuf<int64_t> nt_src, nt_when, nt_s0;  // fs_trie_evict_notify_many staging
    DBuf<int32_t> nt_len, nt_worker, nt_keep, nt_m0;
    TrieScalars h_sc{};
    int nworkers = 0;  // DLPM/LPM workers scheduling on this tree (at most one)
    HBuf<int64_t> h_out;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    float last_ms = 0.f;  // device time of the last unpin_many
    // fs_trie_unpin_many_async: status and timing read at the next fill_end /
    // last_ms / unpin_many; the node list is staged in page-locked memory
    bool unpin_pending = false;
    HBuf<int32_t> h_unpin;
    HBuf<int64_t> h_ustat;
    DBuf<int64_t> ustat;
    DBuf<int32_t> dunpin;
    cudaEvent_t ev_staged = nullptr;
};

// Every entry point synchronizes its stream before returning, so calls made
// one after another are ordered whatever stream they use; a dispatcher's index
// has its own stream so its chain can run while a worker fills (other thread).
static cudaStream_t tstream(fs_trie *t) { return t->stream ? t->stream : t->ctx->stream; }

static TrieView view(fs_trie *t) {
    TrieView v;
    v.arena = t->ctx->arena.p;
    v.pos = t->pos.p;
    v.src = t->src.p; v.start = t->start.p; v.end = t->end.p; v.slen = t->slen.p; v.parent = t->parent.p;
    v.nchild = t->nchild.p; v.ref = t->ref.p; v.first = t->first.p;
    v.ctop = t->ctop.p; v.cpar = t->cpar.p;
    v.la = t->la.p; v.seq = t->seq.p; v.lseq = t->lseq.p; v.flags = t->flags.p;
    v.wmask = t->track ? t->wmask.p : nullptr;
    v.wtime = t->track ? t->wtime.p : nullptr;
    v.nw = t->nw;
    v.hslot = t->hslot.p; v.hmask = t->hsize - 1;
    v.freest = t->freest.p; v.ncap = t->ncap;
    v.sc = t->sc.p;
    v.rsrc = t->rsrc.p; v.rlen = t->rlen.p; v.rkeep = t->rkeep.p; v.rcap = t->rsrc.cap;
    return v;
}

__global__ void k_trie_init(TrieView t, int64_t capacity) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        TrieScalars &s = *t.sc;
        s.used = 0; s.pinned = 0; s.next_seq = 1; s.capacity = capacity; s.nrec = 0;
        s.hw = 1; s.nfree = 0; s.status = 0; s.live = 1; s.tombs = 0; s.pad_ = 0;
        t.src[0] = 0; t.start[0] = 0; t.end[0] = 0; t.slen[0] = 0; t.parent[0] = -1; t.nchild[0] = 0; t.ref[0] = 0;
        t.ctop[0] = 0; t.cpar[0] = -1;
        t.la[0] = 0; t.seq[0] = 0; t.lseq[0] = 0; t.first[0] = -1; t.flags[0] = FS_ALIVE;
        if (t.wmask) t.wmask[0] = 0;
    }
}

__global__ void k_rehash(TrieView t) {
    // rebuild the child hash from the node table (after a resize, or to drop
    // tombstones); the table was reset to empty by the host
    const int32_t hw = t.sc->hw;
    if (blockIdx.x == 0 && threadIdx.x == 0) t.sc->tombs = 0;
    for (int32_t n = 1 + blockIdx.x * blockDim.x + threadIdx.x; n < hw; n += gridDim.x * blockDim.x) {
        if (!(t.flags[n] & FS_ALIVE)) continue;
        const uint64_t key = fs_hkey(t.parent[n], t.first[n]);
        uint32_t i = fs_hmix(key) & t.hmask;
        while (true) {
            const unsigned long long prev = atomicCAS(&t.hslot[i].x, FS_HEMPTY, key);
            if (prev == FS_HEMPTY) { t.hslot[i].y = (unsigned long long)(uint32_t)n; break; }
            i = (i + 1) & t.hmask;
        }
    }
}

static uint32_t pow2_at_least(int64_t x) {
    uint32_t p = 1024;
    while ((int64_t)p < x) p <<= 1;
    return p;
}

// Make room for `extra_nodes` more nodes and paths of length `max_len`.
static int trie_reserve(fs_trie *t, int64_t extra_nodes, int32_t max_len) {
    cudaStream_t s = tstream(t);
    TRY(dgrow(t->segs, (int64_t)max_len + 16, s));
    TRY(dgrow(t->found, (int64_t)max_len + 16, s));
    // the position shadow covers the whole arena (grown with it; -1 = never written)
    if (t->pos.cap < t->ctx->arena.cap) {
        const int64_t old = t->pos.cap;
        TRY(dgrow(t->pos, t->ctx->arena.cap, s, true, old));
        CK(cudaMemsetAsync(t->pos.p + old, 0xff, sizeof(int32_t) * (t->pos.cap - old), s));
    }
    const int64_t need = (int64_t)t->h_sc.hw + extra_nodes + 4;
    if (t->hsize > 0 && (int64_t)t->h_sc.tombs * 4 > (int64_t)t->hsize) {
        // too many deleted slots lengthen probes: rebuild from the node table
        CK(cudaMemsetAsync(t->hslot.p, 0xff, sizeof(ulonglong2) * t->hsize, s));
        k_rehash<<<148, 256, 0, s>>>(view(t));
        counted();
        CK(cudaGetLastError());
        t->h_sc.tombs = 0;
    }
    if (need <= t->ncap) return FS_OK;
    const int64_t old = t->ncap;
    const int64_t nc = std::max<int64_t>(need, old * 2);
    const int64_t keep = old;
    TRY(dgrow(t->src, nc, s, true, keep)); TRY(dgrow(t->la, nc, s, true, keep)); TRY(dgrow(t->seq, nc, s, true, keep));
    TRY(dgrow(t->start, nc, s, true, keep)); TRY(dgrow(t->end, nc, s, true, keep)); TRY(dgrow(t->parent, nc, s, true, keep));
    TRY(dgrow(t->slen, nc, s, true, keep)); TRY(dgrow(t->lseq, nc, s, true, keep));
    TRY(dgrow(t->ctop, nc, s, true, keep)); TRY(dgrow(t->cpar, nc, s, true, keep));
    TRY(dgrow(t->nchild, nc, s, true, keep)); TRY(dgrow(t->ref, nc, s, true, keep)); TRY(dgrow(t->first, nc, s, true, keep));
    TRY(dgrow(t->freest, nc, s, true, keep)); TRY(dgrow(t->flags, nc, s, true, keep));
    if (t->track) { TRY(dgrow(t->wmask, nc, s, true, keep)); TRY(dgrow(t->wtime, nc * t->nw, s, true, keep * t->nw)); }
    t->ncap = (int32_t)std::min<int64_t>(nc, t->src.cap);
    const uint32_t hs = pow2_at_least(2 * (int64_t)t->ncap);
    if (hs != t->hsize) {
        t->hslot.release();
        TRY(dgrow(t->hslot, hs, s));
        t->hsize = hs;
        CK(cudaMemsetAsync(t->hslot.p, 0xff, sizeof(ulonglong2) * hs, s));
        if (old > 0) { k_rehash<<<148, 256, 0, s>>>(view(t)); counted(); }
        CK(cudaGetLastError());
    }
    return FS_OK;
}

static int trie_pull(fs_trie *t) {
    CK(cudaMemcpyAsync(&t->h_sc, t->sc.p, sizeof(TrieScalars), cudaMemcpyDeviceToHost, tstream(t)));
    CK(cudaStreamSynchronize(tstream(t)));
    return FS_OK;
}

extern "C" int fs_trie_create(fs_ctx *c, int64_t capacity, int track_workers, int n_workers, fs_trie **out) {
    if (!c || !out) return fail(FS_ERR_INVALID, "NULL argument");
    if (track_workers && (n_workers <= 0 || n_workers > 64)) return fail(FS_ERR_INVALID, "n_workers must be in [1, 64]");
    TRY(ctx_use(c));
    fs_trie *t = new fs_trie();
    t->ctx = c;
    t->capacity = capacity;
    t->track = track_workers ? 1 : 0;
    t->nw = track_workers ? n_workers : 0;
    // a local tree never holds more than capacity+1 nodes (every edge >= 1
    // token) plus one transient split top; the global index grows on demand
    const int64_t init = capacity >= 0 ? std::min<int64_t>(capacity + 8, 1 << 16) : 4096;
    t->h_sc.hw = 1;
    TRY(dgrow(t->sc, 1, c->stream));
    TRY(trie_reserve(t, init, c->max_len));
    const int64_t rc = capacity >= 0 ? 2 * capacity + 1024 : 1024;
    TRY(dgrow(t->rsrc, rc, c->stream)); TRY(dgrow(t->rlen, rc, c->stream)); TRY(dgrow(t->rkeep, rc, c->stream));
    TRY(dgrow(t->opout, 8, c->stream));
    TRY(hgrow(t->h_out, 8));
    k_trie_init<<<1, 32, 0, c->stream>>>(view(t), capacity);
    counted();
    CK(cudaGetLastError());
    TRY(trie_pull(t));
    *out = t;
    return FS_OK;
}

extern "C" int fs_trie_destroy(fs_trie *t) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t) return FS_OK;
    if (t->nworkers > 0) return fail(FS_ERR_INVALID, "destroy the tree's worker first");
    cudaSetDevice(t->ctx->device);
    cudaStreamSynchronize(tstream(t));
    t->src.release(); t->la.release(); t->seq.release(); t->start.release(); t->end.release();
    t->parent.release(); t->nchild.release(); t->ref.release(); t->first.release(); t->freest.release();
    t->flags.release(); t->wmask.release(); t->wtime.release(); t->hslot.release(); t->slen.release();
    t->lseq.release(); t->ctop.release(); t->cpar.release();
    t->sc.release(); t->pos.release(); t->chk.release(); t->h_chk.release(); t->segs.release(); t->found.release();
    t->rsrc.release(); t->rlen.release(); t->rkeep.release();
    t->opout.release(); t->h_out.release();
    t->h_unpin.release(); t->h_ustat.release(); t->ustat.release(); t->dunpin.release();
    if (t->ev_staged) cudaEventDestroy(t->ev_staged);
    if (t->ev[0]) { cudaEventDestroy(t->ev[0]); cudaEventDestroy(t->ev[1]); }
    t->nt_src.release(); t->nt_when.release(); t->nt_len.release(); t->nt_worker.release(); t->nt_keep.release();
    t->nt_s0.release(); t->nt_m0.release();
    delete t;
    return FS_OK;
}

extern "C" int fs_trie_stats(fs_trie *t, int64_t *used, int64_t *pinned, int64_t *next_seq, int64_t *nodes) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t) return fail(FS_ERR_INVALID, "NULL trie");
    if (used) *used = t->h_sc.used;
    if (pinned) *pinned = t->h_sc.pinned;
    if (next_seq) *next_seq = t->h_sc.next_seq;
    if (nodes) *nodes = t->h_sc.live;
    return FS_OK;
}

struct fs_scratch_match {
    DBuf<int32_t> ids, mlen, cov;
};

extern "C" int fs_trie_match(fs_trie *t, int64_t n, const int32_t *req_ids, int64_t now, int stamp,
                             int32_t *out_mlen, int32_t *out_cov) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    if (n == 0) return FS_OK;
    fs_ctx *c = t->ctx;
    TRY(ctx_use(c));
    for (int64_t i = 0; i < n; i++)
        if (req_ids[i] < 0 || req_ids[i] >= (int64_t)c->h_roff.size()) return fail(FS_ERR_INVALID, "bad request id");
    static thread_local fs_scratch_match sm;
    TRY(trie_reserve(t, 0, c->max_len));
    TRY(dgrow(sm.ids, n, c->stream)); TRY(dgrow(sm.mlen, n, c->stream)); TRY(dgrow(sm.cov, n, c->stream));
    CK(cudaMemcpyAsync(sm.ids.p, req_ids, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
    const int64_t blocks = (n * 32 + 255) / 256;
    const int64_t sq = stamp ? ++t->opseq : 0;
    k_match<4, false><<<(unsigned)blocks, 256, 0, c->stream>>>(view(t), sm.ids.p, (int32_t)n, c->roff.p, c->rlen.p, now,
                                                      stamp, sq, 0u, nullptr, sm.mlen.p, sm.cov.p, nullptr, nullptr,
                                                      nullptr, nullptr, K1Hints{});
    counted();
    CK(cudaGetLastError());
    if (out_mlen) CK(cudaMemcpyAsync(out_mlen, sm.mlen.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    if (out_cov) CK(cudaMemcpyAsync(out_cov, sm.cov.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return FS_OK;
}

static int copy_records(fs_trie *t, int64_t nrec, fs_records *recs) {
    if (!recs) return FS_OK;
    recs->n_rec = nrec;
    const int64_t k = std::min(nrec, recs->rec_cap);
    if (nrec > t->rsrc.cap) return fail(FS_ERR_INTERNAL, "eviction record sink overflow (%lld)", (long long)nrec);
    if (k > 0) {
        CK(cudaMemcpyAsync(recs->rec_src, t->rsrc.p, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, tstream(t)));
        CK(cudaMemcpyAsync(recs->rec_len, t->rlen.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, tstream(t)));
        CK(cudaMemcpyAsync(recs->rec_keep, t->rkeep.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, tstream(t)));
    }
    return FS_OK;
}

extern "C" int fs_trie_read_records(fs_trie *t, int64_t first, int64_t n, int64_t *src, int32_t *len,
                                    int32_t *keep) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t || first < 0 || n < 0 || first + n > t->rsrc.cap) return fail(FS_ERR_INVALID, "record range");
    TRY(ctx_use(t->ctx));
    cudaStream_t s = t->ctx->stream;
    if (n > 0) {
        if (src) CK(cudaMemcpyAsync(src, t->rsrc.p + first, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
        if (len) CK(cudaMemcpyAsync(len, t->rlen.p + first, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
        if (keep) CK(cudaMemcpyAsync(keep, t->rkeep.p + first, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    return FS_OK;
}

// Debug (FS_FILL_CHECK=1): k_check_fill's tree invariants after every
// per-call operation, completion unpin and at the start of every fill of a
// worker's cache, so a violation names the operation that made it.
static int tree_check(fs_trie *t, const char *where, int64_t arg) {
    static const bool on = [] { const char *e = getenv("FS_FILL_CHECK"); return e && atoi(e) != 0; }();
    if (!on || t->nw != 0) return FS_OK;  // worker caches only (the routing index holds no pins)
    cudaStream_t s = tstream(t);
    TRY(dgrow(t->chk, 8, s));
    TRY(hgrow(t->h_chk, 8));
    CK(cudaMemsetAsync(t->chk.p, 0, sizeof(int64_t) * 8, s));
    k_check_fill<<<64, 256, 0, s>>>(view(t), nullptr, t->chk.p, 0, t->chk.p);
    counted();
    CK(cudaMemcpyAsync(t->h_chk.p, t->chk.p, sizeof(int64_t) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (t->h_chk.p[2] != FS_OK)
        return fail(FS_ERR_INTERNAL, "tree check %lld at node %lld after %s (%lld)", (long long)t->h_chk.p[2],
                    (long long)t->h_chk.p[6], where, (long long)arg);
    return FS_OK;
}

static int run_op(fs_trie *t, OpArgs &a, int64_t *out5, fs_records *recs) {
    fs_ctx *c = t->ctx;
    a.t = view(t);
    a.segs = t->segs.p;
    a.found = t->found.p;
    a.out = t->opout.p;
    a.sq = ++t->opseq;
    if (a.op == OP_INSERT || a.op == OP_ADMIT || a.op == OP_EVICT || a.op == OP_NOTIFY) t->version++;
    k_op<<<1, 256, 0, tstream(t)>>>(a);
    counted();
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(t->h_out.p, t->opout.p, sizeof(int64_t) * 5, cudaMemcpyDeviceToHost, tstream(t)));
    CK(cudaMemcpyAsync(&t->h_sc, t->sc.p, sizeof(TrieScalars), cudaMemcpyDeviceToHost, tstream(t)));
    CK(cudaStreamSynchronize(tstream(t)));
    for (int i = 0; i < 5; i++) out5[i] = t->h_out.p[i];
    TRY(copy_records(t, out5[4], recs));
    CK(cudaStreamSynchronize(tstream(t)));
    TRY(tree_check(t, "a per-call operation", a.op));
    return FS_OK;
}

static int check_req(fs_trie *t, int32_t req) {
    if (req < 0 || req >= (int64_t)t->ctx->h_roff.size()) return fail(FS_ERR_INVALID, "bad request id %d", req);
    return FS_OK;
}

extern "C" int fs_trie_insert(fs_trie *t, int32_t req, int64_t now, int32_t worker, int32_t *new_len,
                              int32_t *path_node, fs_records *recs) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t) return fail(FS_ERR_INVALID, "NULL trie");
    TRY(ctx_use(t->ctx)); TRY(check_req(t, req));
    if (worker >= 0 && (!t->track || worker >= t->nw)) {
        if (t->track) return fail(FS_ERR_INVALID, "worker %d outside [0,%d)", worker, t->nw);
        worker = -1;  // worker tags only exist on a track_workers tree (radix.py:160)
    }
    TRY(trie_reserve(t, 2, t->ctx->max_len));
    OpArgs a{};
    a.op = OP_INSERT; a.req_off = t->ctx->h_roff[req]; a.len = t->ctx->h_rlen[req]; a.now = now; a.worker = worker;
    int64_t o[5];
    TRY(run_op(t, a, o, recs));
    if (new_len) *new_len = (int32_t)o[1];
    if (path_node) *path_node = (int32_t)o[2];
    if (o[0] == FS_ERR_CACHE_FULL) return fail(FS_ERR_CACHE_FULL, "cannot free %lld tokens", (long long)o[1]);
    if (o[0] != FS_OK) return fail((int)o[0], "device insert failed (status %lld)", (long long)o[0]);
    return FS_OK;
}

extern "C" int fs_trie_admit(fs_trie *t, int32_t req, int64_t now, int32_t *mlen, int32_t *path_node,
                             fs_records *recs) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t) return fail(FS_ERR_INVALID, "NULL trie");
    TRY(ctx_use(t->ctx)); TRY(check_req(t, req));
    TRY(trie_reserve(t, 2, t->ctx->max_len));
    OpArgs a{};
    a.op = OP_ADMIT; a.req_off = t->ctx->h_roff[req]; a.len = t->ctx->h_rlen[req]; a.now = now; a.worker = -1;
    int64_t o[5];
    TRY(run_op(t, a, o, recs));
    if (mlen) *mlen = (int32_t)o[1];
    if (path_node) *path_node = (int32_t)o[2];
    if (o[0] == FS_ERR_CACHE_FULL) return fail(FS_ERR_CACHE_FULL, "cannot free tokens for admit");
    if (o[0] != FS_OK) return fail((int)o[0], "device admit failed (status %lld)", (long long)o[0]);
    return FS_OK;
}

static int pin_op(fs_trie *t, int32_t node, int op) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t) return fail(FS_ERR_INVALID, "NULL trie");
    TRY(ctx_use(t->ctx));
    if (node < 0) return FS_OK;  // empty path
    if (node >= t->h_sc.hw) return fail(FS_ERR_INVALID, "bad path handle %d", node);
    TRY(trie_reserve(t, 0, t->ctx->max_len));
    OpArgs a{};
    a.op = op; a.node = node;
    int64_t o[5];
    TRY(run_op(t, a, o, nullptr));
    if (o[0] == FS_ERR_UNDERFLOW) return fail(FS_ERR_UNDERFLOW, "unpin below zero (radix.py:183)");
    if (o[0] != FS_OK) return fail((int)o[0], "pin/unpin failed");
    return FS_OK;
}
extern "C" int fs_trie_pin(fs_trie *t, int32_t node) { return pin_op(t, node, OP_PIN); }
extern "C" int fs_trie_unpin(fs_trie *t, int32_t node) { return pin_op(t, node, OP_UNPIN); }

static int unpin_settle(fs_trie *t);

extern "C" int fs_trie_unpin_many(fs_trie *t, int64_t n, const int32_t *nodes) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    TRY(unpin_settle(t));
    if (n == 0) return FS_OK;
    TRY(ctx_use(t->ctx));
    for (int64_t i = 0; i < n; i++)
        if (nodes[i] >= t->h_sc.hw) return fail(FS_ERR_INVALID, "bad path handle %d", nodes[i]);
    cudaStream_t s = t->ctx->stream;
    static thread_local DBuf<int32_t> dn;
    TRY(dgrow(dn, n, s));
    CK(cudaMemcpyAsync(dn.p, nodes, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(t->opout.p, 0, sizeof(int64_t), s));
    if (!t->ev[0]) { CK(cudaEventCreate(&t->ev[0])); CK(cudaEventCreate(&t->ev[1])); }
    CK(cudaEventRecord(t->ev[0], s));
    k_unpin_many<<<(unsigned)((n * 32 + 127) / 128), 128, 0, s>>>(view(t), dn.p, n, t->opout.p);
    counted();
    CK(cudaGetLastError());
    CK(cudaEventRecord(t->ev[1], s));
    CK(cudaMemcpyAsync(t->h_out.p, t->opout.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&t->h_sc, t->sc.p, sizeof(TrieScalars), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaEventElapsedTime(&t->last_ms, t->ev[0], t->ev[1]));
    if (t->h_out.p[0] == FS_ERR_UNDERFLOW) return fail(FS_ERR_UNDERFLOW, "unpin below zero (radix.py:183)");
    TRY(tree_check(t, "unpin_many", n));
    if (t->h_out.p[0] != FS_OK) return fail((int)t->h_out.p[0], "unpin_many failed");
    return FS_OK;
}

// Settle an fs_trie_unpin_many_async: wait for it, take its device time and
// report its status (FS_ERR_UNDERFLOW like fs_trie_unpin_many).
static int unpin_settle(fs_trie *t) {
    if (!t->unpin_pending) return FS_OK;
    t->unpin_pending = false;
    CK(cudaEventSynchronize(t->ev[1]));
    CK(cudaStreamSynchronize(t->ctx->stream));  // the status read-back follows the kernel
    CK(cudaEventElapsedTime(&t->last_ms, t->ev[0], t->ev[1]));
    if (t->h_ustat.p[0] == FS_ERR_UNDERFLOW) return fail(FS_ERR_UNDERFLOW, "unpin below zero (radix.py:183)");
    if (t->h_ustat.p[0] != FS_OK) return fail((int)t->h_ustat.p[0], "unpin_many failed");
    TRY(tree_check(t, "unpin_many_async", 0));
    return FS_OK;
}

extern "C" int fs_trie_unpin_many_async(fs_trie *t, int64_t n, const int32_t *nodes) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    TRY(unpin_settle(t));
    if (n == 0) return FS_OK;
    TRY(ctx_use(t->ctx));
    for (int64_t i = 0; i < n; i++)
        if (nodes[i] >= t->h_sc.hw) return fail(FS_ERR_INVALID, "bad path handle %d", nodes[i]);
    cudaStream_t s = t->ctx->stream;
    if (!t->ev[0]) { CK(cudaEventCreate(&t->ev[0])); CK(cudaEventCreate(&t->ev[1])); }
    if (!t->ev_staged) CK(cudaEventCreateWithFlags(&t->ev_staged, cudaEventDisableTiming));
    CK(cudaEventSynchronize(t->ev_staged));  // the staging buffer's last copy has left
    TRY(hgrow(t->h_unpin, n)); TRY(hgrow(t->h_ustat, 1));
    TRY(dgrow(t->dunpin, n, s)); TRY(dgrow(t->ustat, 1, s));
    std::memcpy(t->h_unpin.p, nodes, sizeof(int32_t) * n);
    CK(cudaMemcpyAsync(t->dunpin.p, t->h_unpin.p, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(t->ev_staged, s));
    CK(cudaMemsetAsync(t->ustat.p, 0, sizeof(int64_t), s));
    CK(cudaEventRecord(t->ev[0], s));
    k_unpin_many<<<(unsigned)((n * 32 + 127) / 128), 128, 0, s>>>(view(t), t->dunpin.p, n, t->ustat.p);
    counted();
    CK(cudaGetLastError());
    CK(cudaEventRecord(t->ev[1], s));
    CK(cudaMemcpyAsync(t->h_ustat.p, t->ustat.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    t->unpin_pending = true;
    return FS_OK;
}

extern "C" int fs_trie_last_ms(fs_trie *t, float *ms) {
    if (!t || !ms) return fail(FS_ERR_INVALID, "NULL argument");
    TRY(unpin_settle(t));
    *ms = t->last_ms;
    return FS_OK;
}

extern "C" int fs_trie_evict_lru(fs_trie *t, int64_t needed, fs_records *recs) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t) return fail(FS_ERR_INVALID, "NULL trie");
    TRY(ctx_use(t->ctx));
    OpArgs a{};
    a.op = OP_EVICT; a.needed = needed;
    int64_t o[5];
    TRY(run_op(t, a, o, recs));
    if (o[0] != FS_OK) return fail((int)o[0], "evict failed");
    return FS_OK;
}

extern "C" int fs_trie_longest_match_workers(fs_trie *t, int32_t req, int64_t now, int32_t *mlen, uint64_t *mask) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t) return fail(FS_ERR_INVALID, "NULL trie");
    TRY(ctx_use(t->ctx)); TRY(check_req(t, req));
    TRY(trie_reserve(t, 0, t->ctx->max_len));
    OpArgs a{};
    a.op = OP_LMW; a.req_off = t->ctx->h_roff[req]; a.len = t->ctx->h_rlen[req]; a.now = now;
    int64_t o[5];
    TRY(run_op(t, a, o, nullptr));
    if (mlen) *mlen = (int32_t)o[1];
    if (mask) *mask = (uint64_t)o[3];
    return FS_OK;
}

extern "C" int fs_trie_evict_notify(fs_trie *t, int64_t path_src, int32_t path_len, int32_t worker,
                                    int32_t keep_len, int64_t notice_time) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t || !t->track) return fail(FS_ERR_INVALID, "evict_notify needs a track_workers trie");
    TRY(ctx_use(t->ctx));
    if (path_src < 0 || path_len < 0 || path_src + path_len > t->ctx->arena_used) return fail(FS_ERR_INVALID, "path range");
    TRY(trie_reserve(t, 2, std::max(t->ctx->max_len, path_len)));
    OpArgs a{};
    a.op = OP_NOTIFY; a.req_off = path_src; a.len = path_len; a.worker = worker; a.keep = keep_len; a.notice = notice_time;
    int64_t o[5];
    TRY(run_op(t, a, o, nullptr));
    if (o[0] != FS_OK) return fail((int)o[0], "evict_notify failed");
    return FS_OK;
}

extern "C" int fs_trie_evict_notify_many(fs_trie *t, int64_t n, const int64_t *path_src, const int32_t *path_len,
                                         const int32_t *worker, const int32_t *keep_len, const int64_t *notice_time) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t || !t->track) return fail(FS_ERR_INVALID, "evict_notify needs a track_workers trie");
    if (n < 0) return fail(FS_ERR_INVALID, "bad count");
    if (n == 0) return FS_OK;
    fs_ctx *c = t->ctx;
    TRY(ctx_use(c));
    int32_t maxlen = c->max_len;
    for (int64_t i = 0; i < n; i++) {
        if (path_src[i] < 0 || path_len[i] < 0 || path_src[i] + path_len[i] > c->arena_used)
            return fail(FS_ERR_INVALID, "path range of notice %lld", (long long)i);
        if (worker[i] < 0 || worker[i] >= t->nw) return fail(FS_ERR_INVALID, "worker of notice %lld", (long long)i);
        maxlen = std::max(maxlen, path_len[i]);
    }
    cudaStream_t s = tstream(t);
    TRY(trie_reserve(t, 2 * n, maxlen));
    TRY(dgrow(t->nt_src, n, s)); TRY(dgrow(t->nt_when, n, s)); TRY(dgrow(t->nt_len, n, s));
    TRY(dgrow(t->nt_worker, n, s)); TRY(dgrow(t->nt_keep, n, s));
    CK(cudaMemcpyAsync(t->nt_src.p, path_src, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(t->nt_when.p, notice_time, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(t->nt_len.p, path_len, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(t->nt_worker.p, worker, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(t->nt_keep.p, keep_len, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    // batch-start matches of every path in parallel (K1 over arena ranges, no
    // stamping); the serial chain resumes each walk from them
    TRY(dgrow(t->nt_m0, n, s)); TRY(dgrow(t->nt_s0, n, s));
    k_match<1, true><<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(
        view(t), nullptr, (int32_t)n, t->nt_src.p, t->nt_len.p, 0, 0, 0, 0u, nullptr, t->nt_m0.p, nullptr, nullptr,
        t->nt_s0.p, nullptr, nullptr, K1Hints{});
    counted();
    k_notify_many<<<1, 256, 0, s>>>(view(t), (int32_t)n, t->nt_src.p, t->nt_len.p, t->nt_worker.p, t->nt_keep.p,
                                    t->nt_when.p, t->nt_m0.p, t->nt_s0.p, t->segs.p, t->found.p, t->opout.p);
    counted();
    CK(cudaGetLastError());
    t->opseq += 1;
    t->version++;
    CK(cudaMemcpyAsync(t->h_out.p, t->opout.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&t->h_sc, t->sc.p, sizeof(TrieScalars), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (t->h_out.p[0] != FS_OK) return fail((int)t->h_out.p[0], "evict_notify_many failed");
    return FS_OK;
}

extern "C" int fs_trie_last_notify_profile(fs_trie *t, int64_t *prof4) {
    if (!t || !prof4) return fail(FS_ERR_INVALID, "NULL argument");
    TRY(ctx_use(t->ctx));
    CK(cudaMemcpyAsync(prof4, t->opout.p + 1, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, tstream(t)));
    CK(cudaStreamSynchronize(tstream(t)));
    return FS_OK;
}

extern "C" int fs_trie_export(fs_trie *t, int64_t cap, int64_t *n, int64_t *src, int32_t *start, int32_t *end,
                              int32_t *parent, int32_t *ref, int64_t *last_access, uint64_t *wmask) {
    if (t && t->busy) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!t || !n) return fail(FS_ERR_INVALID, "NULL argument");
    TRY(ctx_use(t->ctx));
    TRY(trie_pull(t));
    const int64_t hw = t->h_sc.hw;
    *n = hw;
    const int64_t k = std::min(cap, hw);
    cudaStream_t s = t->ctx->stream;
    if (k > 0) {
        if (src) CK(cudaMemcpyAsync(src, t->src.p, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
        if (start) CK(cudaMemcpyAsync(start, t->start.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
        if (end) CK(cudaMemcpyAsync(end, t->end.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
        if (parent) CK(cudaMemcpyAsync(parent, t->parent.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
        if (ref) CK(cudaMemcpyAsync(ref, t->ref.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, s));
        if (wmask && t->track) CK(cudaMemcpyAsync(wmask, t->wmask.p, sizeof(uint64_t) * k, cudaMemcpyDeviceToHost, s));
        if (wmask && !t->track) std::memset(wmask, 0, sizeof(uint64_t) * k);
    }
    if (last_access && k > 0) {
        // device la holds the latest stamp of a path ending at each node; the
        // reference's last_access is the most recent stamp in its subtree
        std::vector<int64_t> la(hw), lsq(hw);
        std::vector<int32_t> par(hw), dep(hw);
        CK(cudaMemcpyAsync(la.data(), t->la.p, sizeof(int64_t) * hw, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(lsq.data(), t->lseq.p, sizeof(int64_t) * hw, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(par.data(), t->parent.p, sizeof(int32_t) * hw, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(dep.data(), t->end.p, sizeof(int32_t) * hw, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<int32_t> order;
        for (int32_t i = 1; i < hw; i++) if (par[i] >= 0) order.push_back(i);
        std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return dep[a] > dep[b]; });
        for (int32_t i : order)
            if (par[i] > 0 && lsq[i] > lsq[par[i]]) { la[par[i]] = la[i]; lsq[par[i]] = lsq[i]; }
        std::memcpy(last_access, la.data(), sizeof(int64_t) * k);
    }
    CK(cudaStreamSynchronize(s));
    return FS_OK;
}

// ---------------------------------------------------------------- worker
struct fs_worker {
    fs_ctx *ctx = nullptr;
    fs_trie *tree = nullptr;
    bool inflight = false;           // between fs_worker_fill_begin and fs_worker_fill_end
    HBuf<uint8_t> h_stage;           // page-locked staging of a fill's results
    int64_t f_n = 0, f_launches0 = 0;
    std::chrono::steady_clock::time_point f_h0, f_h1, f_h2;
    int32_t wid = 0;                 // unique id (owner of K1 match hints)
    int64_t hint_version = -1;       // tree version at the end of the last fill
    bool hints_ok = false;           // last fill completed with a complete admission filter
    bool k1_full = false;            // fs_worker_set_option(FS_OPT_K1_FULL): ignore match hints
    int policy = 0;
    int64_t quantum = 1, M = 0, R = 0, w_e = 1, w_q = 2;
    int32_t nclients = 0;
    // host shadows (authoritative between fills for the monitor's reads)
    std::vector<int64_t> h_q, h_refills;
    std::vector<uint8_t> h_known;
    std::vector<int32_t> dl_client;
    std::vector<int64_t> dl_delta;
    DBuf<int64_t> q, refills;
    DBuf<uint8_t> known;
    DBuf<int32_t> pend_cnt;
    bool known_dirty = false;
    // queue mirror
    std::vector<int32_t> pending_new;
    int64_t qn = 0;          // entries in `queue` (label order)
    int64_t admitted_last = 0;
    DBuf<int32_t> queue, queue2, newids, ins;
    DBuf<int64_t> newlab;
    DBuf<uint32_t> keys;
    DBuf<int32_t> mlen, cov, fnode, next;
    DBuf<int32_t> s_req, s_len, s_fnode, s_mlen0, s_tok0;
    // queue order (fs_order.cuh): previous fill's sorted ids, settled marks,
    // B sort buffers, A's (key, position) pairs, look-back status words
    DBuf<int32_t> p_req, p_len, p_mlen0, p_tok0;
    DBuf<int64_t> p_src0;
    int64_t prev_n = 0;
    bool prev_ok = false;            // p_req holds the last K1 fill's sorted order
    DBuf<int64_t> settled;
    int64_t stag = 0;
    DBuf<uint32_t> bkey, bkey2, bkey3;
    DBuf<int32_t> bpos, bpos2, bpos3, sblk;
    DBuf<uint8_t> slow_flag;
    DBuf<unsigned long long> akq, st_up, st_ma;
    DBuf<OrderCtl> octl;
    uint32_t lb_epoch = 0;
    DBuf<SweepCtl> ctl;
    DBuf<int32_t> vrank, vhead;  // VTC: client name ranks, per-client head scratch
    std::vector<int32_t> h_vrank;
    bool vrank_dirty = true;
    DBuf<FevCtl> fev_ctl;          // asynchronous cold eviction (k_schedule CTA 1)
    DBuf<int64_t> fev_need, fev_rec_end;
    DBuf<int32_t> fev_free;
    DBuf<unsigned char> fev_vrec;
    int32_t fev_tag = 0;
    DBuf<int32_t> k1jobs, k1njobs;  // K1 positions the fast path left to the walk
    DBuf<int32_t> tok0q;            // K1: token at each queue position's match (miss key)
    DBuf<int32_t> rw_list;
    DBuf<unsigned long long> gkey;
    DBuf<int32_t> gep;
    int nhelp = -1;  // helper CTAs of the grid sweep (-1: not yet sized)
    DBuf<int64_t> s0, s_src0;
    DBuf<int4> slot;
    DBuf<int32_t> dlc;
    DBuf<int64_t> dld;
    // outputs
    DBuf<int32_t> adm_req, adm_mlen, adm_node;
    DBuf<int64_t> adm_unp, adm_pinb, adm_rec_end, hdr;
    HBuf<int64_t> h_hdr;
    HBuf<int32_t> h_st32;
    HBuf<int64_t> h_st64;
    cudaEvent_t ev[5];
    cudaEvent_t ev_done = nullptr, ev_prev_done = nullptr;  // end of the result staging (this / last fill)
    float gaps[2] = {-1.f, -1.f};
    bool gaps_ready = false, have_prev_done = false;  // [staging after the fill, GPU time from the last fill's staging end to this fill]
    float phases[4] = {0, 0, 0, 0};
    DBuf<int64_t> alg;         // K1 algorithmic-token accumulator
    int64_t stats[24] = {0};
    int64_t stats_ext[8] = {0};  // hdr[24..31]: scheduler cycle counters (pin, on_walk, evictor-setup waits)
};

__global__ void k_set_state(int8_t *st, const int32_t *ids, int64_t n, int8_t v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) st[ids[i]] = v;
}

extern "C" int fs_worker_create(fs_ctx *c, fs_trie *tree, int policy, int64_t quantum, int64_t M,
                                int64_t output_reserve, int64_t w_e, int64_t w_q, int32_t max_clients,
                                fs_worker **out) {
    if (!c || !tree || !out || tree->ctx != c) return fail(FS_ERR_INVALID, "bad arguments");
    if (policy != 0 && policy != 1 && policy != 2) return fail(FS_ERR_INVALID, "policy must be 0 (dlpm), 1 (lpm) or 2 (vtc)");
    if (policy == 0 && quantum <= 0) return fail(FS_ERR_INVALID, "quantum must be positive");  // local_policies.py:81-82
    if (max_clients <= 0) return fail(FS_ERR_INVALID, "max_clients must be positive");
    // a Worker owns its cache (worker.py:72): a second scheduler on the same
    // tree would not see the first one's admissions in its match hints and
    // admission filter
    if (tree->nworkers > 0) return fail(FS_ERR_INVALID, "the tree already has a worker (one worker per RadixTree)");
    if (tree->track) return fail(FS_ERR_INVALID, "a worker needs a local tree (track_workers = 0)");
    TRY(ctx_use(c));
    fs_worker *w = new fs_worker();
    tree->nworkers++;
    static std::atomic<int32_t> next_wid{0};
    w->wid = next_wid.fetch_add(1);
    w->ctx = c; w->tree = tree; w->policy = policy; w->quantum = quantum > 0 ? quantum : 1;
    w->M = M; w->R = output_reserve; w->w_e = w_e; w->w_q = w_q; w->nclients = max_clients;
    w->h_q.assign(max_clients, 0); w->h_refills.assign(max_clients, 0); w->h_known.assign(max_clients, 0);
    TRY(dgrow(w->q, max_clients, c->stream)); TRY(dgrow(w->refills, max_clients, c->stream));
    TRY(dgrow(w->known, max_clients, c->stream)); TRY(dgrow(w->pend_cnt, max_clients, c->stream));
    CK(cudaMemsetAsync(w->q.p, 0, sizeof(int64_t) * max_clients, c->stream));
    CK(cudaMemsetAsync(w->refills.p, 0, sizeof(int64_t) * max_clients, c->stream));
    CK(cudaMemsetAsync(w->known.p, 0, max_clients, c->stream));
    CK(cudaMemsetAsync(w->pend_cnt.p, 0, sizeof(int32_t) * max_clients, c->stream));
    TRY(dgrow(w->hdr, 32, c->stream)); TRY(hgrow(w->h_hdr, 32 + 128));
    TRY(dgrow(w->octl, 1, c->stream));
    TRY(dgrow(w->alg, 128, c->stream));
    for (int i = 0; i < 5; i++) CK(cudaEventCreate(&w->ev[i]));
    CK(cudaStreamSynchronize(c->stream));
    *out = w;
    return FS_OK;
}

extern "C" int fs_worker_destroy(fs_worker *w) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w) return FS_OK;
    cudaSetDevice(w->ctx->device);
    cudaStreamSynchronize(w->ctx->stream);
    w->tree->nworkers--;
    w->q.release(); w->refills.release(); w->known.release(); w->pend_cnt.release(); w->h_stage.release();
    w->queue.release(); w->queue2.release(); w->newids.release(); w->newlab.release();
    w->keys.release(); w->mlen.release(); w->ins.release(); w->p_req.release(); w->settled.release();
    w->p_len.release(); w->p_mlen0.release(); w->p_tok0.release(); w->p_src0.release();
    w->s0.release(); w->s_mlen0.release(); w->s_src0.release(); w->alg.release();
    w->bkey.release(); w->bkey2.release(); w->bpos.release(); w->bpos2.release(); w->akq.release();
    w->bkey3.release(); w->bpos3.release(); w->sblk.release(); w->slow_flag.release();
    w->st_up.release(); w->st_ma.release(); w->octl.release();
    w->cov.release(); w->fnode.release(); w->next.release(); w->s_req.release(); w->s_len.release();
    w->s_fnode.release(); w->s_tok0.release(); w->ctl.release(); w->vrank.release(); w->vhead.release(); w->fev_ctl.release(); w->fev_need.release(); w->fev_rec_end.release(); w->fev_free.release(); w->fev_vrec.release(); w->tok0q.release(); w->k1jobs.release(); w->k1njobs.release(); w->rw_list.release(); w->gkey.release(); w->gep.release(); w->slot.release(); w->dlc.release();
    w->dld.release(); w->adm_req.release(); w->adm_mlen.release(); w->adm_node.release();
    w->adm_unp.release(); w->adm_pinb.release(); w->adm_rec_end.release(); w->hdr.release();
    w->h_hdr.release(); w->h_st32.release(); w->h_st64.release();
    for (int i = 0; i < 5; i++) cudaEventDestroy(w->ev[i]);
    if (w->ev_done) cudaEventDestroy(w->ev_done);
    if (w->ev_prev_done) cudaEventDestroy(w->ev_prev_done);
    delete w;
    return FS_OK;
}

extern "C" int fs_worker_enqueue(fs_worker *w, int64_t n, const int32_t *ids) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    fs_ctx *c = w->ctx;
    for (int64_t i = 0; i < n; i++) {
        const int32_t r = ids[i];
        if (r < 0 || r >= (int64_t)c->h_roff.size()) return fail(FS_ERR_INVALID, "bad request id %d", r);
        const int32_t cl = c->h_rclient[r];
        if (cl < 0 || cl >= w->nclients) return fail(FS_ERR_INVALID, "client id %d outside [0,%d)", cl, w->nclients);
        w->pending_new.push_back(r);
        if (!w->h_known[cl]) {  // Dlpm.on_request_enqueued (local_policies.py:88-92)
            w->h_known[cl] = 1;
            w->known_dirty = true;
        }
    }
    return FS_OK;
}

extern "C" int fs_worker_outputs(fs_worker *w, int64_t n, const int32_t *clients, const int64_t *counts) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    for (int64_t i = 0; i < n; i++) {
        const int32_t cl = clients[i];
        if (cl < 0 || cl >= w->nclients) return fail(FS_ERR_INVALID, "client id %d out of range", cl);
        if (w->policy == 1) continue;  // Lpm keeps no counters
        // Dlpm.on_outputs subtracts (local_policies.py:130-133), Vtc.on_outputs adds (191-194)
        const int64_t d = (w->policy == 2 ? 1 : -1) * w->w_q * counts[i];
        w->h_q[cl] += d;  // mirror; the device applies the same delta at the next fill
        w->dl_client.push_back(cl);
        w->dl_delta.push_back(d);
    }
    return FS_OK;
}

static int worker_flush_small(fs_worker *w) {
    fs_ctx *c = w->ctx;
    if (w->known_dirty) {
        CK(cudaMemcpyAsync(w->known.p, w->h_known.data(), w->nclients, cudaMemcpyHostToDevice, c->stream));
        w->known_dirty = false;
    }
    return FS_OK;
}

extern "C" int fs_worker_check_refill(fs_worker *w, int64_t n, const int32_t *queued, int *refilled) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w) return fail(FS_ERR_INVALID, "NULL worker");
    fs_ctx *c = w->ctx;
    TRY(ctx_use(c));
    TRY(worker_flush_small(w));
    // apply pending on_outputs deltas first so device q == host mirror
    std::vector<int64_t> q(w->h_q);
    CK(cudaMemcpyAsync(w->q.p, q.data(), sizeof(int64_t) * w->nclients, cudaMemcpyHostToDevice, c->stream));
    w->dl_client.clear(); w->dl_delta.clear();
    std::vector<uint8_t> flags(w->nclients, 0);
    for (int64_t i = 0; i < n; i++) {
        if (queued[i] < 0 || queued[i] >= w->nclients) return fail(FS_ERR_INVALID, "client id out of range");
        flags[queued[i]] = 1;
    }
    DBuf<uint8_t> dq;
    TRY(dgrow(dq, w->nclients, c->stream));
    CK(cudaMemcpyAsync(dq.p, flags.data(), w->nclients, cudaMemcpyHostToDevice, c->stream));
    k_check_refill<<<1, 32, 0, c->stream>>>(w->q.p, w->refills.p, w->known.p, w->nclients, dq.p, w->quantum, w->hdr.p);
    counted();
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(w->h_hdr.p, w->hdr.p, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(w->h_q.data(), w->q.p, sizeof(int64_t) * w->nclients, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(w->h_refills.data(), w->refills.p, sizeof(int64_t) * w->nclients, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    dq.release();
    if (refilled) *refilled = (int)w->h_hdr.p[0];
    return FS_OK;
}

extern "C" int fs_worker_counters(fs_worker *w, int32_t n, int64_t *q, int64_t *refills, uint8_t *known) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w) return fail(FS_ERR_INVALID, "NULL worker");
    const int32_t k = std::min(n, w->nclients);
    if (q) std::memcpy(q, w->h_q.data(), sizeof(int64_t) * k);
    if (refills) std::memcpy(refills, w->h_refills.data(), sizeof(int64_t) * k);
    if (known) std::memcpy(known, w->h_known.data(), k);
    return FS_OK;
}

extern "C" int fs_worker_set_counter(fs_worker *w, int32_t client, int64_t qv) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w || client < 0 || client >= w->nclients) return fail(FS_ERR_INVALID, "bad client");
    const int64_t d = qv - w->h_q[client];
    w->h_q[client] = qv;
    w->dl_client.push_back(client);
    w->dl_delta.push_back(d);
    return FS_OK;
}

extern "C" int fs_worker_set_client_ranks(fs_worker *w, int32_t n, const int32_t *ranks) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w || n < 0 || (n > 0 && !ranks)) return fail(FS_ERR_INVALID, "bad arguments");
    if ((int64_t)w->h_vrank.size() < n) w->h_vrank.resize(n);
    for (int32_t i = 0; i < n; i++) w->h_vrank[i] = ranks[i];
    w->vrank_dirty = true;
    return FS_OK;
}

extern "C" int fs_worker_reserve_clients(fs_worker *w, int32_t max_clients) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w) return fail(FS_ERR_INVALID, "NULL worker");
    if (max_clients <= w->nclients) return FS_OK;
    fs_ctx *c = w->ctx;
    cudaStream_t s = c->stream;
    TRY(ctx_use(c));
    const int32_t old = w->nclients;
    const int32_t nc = std::max(max_clients, old * 2);
    TRY(dgrow(w->q, nc, s, true, old)); TRY(dgrow(w->refills, nc, s, true, old));
    TRY(dgrow(w->known, nc, s, true, old)); TRY(dgrow(w->pend_cnt, nc, s, true, old));
    CK(cudaMemsetAsync(w->pend_cnt.p + old, 0, sizeof(int32_t) * (nc - old), s));
    CK(cudaMemsetAsync(w->q.p + old, 0, sizeof(int64_t) * (nc - old), s));
    CK(cudaMemsetAsync(w->refills.p + old, 0, sizeof(int64_t) * (nc - old), s));
    CK(cudaMemsetAsync(w->known.p + old, 0, nc - old, s));
    w->h_q.resize(nc, 0); w->h_refills.resize(nc, 0); w->h_known.resize(nc, 0);
    w->nclients = nc;
    CK(cudaStreamSynchronize(s));
    return FS_OK;
}

extern "C" int fs_worker_mark_known(fs_worker *w, int64_t n, const int32_t *clients) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w) return fail(FS_ERR_INVALID, "NULL worker");
    for (int64_t i = 0; i < n; i++) {
        if (clients[i] < 0 || clients[i] >= w->nclients) return fail(FS_ERR_INVALID, "client id out of range");
        if (!w->h_known[clients[i]]) { w->h_known[clients[i]] = 1; w->known_dirty = true; }
    }
    return FS_OK;
}

extern "C" int fs_worker_device_counters(fs_worker *w, int32_t n, int64_t *q, int64_t *refills) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w) return fail(FS_ERR_INVALID, "NULL worker");
    TRY(ctx_use(w->ctx));
    const int32_t k = std::min(n, w->nclients);
    if (q) CK(cudaMemcpyAsync(q, w->q.p, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, w->ctx->stream));
    if (refills) CK(cudaMemcpyAsync(refills, w->refills.p, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, w->ctx->stream));
    CK(cudaStreamSynchronize(w->ctx->stream));
    return FS_OK;
}

extern "C" int fs_worker_queue_len(fs_worker *w, int64_t *n) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w || !n) return fail(FS_ERR_INVALID, "NULL");
    *n = w->qn - w->admitted_last + (int64_t)w->pending_new.size();
    return FS_OK;
}

extern "C" int fs_worker_set_option(fs_worker *w, int option, int64_t value) {
    if (w && w->inflight) return fail(FS_ERR_INVALID, "a fill is in flight (call fs_worker_fill_end first)");
    if (!w) return fail(FS_ERR_INVALID, "NULL worker");
    switch (option) {
        case 1: w->k1_full = value != 0; return FS_OK;  // FS_OPT_K1_FULL
        default: return fail(FS_ERR_INVALID, "unknown option %d", option);
    }
}

extern "C" int fs_worker_last_stats(fs_worker *w, int64_t *stats16) {
    if (!w || !stats16) return fail(FS_ERR_INVALID, "NULL");
    for (int i = 0; i < 24; i++) stats16[i] = w->stats[i];
    return FS_OK;
}

extern "C" int fs_worker_last_stats_ext(fs_worker *w, int64_t *ext8) {
    if (!w || !ext8) return fail(FS_ERR_INVALID, "NULL");
    for (int i = 0; i < 8; i++) ext8[i] = w->stats_ext[i];
    return FS_OK;
}

extern "C" int fs_worker_last_gaps(fs_worker *w, float *ms2) {
    if (!w || !ms2) return fail(FS_ERR_INVALID, "NULL");
    ms2[0] = w->gaps[0];
    ms2[1] = w->gaps[1];
    return FS_OK;
}

extern "C" int fs_worker_last_phases(fs_worker *w, float *ms4) {
    if (!w || !ms4) return fail(FS_ERR_INVALID, "NULL");
    for (int i = 0; i < 4; i++) ms4[i] = w->phases[i];
    return FS_OK;
}

// Look-back status words are tagged with a launch epoch; a fresh buffer is
// zeroed so that no stale word can carry a live epoch.
static int st_grow(DBuf<unsigned long long> &b, int64_t n, cudaStream_t s) {
    const int64_t old = b.cap;
    TRY(dgrow(b, n, s));
    if (b.cap != old) CK(cudaMemsetAsync(b.p, 0, sizeof(unsigned long long) * b.cap, s));
    return FS_OK;
}

static uint32_t lb_next(fs_worker *w, cudaStream_t s) {
    if (++w->lb_epoch >= FS_LB_EPOCH_MASK) {
        // epoch wrap (every 16M launches): forget every status word
        DBuf<unsigned long long> *bufs[] = {&w->st_up, &w->st_ma};
        for (auto *b : bufs)
            if (b->p) cudaMemsetAsync(b->p, 0, sizeof(unsigned long long) * b->cap, s);
        w->lb_epoch = 1;
    }
    return w->lb_epoch;
}

static uint32_t key_bits(int32_t max_len) {
    uint32_t b = 1;
    while (((int64_t)1 << b) <= max_len) b++;
    return b;
}

// A fill's results: one kernel queued right behind the scheduler writes them
// straight into mapped page-locked staging (the scalars, the counters, the
// header and -- up to FS_RES_SPEC rows -- the admissions and eviction
// records; only the rows the fill produced), so fs_worker_fill_end waits once
// and copies out.  (Fourteen separate DMA copies of the whole capacity cost
// ~80 us of GPU-side latency per fill after the scheduler ended.)
#ifndef FS_RES_SPEC
#define FS_RES_SPEC 2048
#endif
struct StageLayout {
    int64_t K, R;
    size_t o_sc, o_q, o_rf, o_ar, o_am, o_an, o_au, o_ap, o_ae, o_rs, o_rl, o_rk, bytes;
};
static StageLayout stage_layout(fs_worker *w) {
    StageLayout L{};
    fs_trie *t = w->tree;
    L.K = std::min<int64_t>(w->adm_req.cap, FS_RES_SPEC);
    L.R = std::min<int64_t>(t->rsrc.cap, FS_RES_SPEC);
    const int64_t nc = w->nclients;
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off += (bytes + 15) & ~(size_t)15; return o; };
    L.o_sc = take(sizeof(TrieScalars)); L.o_q = take(8 * nc); L.o_rf = take(8 * nc);
    L.o_ar = take(4 * L.K); L.o_am = take(4 * L.K); L.o_an = take(4 * L.K); L.o_au = take(8 * L.K);
    L.o_ap = take(8 * L.K); L.o_ae = take(8 * L.K); L.o_rs = take(8 * L.R); L.o_rl = take(4 * L.R);
    L.o_rk = take(4 * L.R);
    L.bytes = off;
    return L;
}
struct StageArgs {
    const TrieScalars *sc;
    const int64_t *q, *refills;
    const int32_t *ar, *am, *an;
    const int64_t *au, *ap, *ae;
    const int64_t *rs;
    const int32_t *rl, *rk;
    const int64_t *hdr, *alg;
    uint8_t *hs;   // staging (device view of the mapped host buffer)
    int64_t *hh;   // header + K1 counters (32 + 128)
    int64_t nc, K, R;
    int64_t o_sc, o_q, o_rf, o_ar, o_am, o_an, o_au, o_ap, o_ae, o_rs, o_rl, o_rk;
};
// One warp per array (their loads are independent: no array waits for the
// previous one's round trip), lanes stride over the rows.
template <typename T>
__device__ __forceinline__ void stage_copy(uint8_t *hs, int64_t o, const T *src, int64_t n, int lane) {
    T *d = reinterpret_cast<T *>(hs + o);
    for (int64_t i = lane; i < n; i += 32) d[i] = src[i];
}
__global__ void __launch_bounds__(512) k_stage_results(StageArgs a) {
    const int64_t nadm = min(max(a.hdr[0], (int64_t)0), a.K), nrec = min(max(a.hdr[1], (int64_t)0), a.R);
    const int lane = threadIdx.x & 31;
    switch (threadIdx.x >> 5) {
        case 0: for (int i = lane; i < 32 + 128; i += 32) a.hh[i] = i < 32 ? a.hdr[i] : a.alg[i - 32]; break;
        case 1: stage_copy(a.hs, a.o_sc, reinterpret_cast<const int32_t *>(a.sc), (int64_t)(sizeof(TrieScalars) / 4), lane); break;
        case 2: stage_copy(a.hs, a.o_q, a.q, a.nc, lane); break;
        case 3: stage_copy(a.hs, a.o_rf, a.refills, a.nc, lane); break;
        case 4: stage_copy(a.hs, a.o_ar, a.ar, nadm, lane); break;
        case 5: stage_copy(a.hs, a.o_am, a.am, nadm, lane); break;
        case 6: stage_copy(a.hs, a.o_an, a.an, nadm, lane); break;
        case 7: stage_copy(a.hs, a.o_au, a.au, nadm, lane); break;
        case 8: stage_copy(a.hs, a.o_ap, a.ap, nadm, lane); break;
        case 9: stage_copy(a.hs, a.o_ae, a.ae, nadm, lane); break;
        case 10: stage_copy(a.hs, a.o_rs, a.rs, nrec, lane); break;
        case 11: stage_copy(a.hs, a.o_rl, a.rl, nrec, lane); break;
        case 12: stage_copy(a.hs, a.o_rk, a.rk, nrec, lane); break;
        default: break;
    }
}
static_assert(sizeof(TrieScalars) % 4 == 0, "scalars are staged as 32-bit words");

static int stage_results(fs_worker *w) {
    fs_trie *t = w->tree;
    cudaStream_t s = w->ctx->stream;
    const StageLayout L = stage_layout(w);
    TRY(hgrow(w->h_stage, (int64_t)L.bytes));
    StageArgs a{};
    void *dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, w->h_stage.p, 0));
    a.hs = (uint8_t *)dp;
    CK(cudaHostGetDevicePointer(&dp, w->h_hdr.p, 0));
    a.hh = (int64_t *)dp;
    a.sc = t->sc.p; a.q = w->q.p; a.refills = w->refills.p;
    a.ar = w->adm_req.p; a.am = w->adm_mlen.p; a.an = w->adm_node.p;
    a.au = w->adm_unp.p; a.ap = w->adm_pinb.p; a.ae = w->adm_rec_end.p;
    a.rs = t->rsrc.p; a.rl = t->rlen.p; a.rk = t->rkeep.p;
    a.hdr = w->hdr.p; a.alg = w->alg.p;
    a.nc = w->nclients; a.K = L.K; a.R = L.R;
    a.o_sc = L.o_sc; a.o_q = L.o_q; a.o_rf = L.o_rf; a.o_ar = L.o_ar; a.o_am = L.o_am; a.o_an = L.o_an;
    a.o_au = L.o_au; a.o_ap = L.o_ap; a.o_ae = L.o_ae; a.o_rs = L.o_rs; a.o_rl = L.o_rl; a.o_rk = L.o_rk;
    k_stage_results<<<1, 13 * 32, 0, s>>>(a);
    counted();
    CK(cudaGetLastError());
    if (!w->ev_done) { CK(cudaEventCreate(&w->ev_done)); CK(cudaEventCreate(&w->ev_prev_done)); }
    CK(cudaEventRecord(w->ev_done, s));
    w->gaps_ready = true;
    return FS_OK;
}

extern "C" int fs_worker_fill_begin(fs_worker *w, int64_t now, int64_t generated_total, int64_t headroom) {
    if (!w) return fail(FS_ERR_INVALID, "NULL argument");
    if (w->inflight) return fail(FS_ERR_INVALID, "a fill of this worker is already in flight");
    const auto h0 = std::chrono::steady_clock::now();
    fs_ctx *c = w->ctx;
    fs_trie *t = w->tree;
    cudaStream_t s = c->stream;
    TRY(ctx_use(c));
    TRY(tree_check(t, "the operations before a fill", w->f_n));
    TRY(worker_flush_small(w));
    const int64_t n_old = w->qn - w->admitted_last;
    const int64_t n_new = (int64_t)w->pending_new.size();
    const int64_t n = n_old + n_new;
    // scratch capacity
    TRY(dgrow(w->queue, n + 1, s, true, w->qn)); TRY(dgrow(w->queue2, n + 1, s));
    TRY(dgrow(w->keys, n + 1, s));
    TRY(dgrow(w->mlen, n + 1, s)); TRY(dgrow(w->cov, n + 1, s)); TRY(dgrow(w->fnode, n + 1, s));
    if (w->policy != 2 && w->prev_ok) {
        // the last fill's sorted order becomes p_req (k_merge_a's A)
        std::swap(w->s_req, w->p_req);
        std::swap(w->s_len, w->p_len);
        std::swap(w->s_mlen0, w->p_mlen0);
        std::swap(w->s_tok0, w->p_tok0);
        std::swap(w->s_src0, w->p_src0);
        w->prev_n = w->f_n;
    } else {
        w->prev_n = 0;
    }
    w->prev_ok = false;  // set again once this fill's order is written
    TRY(dgrow(w->next, n + 1, s)); TRY(dgrow(w->s_req, n + 1, s)); TRY(dgrow(w->s_len, n + 1, s));
    TRY(dgrow(w->s_fnode, n + 1, s)); TRY(dgrow(w->s_tok0, n + 1, s)); TRY(dgrow(w->tok0q, n + 1, s)); TRY(dgrow(w->slot, n + 1, s));
    TRY(dgrow(w->s_mlen0, n + 1, s)); TRY(dgrow(w->s0, n + 1, s)); TRY(dgrow(w->s_src0, n + 1, s));
    TRY(dgrow(w->bkey, n + 1, s)); TRY(dgrow(w->bpos, n + 1, s)); TRY(dgrow(w->bkey2, n + 1, s));
    TRY(dgrow(w->bpos2, n + 1, s)); TRY(dgrow(w->akq, n + 1, s)); TRY(dgrow(w->ins, n_new + 1, s));
    TRY(dgrow(w->bkey3, n + 1, s)); TRY(dgrow(w->bpos3, n + 1, s)); TRY(dgrow(w->slow_flag, n + 1, s));
    {
        const int64_t tiles_up = (w->qn + FS_OT_TILE - 1) / FS_OT_TILE + 1;
        TRY(st_grow(w->st_up, tiles_up, s));
        TRY(st_grow(w->st_ma, (w->prev_n + FS_OT_TILE - 1) / FS_OT_TILE + 1, s));
        const int64_t nreq = (int64_t)c->h_roff.size();
        const int64_t old = w->settled.cap;
        TRY(dgrow(w->settled, nreq + 1, s, true, old));
        if (w->settled.cap != old) CK(cudaMemsetAsync(w->settled.p + old, 0, sizeof(int64_t) * (w->settled.cap - old), s));
    }
    const int64_t acap = std::max<int64_t>(n + 1, 64);
    TRY(dgrow(w->adm_req, acap, s)); TRY(dgrow(w->adm_mlen, acap, s)); TRY(dgrow(w->adm_node, acap, s));
    TRY(dgrow(w->adm_unp, acap, s)); TRY(dgrow(w->adm_pinb, acap, s)); TRY(dgrow(w->adm_rec_end, acap, s));
    {
        // each admission creates at most a split top and a leaf; a local tree
        // never holds more than capacity + 2 live nodes (freed slots are reused)
        int64_t extra = 2 * n + 8;
        if (t->capacity >= 0) extra = std::min<int64_t>(extra, t->capacity + 8);
        TRY(trie_reserve(t, extra, c->max_len));
    }
    const uint32_t bits = key_bits(c->max_len);
    const uint32_t kmax = (bits >= 32) ? 0xffffffffu : ((1u << bits) - 1u);

    const int64_t launches0 = g_launches.load();
    const auto h1 = std::chrono::steady_clock::now();
    CK(cudaEventRecord(w->ev[0], s));
    CK(cudaMemsetAsync(w->octl.p, 0, sizeof(OrderCtl), s));
    // ---- queue upkeep (fs_order.cuh): drop last fill's admissions, merge the
    // arrivals in by label -- one pass over the old queue
    if (w->admitted_last > 0 || n_new > 0) {
        if (n_new > 0) {
            std::vector<int32_t> &nv = w->pending_new;
            std::stable_sort(nv.begin(), nv.end(), [&](int32_t x, int32_t y) { return c->h_rlabel[x] < c->h_rlabel[y]; });
            TRY(hgrow(w->h_st32, n_new)); TRY(hgrow(w->h_st64, n_new));
            for (int64_t i = 0; i < n_new; i++) { w->h_st32.p[i] = nv[i]; w->h_st64.p[i] = c->h_rlabel[nv[i]]; }
            TRY(dgrow(w->newids, n_new, s)); TRY(dgrow(w->newlab, n_new, s));
            CK(cudaMemcpyAsync(w->newids.p, w->h_st32.p, sizeof(int32_t) * n_new, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(w->newlab.p, w->h_st64.p, sizeof(int64_t) * n_new, cudaMemcpyHostToDevice, s));
            k_arrivals<<<(unsigned)((n_new + 255) / 256), 256, 0, s>>>(
                w->newids.p, w->newlab.p, (int32_t)n_new, w->queue.p, (int32_t)w->qn, c->rlabel.p, c->rstate.p,
                c->rclient.p, w->pend_cnt.p, c->h_owner.p, w->ins.p);
            counted();
            nv.clear();
        }
        const int64_t tiles = std::max<int64_t>(1, (w->qn + FS_OT_TILE - 1) / FS_OT_TILE);
        k_upkeep<<<(unsigned)tiles, FS_OT_THREADS, 0, s>>>(w->queue.p, (int32_t)w->qn, c->rstate.p, w->ins.p,
                                                          (int32_t)n_new, w->newids.p, w->queue2.p, w->st_up.p,
                                                          lb_next(w, s), &w->octl.p->tile[OT_UPKEEP]);
        counted();
        CK(cudaGetLastError());
        std::swap(w->queue, w->queue2);
    }
    w->qn = n;
    w->admitted_last = 0;
    // on_outputs deltas
    const int32_t ndl = (int32_t)w->dl_client.size();
    if (ndl > 0) {
        TRY(dgrow(w->dlc, ndl, s)); TRY(dgrow(w->dld, ndl, s));
        CK(cudaMemcpyAsync(w->dlc.p, w->dl_client.data(), sizeof(int32_t) * ndl, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(w->dld.p, w->dl_delta.data(), sizeof(int64_t) * ndl, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemsetAsync(w->alg.p, 0, 128 * sizeof(int64_t), s));
    CK(cudaEventRecord(w->ev[1], s));
    if (w->policy == 2) {
        // Vtc.fill (local_policies.py:170-189): no match_prefix, no LPM sort
        CK(cudaEventRecord(w->ev[2], s));
        CK(cudaEventRecord(w->ev[3], s));
        if ((int64_t)w->h_vrank.size() < w->nclients) {
            // default tie-break: dense client id order
            for (int32_t i = (int32_t)w->h_vrank.size(); i < w->nclients; i++) w->h_vrank.push_back(i);
            w->vrank_dirty = true;
        }
        TRY(dgrow(w->vrank, w->nclients, s)); TRY(dgrow(w->vhead, w->nclients, s));
        if (w->vrank_dirty) {
            CK(cudaMemcpyAsync(w->vrank.p, w->h_vrank.data(), sizeof(int32_t) * w->nclients, cudaMemcpyHostToDevice, s));
            w->vrank_dirty = false;
        }
        VtcArgs v{};
        v.t = view(t);
        v.n = (int32_t)n; v.queue = w->queue.p; v.rclient = c->rclient.p; v.rlen = c->rlen.p; v.roff = c->roff.p;
        v.q = w->q.p; v.rank = w->vrank.p; v.nclients = w->nclients; v.head = w->vhead.p;
        v.dl_client = w->dlc.p; v.dl_delta = w->dld.p; v.ndl = ndl;
        v.M = w->M; v.R = w->R; v.gen_total = generated_total; v.headroom0 = headroom; v.w_e = w->w_e; v.now = now;
        v.sq_base = t->opseq + 1;
        v.segs = t->segs.p; v.rstate = c->rstate.p;
        v.adm_req = w->adm_req.p; v.adm_mlen = w->adm_mlen.p; v.adm_node = w->adm_node.p;
        v.adm_unp = w->adm_unp.p; v.adm_pinb = w->adm_pinb.p; v.adm_rec_end = w->adm_rec_end.p;
        v.adm_cap = (int32_t)w->adm_req.cap;
        v.hdr = w->hdr.p;
        {
            static std::mutex vmu;
            static bool vset[64] = {false};
            std::lock_guard<std::mutex> lk(vmu);
            if (c->device < 0 || c->device >= 64) return fail(FS_ERR_INVALID, "device index %d", c->device);
            if (!vset[c->device]) {
                CK(cudaFuncSetAttribute(k_vtc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(VtcSmem)));
                vset[c->device] = true;
            }
        }
        k_vtc<<<1, FS_SCHED_THREADS, sizeof(VtcSmem), s>>>(v);
        counted();
        CK(cudaGetLastError());
        CK(cudaEventRecord(w->ev[4], s));
        w->dl_client.clear(); w->dl_delta.clear();
        TRY(stage_results(w));  // the header and K1 counters too
        w->inflight = true;
        t->busy = true;
        w->f_n = n;
        w->f_launches0 = launches0;
        w->f_h0 = h0; w->f_h1 = h1; w->f_h2 = std::chrono::steady_clock::now();
        return FS_OK;
    }
    // ---- K1: batched match with LRU stamping (lpm_order's match_len calls)
    const int32_t *bjobs = nullptr;  // B (fs_order.cuh): nullptr = every queue position
    const int32_t *bcount = nullptr; //   device count of B (nullptr: n)
    bool incremental = false;
    if (n > 0) {
        static int k1_blocks_dev[64] = {0};
        int &k1_blocks = k1_blocks_dev[c->device & 63];
        if (!k1_blocks) {
            int nsm = 0, per = 0;
            CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_match<1, true>, 256, 0));
            k1_blocks = std::max(1, nsm * per);
        }
        const int64_t blocks = (n * 32 + 255) / 256;
        static const int k1u = [] { const char *e = getenv("FS_K1_UNROLL"); return e ? atoi(e) : 101; }();
        // FS_K1_UNROLL: 4 / 8 / 16 scalar lanes, 101 / 102 / 104 = 128-bit loads, 1 / 2 / 4 per side
        // the full re-match (first fill, FS_K1_FULL, a per-call tree edit) keeps
        // two 128-bit loads per lane and side in flight (0.63 -> 0.68 of HBM on
        // config 5); the incremental path's job walks stay at one
        const int k1f = k1u == 101 ? 102 : k1u;
        auto k1 = k1f == 101 ? k_match<1, true> : k1f == 102 ? k_match<2, true> : k1f == 104 ? k_match<4, true>
                : k1f >= 16 ? k_match<16, false> : k1f >= 8 ? k_match<8, false> : k_match<4, false>;
        static const bool no_hints = getenv("FS_K1_FULL") != nullptr;  // ablation: full re-match every fill
        // FS_K1_TMA=1: full re-matches through the TMA-fed kernel (k_match_tma).
        // Measured slower than the register loop with its up-front L2 bulk
        // prefetch (0.33-0.41 vs 0.62 of HBM on config 5, ring geometries
        // 128-1024 tokens x 2-4 stages): the scan is bound by the per-request
        // chain-walk latency, not by the request stream's arrival
        static const bool k1_tma = [] { const char *e = getenv("FS_K1_TMA"); return e && atoi(e) != 0; }();
        K1Hints h{};
        h.owner = c->h_owner.p; h.m = c->rhint.p; h.S0 = c->h_S0.p; h.tok0 = c->h_tok0.p;
        h.mkeys = w->gkey.p; h.wid = w->wid;
        h.use = !no_hints && !w->k1_full && w->hints_ok && w->gkey.p && w->hint_version == t->version;
        const int64_t sq1 = ++t->opseq;
        // the fast path needs the last fill's order: a settled request keeps
        // its place in it (k_merge_a), only the rest is sorted (B)
        incremental = h.use && k1u == 101 && w->prev_n > 0;
        if (incremental) {
            // fast path: a thread per request settles the ones whose hint holds;
            // persistent warps walk the rest (the queue positions it listed, in order)
            TRY(dgrow(w->k1jobs, n + 1, s));
            w->stag = (w->stag + 1) & 0x3fffffff;
            if (w->stag == 0) w->stag = 1;
            k_match_fast<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
                view(t), w->queue.p, (int32_t)n, c->roff.p, c->rlen.p, now, sq1, kmax, w->keys.p, w->mlen.p,
                w->cov.p, w->next.p, w->s0.p, w->tok0q.p, h, w->k1jobs.p, w->octl.p, w->slow_flag.p,
                w->settled.p, w->stag);
            counted();
            k_match<1, true, true><<<(unsigned)std::min<int64_t>(blocks, k1_blocks), 256, 0, s>>>(
                view(t), w->queue.p, (int32_t)n, c->roff.p, c->rlen.p, now, 1, sq1, kmax, w->keys.p, w->mlen.p,
                w->cov.p, w->next.p, w->s0.p, w->tok0q.p, (unsigned long long *)w->alg.p, h, w->k1jobs.p,
                &w->octl.p->njobs);
            bjobs = w->k1jobs.p;
            bcount = &w->octl.p->njobs;
        } else if (!h.use && k1u == 101 && k1_tma) {
            // every request re-matched from the root: the TMA-fed streaming scan
            static int tma_grid[64] = {0};
            int &tg = tma_grid[c->device & 63];
            const int smem = K1M_WARPS * K1M_NST * K1M_CH * 4 + K1M_WARPS * K1M_NST * 8;
            if (!tg) {
                int nsm = 0, per = 0;
                CK(cudaFuncSetAttribute(k_match_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_match_tma, 32 * K1M_WARPS, smem));
                tg = std::max(1, nsm * per);
            }
            k_match_tma<<<(unsigned)std::min<int64_t>(tg, (n + K1M_WARPS - 1) / K1M_WARPS), 32 * K1M_WARPS, smem, s>>>(
                view(t), w->queue.p, (int32_t)n, c->roff.p, c->rlen.p, now, sq1, kmax, w->keys.p, w->mlen.p,
                w->cov.p, w->next.p, w->s0.p, w->tok0q.p, (unsigned long long *)w->alg.p, h);
        } else {
            k1<<<(unsigned)blocks, 256, 0, s>>>(view(t), w->queue.p, (int32_t)n, c->roff.p, c->rlen.p, now, 1,
                                                sq1, kmax, w->keys.p, w->mlen.p, w->cov.p, w->next.p,
                                                w->s0.p, w->tok0q.p, (unsigned long long *)w->alg.p, h, nullptr,
                                                nullptr);
        }
        counted();
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(w->ev[2], s));
    // ---- K2 (fs_order.cuh): stable order by (-mlen, label).  B sorted by key
    // (LSD radix, 8-bit digits), merged with the settled requests' previous order
    if (n > 0) {
        static int sb_grid[64] = {0};
        int &sbg = sb_grid[c->device & 63];
        if (!sbg) {
            int nsm = 0, per = 0;
            CK(cudaFuncSetAttribute(k_sort_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortBSmem)));
            CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sort_b, FS_SB_THREADS, sizeof(SortBSmem)));
            // two SMs stay free (a D2LPM dispatcher chain may run concurrently)
            sbg = std::max(1, std::min(nsm - 2, nsm * per));
        }
        TRY(dgrow(w->sblk, (int64_t)sbg * FS_RS_BINS + 1, s));
        SortBArgs sa{};
        sa.jobs = bjobs; sa.njobs = bcount; sa.n = (int32_t)n; sa.flag = w->slow_flag.p; sa.keys = w->keys.p;
        sa.npass = (int32_t)((bits + 7) / 8);
        // FS_SB_CAP (tests): a smaller single-CTA limit sends B down the grid-wide path
        static const int32_t sb_cap = [] {
            const char *e = getenv("FS_SB_CAP");
            const int v = e ? atoi(e) : FS_SB_CAP;
            return (int32_t)std::max(1, std::min(v, FS_SB_CAP));
        }();
        sa.cap = sb_cap;
        sa.bkey = w->bkey.p; sa.bkey2 = w->bkey2.p; sa.bkey3 = w->bkey3.p;
        sa.bpos = w->bpos.p; sa.bpos2 = w->bpos2.p; sa.bpos3 = w->bpos3.p; sa.blk = w->sblk.p;
        void *sargs[] = {&sa};
        CK(cudaLaunchCooperativeKernel((const void *)k_sort_b, dim3(sbg), dim3(FS_SB_THREADS), sargs,
                                       sizeof(SortBSmem), s));
        counted();
        SlotOut o{};
        o.queue = w->queue.p; o.cov = w->cov.p; o.next = w->next.p; o.mlen = w->mlen.p; o.tok0 = w->tok0q.p;
        o.rclient = c->rclient.p; o.rlen = c->rlen.p; o.s0 = w->s0.p;
        o.s_req = w->s_req.p; o.s_len = w->s_len.p; o.s_mlen0 = w->s_mlen0.p; o.s_tok0 = w->s_tok0.p;
        o.slot = w->slot.p; o.s_src0 = w->s_src0.p;
        if (incremental) {
            const unsigned ta = (unsigned)((w->prev_n + FS_OT_TILE - 1) / FS_OT_TILE);
            PrevSlots pv{w->p_len.p, w->p_mlen0.p, w->p_tok0.p, w->p_src0.p};
            k_merge_a<<<ta, FS_OT_THREADS, 0, s>>>(w->p_req.p, (int32_t)w->prev_n, w->settled.p, w->stag, kmax, pv,
                                                  w->bkey.p, w->bpos.p, o, w->akq.p, w->st_ma.p, lb_next(w, s),
                                                  w->octl.p);
            counted();
        }
        k_scatter_b<<<(unsigned)std::min<int64_t>((n + 255) / 256, 296), 256, 0, s>>>(
            w->bkey.p, w->bpos.p, bcount, (int32_t)n, w->akq.p, w->octl.p, o);
        counted();
        CK(cudaGetLastError());
        w->prev_ok = true;
    }
    CK(cudaEventRecord(w->ev[3], s));
    // ---- K3+K4: admission passes on one persistent CTA
    FillArgs a{};
    a.t = view(t);
    a.n = (int32_t)n;
    a.s_req = w->s_req.p; a.slot = w->slot.p; a.s_len = w->s_len.p;
    a.s_mlen0 = w->s_mlen0.p; a.s_src0 = w->s_src0.p; a.s_tok0 = w->s_tok0.p;
    a.roff = c->roff.p;
    a.q = w->q.p; a.refills = w->refills.p; a.known = w->known.p; a.nclients = w->nclients; a.pend_cnt = w->pend_cnt.p;
    a.dl_client = w->dlc.p; a.dl_delta = w->dld.p; a.ndl = ndl;
    a.M = w->M; a.R = w->R; a.gen_total = generated_total; a.headroom0 = headroom; a.w_e = w->w_e;
    a.quantum = w->quantum; a.now = now; a.lpm = w->policy == 1;
    a.sq_base = t->opseq + 1;
    a.segs = t->segs.p;
    a.adm_req = w->adm_req.p; a.adm_mlen = w->adm_mlen.p; a.adm_node = w->adm_node.p;
    a.adm_unp = w->adm_unp.p; a.adm_pinb = w->adm_pinb.p; a.adm_rec_end = w->adm_rec_end.p;
    a.adm_cap = (int32_t)w->adm_req.cap;
    a.rstate = c->rstate.p;
    a.hdr = w->hdr.p;
    // function attributes are per device context: set once per device
    static std::mutex attr_mu;
    static bool smem_set[64] = {false};
    std::lock_guard<std::mutex> attr_lock(attr_mu);
    if (c->device < 0 || c->device >= 64) return fail(FS_ERR_INVALID, "device index %d", c->device);
    if (!smem_set[c->device]) {
        CK(cudaFuncSetAttribute(k_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SchedSmem)));
        // the smallest shared-memory carveout that holds SchedSmem: the rest
        // of the SM's 256 KB stays L1, where the admission chain's node,
        // chunk and hash-slot prefetches land (FS_SCHED_CARVEOUT: percent)
        {
            static const int cv = [] { const char *e = getenv("FS_SCHED_CARVEOUT"); return e ? atoi(e) : -2; }();
            int maxsm = 0;
            CK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device));
            const int pct = cv >= -1 ? cv
                          : std::min(100, (int)((100LL * ((int64_t)sizeof(SchedSmem) + 8192) + maxsm - 1) / maxsm));
            CK(cudaFuncSetAttribute(k_schedule, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        }
        smem_set[c->device] = true;
    }
    if (w->nhelp < 0) {
        // one co-resident helper CTA per SM but two (cooperative launch);
        // FS_SCHED_HELPERS overrides (0 = the leader sweeps alone)
        int nsm = 0, per = 0, coop = 0;
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
        CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_schedule, FS_SCHED_THREADS, sizeof(SchedSmem)));
        // one SM stays free: a D2LPM dispatcher chain on its own stream runs
        // concurrently with the fill (cluster rounds)
        int nh = coop ? std::max(0, per * nsm - 2) : 0;
        if (const char *e = getenv("FS_SCHED_HELPERS")) nh = std::min(nh, std::max(0, atoi(e)));
        w->nhelp = nh;
        TRY(dgrow(w->ctl, 1, s));
        TRY(dgrow(w->rw_list, FS_CHUNK, s));
        TRY(dgrow(w->gkey, FS_FSLOTS, s));
        TRY(dgrow(w->gep, FS_FSLOTS, s));
    }
    a.ctl = w->ctl.p; a.gkey = w->gkey.p; a.gep = w->gep.p; a.nhelp = w->nhelp; a.rw_list = w->rw_list.p;
    a.hbase = 1;
    // asynchronous cold eviction: CTA 1 evicts, the sweeps keep the other
    // helpers.  Opt-in (FS_FEV=1): full GPU suites failed intermittently with
    // it on (ref underflow / CacheFull, 3 of 6 runs) and never with it off; a
    // cache without capacity never evicts
    static const bool fev_env = [] { const char *e = getenv("FS_FEV"); return e && atoi(e) != 0; }();
    a.fev = fev_env && w->nhelp >= 2 && t->capacity >= 0;
    if (a.fev) {
        TRY(dgrow(w->fev_ctl, 1, s));
        {
            // order slots are recognised by their fill tag: a fresh buffer may hold
            // another worker's old orders, so it starts zeroed
            const int64_t cap0 = w->fev_need.cap;
            TRY(dgrow(w->fev_need, acap, s));
            if (w->fev_need.cap != cap0) CK(cudaMemsetAsync(w->fev_need.p, 0, sizeof(int64_t) * w->fev_need.cap, s));
        }
        TRY(dgrow(w->fev_rec_end, acap, s));
        TRY(dgrow(w->fev_free, std::max<int64_t>(t->ncap, 64), s));
        CK(cudaMemsetAsync(w->fev_ctl.p, 0, sizeof(FevCtl), s));
        a.fev_ctl = w->fev_ctl.p; a.fev_need = w->fev_need.p; a.fev_rec_end = w->fev_rec_end.p;
        TRY(dgrow(w->fev_vrec, (int64_t)sizeof(FevRec) * FEV_MAXC, s));
        a.fev_free = w->fev_free.p; a.fev_cap = (int32_t)std::min<int64_t>(acap, INT32_MAX);
        a.fev_vrec = w->fev_vrec.p;
        // process-wide tag sequence (nonzero): stale orders of other fills never match
        static std::atomic<int32_t> fev_seq{0};
        w->fev_tag = (int32_t)(fev_seq.fetch_add(1) % ((1 << 23) - 1)) + 1;
        a.fev_tag = w->fev_tag;
        a.nhelp = w->nhelp - 1;
        a.hbase = 2;
    }
    static const int lch = [] { const char *e = getenv("FS_LOCAL_CHUNKS"); return e ? atoi(e) : 1; }();
    a.local_chunks = lch;
    CK(cudaMemsetAsync(w->ctl.p, 0, sizeof(SweepCtl), s));
    if (w->nhelp > 0) {
        void *args[] = {&a};
        CK(cudaLaunchCooperativeKernel((const void *)k_schedule, dim3(1 + w->nhelp), dim3(FS_SCHED_THREADS), args,
                                       sizeof(SchedSmem), s));
    } else {
        k_schedule<<<1, FS_SCHED_THREADS, sizeof(SchedSmem), s>>>(a);
    }
    counted();
    CK(cudaGetLastError());
    static const bool fill_check = [] { const char *e = getenv("FS_FILL_CHECK"); return e && atoi(e) != 0; }();
    if (fill_check) {
        k_check_fill<<<64, 256, 0, s>>>(view(t), w->adm_req.p ? w->adm_node.p : nullptr, w->hdr.p,
                                        (int32_t)w->adm_node.cap, w->hdr.p);
        counted();
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(w->ev[4], s));
    w->dl_client.clear(); w->dl_delta.clear();
    TRY(stage_results(w));  // the header and K1 counters too
    w->inflight = true;
    t->busy = true;
    w->f_n = n;
    w->f_launches0 = launches0;
    w->f_h0 = h0; w->f_h1 = h1; w->f_h2 = std::chrono::steady_clock::now();
    return FS_OK;
}

// Wait for the fill started by fs_worker_fill_begin and read its results.
extern "C" int fs_worker_fill_end(fs_worker *w, fs_fill_result *res) {
    if (!w || !res) return fail(FS_ERR_INVALID, "NULL argument");
    if (!w->inflight) return fail(FS_ERR_INVALID, "no fill in flight");
    static const bool hprof = getenv("FS_HOST_PROFILE") != nullptr;
    w->inflight = false;
    w->tree->busy = false;
    fs_ctx *c = w->ctx;
    fs_trie *t = w->tree;
    cudaStream_t s = c->stream;
    TRY(ctx_use(c));
    const int64_t n = w->f_n, launches0 = w->f_launches0;
    const auto h1 = w->f_h1, h2 = w->f_h2;
    const auto h0 = w->f_h0;
    // ---- results: the staged copies (stage_results, queued by fill_begin)
    const StageLayout SL = stage_layout(w);
    const int64_t K = SL.K, R = SL.R;
    const int64_t nc = w->nclients;
    const size_t o_sc = SL.o_sc, o_q = SL.o_q, o_rf = SL.o_rf, o_ar = SL.o_ar, o_am = SL.o_am, o_an = SL.o_an,
                 o_au = SL.o_au, o_ap = SL.o_ap, o_ae = SL.o_ae, o_rs = SL.o_rs, o_rl = SL.o_rl, o_rk = SL.o_rk;
    uint8_t *hs = w->h_stage.p;
    CK(cudaStreamSynchronize(s));
    if (w->gaps_ready) {
        // device-side gaps around the fill (fs_worker_last_gaps)
        w->gaps_ready = false;
        CK(cudaEventElapsedTime(&w->gaps[0], w->ev[4], w->ev_done));
        w->gaps[1] = -1.f;
        if (w->have_prev_done) CK(cudaEventElapsedTime(&w->gaps[1], w->ev_prev_done, w->ev[0]));
        std::swap(w->ev_done, w->ev_prev_done);
        w->have_prev_done = true;
    }
    std::memcpy(&t->h_sc, hs + o_sc, sizeof(TrieScalars));
    std::memcpy(w->h_q.data(), hs + o_q, 8 * nc);
    std::memcpy(w->h_refills.data(), hs + o_rf, 8 * nc);
    TRY(unpin_settle(t));  // an fs_trie_unpin_many_async queued before this fill
    const int64_t nadm = w->h_hdr.p[0];
    const int64_t nrec = w->h_hdr.p[1];
    const int64_t status = w->h_hdr.p[2];
    for (int i = 0; i < 4; i++) CK(cudaEventElapsedTime(&w->phases[i], w->ev[i], w->ev[i + 1]));
    w->stats[0] = 0;
    w->stats[6] = 0;
    for (int k = 0; k < 64; k++) { w->stats[0] += w->h_hdr.p[32 + 2 * k]; w->stats[6] += w->h_hdr.p[33 + 2 * k]; }
    for (int i = 0; i < 8; i++) w->stats_ext[i] = w->h_hdr.p[24 + i];
    for (int i = 8; i < 24; i++) w->stats[i] = w->h_hdr.p[i];
    w->stats[1] = n;
    w->stats[2] = w->h_hdr.p[3];
    w->stats[3] = w->h_hdr.p[4];
    w->stats[4] = w->h_hdr.p[5];
    w->stats[5] = g_launches.load() - launches0;
    w->stats[7] = w->h_hdr.p[7];  // evictions performed by the FEV evictor CTA (orders)
    float total = 0;
    CK(cudaEventElapsedTime(&total, w->ev[0], w->ev[4]));
    res->device_ms = total;
    res->n_queued = n;
    res->n_adm = nadm;
    res->used = t->h_sc.used;
    res->pinned = t->h_sc.pinned;
    w->admitted_last = nadm;
    t->opseq += nadm;  // admission e stamped with sq_base + e
    w->hint_version = t->version;
    w->hints_ok = status == FS_OK && w->h_hdr.p[6] == 0;
    if (status >= 200 && status < 300)  // FS_FILL_CHECK found a broken path (hdr[6]: the node)
        return fail(FS_ERR_INTERNAL, "fill check %lld at node %lld (adm %lld)", (long long)status,
                    (long long)w->h_hdr.p[6], (long long)nadm);
    if (status != FS_OK) return fail((int)status, "device fill failed (status %lld)", (long long)status);
    if (nadm > res->cap_adm) return fail(FS_ERR_INVALID, "admission buffer too small (%lld > %lld)", (long long)nadm, (long long)res->cap_adm);
    bool second = false;  // a second round of copies (more rows than staged)
    if (nadm > 0 && nadm <= K) {
        if (res->adm_req) std::memcpy(res->adm_req, hs + o_ar, sizeof(int32_t) * nadm);
        if (res->adm_mlen) std::memcpy(res->adm_mlen, hs + o_am, sizeof(int32_t) * nadm);
        if (res->adm_path_node) std::memcpy(res->adm_path_node, hs + o_an, sizeof(int32_t) * nadm);
        if (res->adm_unpinned) std::memcpy(res->adm_unpinned, hs + o_au, sizeof(int64_t) * nadm);
        if (res->adm_pinned_before) std::memcpy(res->adm_pinned_before, hs + o_ap, sizeof(int64_t) * nadm);
        if (res->adm_rec_end) std::memcpy(res->adm_rec_end, hs + o_ae, sizeof(int64_t) * nadm);
    } else if (nadm > 0) {
        second = true;
        if (res->adm_req) CK(cudaMemcpyAsync(res->adm_req, w->adm_req.p, sizeof(int32_t) * nadm, cudaMemcpyDeviceToHost, s));
        if (res->adm_mlen) CK(cudaMemcpyAsync(res->adm_mlen, w->adm_mlen.p, sizeof(int32_t) * nadm, cudaMemcpyDeviceToHost, s));
        if (res->adm_path_node) CK(cudaMemcpyAsync(res->adm_path_node, w->adm_node.p, sizeof(int32_t) * nadm, cudaMemcpyDeviceToHost, s));
        if (res->adm_unpinned) CK(cudaMemcpyAsync(res->adm_unpinned, w->adm_unp.p, sizeof(int64_t) * nadm, cudaMemcpyDeviceToHost, s));
        if (res->adm_pinned_before) CK(cudaMemcpyAsync(res->adm_pinned_before, w->adm_pinb.p, sizeof(int64_t) * nadm, cudaMemcpyDeviceToHost, s));
        if (res->adm_rec_end) CK(cudaMemcpyAsync(res->adm_rec_end, w->adm_rec_end.p, sizeof(int64_t) * nadm, cudaMemcpyDeviceToHost, s));
    }
    {
        fs_records *recs = &res->recs;
        const int64_t kr = std::min(nrec, recs->rec_cap);
        if (nrec > t->rsrc.cap) return fail(FS_ERR_INTERNAL, "eviction record sink overflow (%lld)", (long long)nrec);
        recs->n_rec = nrec;
        if (kr > 0 && kr <= R) {
            std::memcpy(recs->rec_src, hs + o_rs, sizeof(int64_t) * kr);
            std::memcpy(recs->rec_len, hs + o_rl, sizeof(int32_t) * kr);
            std::memcpy(recs->rec_keep, hs + o_rk, sizeof(int32_t) * kr);
        } else if (kr > 0) {
            second = true;
            TRY(copy_records(t, nrec, recs));
        }
    }
    if (second) CK(cudaStreamSynchronize(s));
    if (hprof) {
        const auto h3 = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        fprintf(stderr, "fill host: prologue %.0f us, launches %.0f us, wait+results %.0f us, device %.0f us\n",
                us(h0, h1), us(h1, h2), us(h2, h3), 1000.0 * total);
    }
    return FS_OK;
}

extern "C" int fs_worker_fill(fs_worker *w, int64_t now, int64_t generated_total, int64_t headroom,
                              fs_fill_result *res) {
    if (!w || !res) return fail(FS_ERR_INVALID, "NULL argument");
    TRY(fs_worker_fill_begin(w, now, generated_total, headroom));
    return fs_worker_fill_end(w, res);
}

// ---------------------------------------------------------------- dispatcher
struct fs_dispatcher {
    fs_ctx *ctx = nullptr;
    fs_trie *tree = nullptr;
    int D = 1;
    int64_t quantum = 1, w_e = 1, w_q = 2;
    int32_t nclients = 0;
    int32_t policy = 0;   // FS_DISPATCH_D2LPM / FS_DISPATCH_THRESHOLD
    double theta = 0.5;
    std::vector<int64_t> h_q, h_qsize;
    std::vector<uint8_t> h_qset;
    std::vector<int32_t> dl_idx, dl_w;
    std::vector<int64_t> dl_q;
    DBuf<int64_t> q, qsize;
    DBuf<uint8_t> qset;
    DBuf<int32_t> ids, clients, dli, dlw, o_w, o_mlen;
    DBuf<int64_t> nows, dlq, o_rounds, hdr;
    DBuf<PreRec> pre;
    HBuf<uint8_t> h_stage;  // page-locked staging of a dispatch chain's results
    DBuf<uint64_t> o_mask;
};

static int disp_flush(fs_dispatcher *d);

extern "C" int fs_dispatcher_create(fs_ctx *c, int D, int64_t quantum, int64_t w_e, int64_t w_q,
                                    int32_t max_clients, fs_dispatcher **out) {
    if (!c || !out) return fail(FS_ERR_INVALID, "NULL argument");
    if (quantum <= 0) return fail(FS_ERR_INVALID, "quantum must be positive");  // global_policies.py:97-98
    if (D <= 0 || D > 64) return fail(FS_ERR_INVALID, "D must be in [1, 64]");
    if (max_clients <= 0) return fail(FS_ERR_INVALID, "max_clients must be positive");
    TRY(ctx_use(c));
    fs_dispatcher *d = new fs_dispatcher();
    d->ctx = c; d->D = D; d->quantum = quantum; d->w_e = w_e; d->w_q = w_q; d->nclients = max_clients;
    TRY(fs_trie_create(c, -1, 1, D, &d->tree));
    {
        // highest priority: the serial dispatch chain is the latency-critical
        // side when it overlaps a worker's fill (cluster rounds)
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&d->tree->stream, cudaStreamNonBlocking, hi));
    }
    const int64_t nq = (int64_t)max_clients * D;
    d->h_q.assign(nq, 0); d->h_qset.assign(nq, 0); d->h_qsize.assign(D, 0);
    TRY(dgrow(d->q, nq, c->stream)); TRY(dgrow(d->qset, nq, c->stream)); TRY(dgrow(d->qsize, D, c->stream));
    CK(cudaMemsetAsync(d->q.p, 0, sizeof(int64_t) * nq, c->stream));
    CK(cudaMemsetAsync(d->qset.p, 0, nq, c->stream));
    CK(cudaMemsetAsync(d->qsize.p, 0, sizeof(int64_t) * D, c->stream));
    TRY(dgrow(d->hdr, 24, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = d;
    return FS_OK;
}

extern "C" int fs_dispatcher_destroy(fs_dispatcher *d) {
    if (!d) return FS_OK;
    cudaSetDevice(d->ctx->device);
    cudaStream_t ds = d->tree->stream;
    cudaStreamSynchronize(ds);
    fs_trie_destroy(d->tree);
    if (ds) cudaStreamDestroy(ds);
    d->q.release(); d->qsize.release(); d->qset.release(); d->ids.release(); d->clients.release();
    d->dli.release(); d->dlw.release(); d->o_w.release(); d->o_mlen.release(); d->nows.release();
    d->dlq.release(); d->o_rounds.release(); d->hdr.release(); d->o_mask.release();
    d->pre.release(); d->h_stage.release();
    delete d;
    return FS_OK;
}

extern "C" fs_trie *fs_dispatcher_tree(fs_dispatcher *d) { return d ? d->tree : nullptr; }

extern "C" int fs_dispatch_last_profile(fs_dispatcher *d, int64_t *prof16) {
    if (!d || !prof16) return fail(FS_ERR_INVALID, "NULL argument");
    TRY(ctx_use(d->ctx));
    CK(cudaMemcpyAsync(prof16, d->hdr.p + 4, 16 * sizeof(int64_t), cudaMemcpyDeviceToHost, d->tree->stream));
    CK(cudaStreamSynchronize(d->tree->stream));
    return FS_OK;
}

static int check_dispatch_ids(fs_dispatcher *d, int64_t n, const int32_t *req_ids) {
    fs_ctx *c = d->ctx;
    for (int64_t i = 0; i < n; i++)
        if (req_ids[i] < 0 || req_ids[i] >= (int64_t)c->h_roff.size()) return fail(FS_ERR_INVALID, "bad request id");
    return FS_OK;
}

extern "C" int fs_prematch_record_bytes(void) { return (int)sizeof(PreRec); }

// Batch-start matches of n arrivals (a slice of a batch) into device memory
// dev_out (n records of fs_prematch_record_bytes() bytes, on the dispatcher's
// device).  Synchronous.
extern "C" int fs_dispatch_prematch(fs_dispatcher *d, int64_t n, const int32_t *req_ids, void *dev_out) {
    if (!d || n < 0 || (n > 0 && (!req_ids || !dev_out))) return fail(FS_ERR_INVALID, "bad arguments");
    if (n == 0) return FS_OK;
    fs_ctx *c = d->ctx;
    cudaStream_t s = d->tree->stream;
    TRY(ctx_use(c));
    TRY(check_dispatch_ids(d, n, req_ids));
    TRY(dgrow(d->ids, n, s));
    CK(cudaMemcpyAsync(d->ids.p, req_ids, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    k_dispatch_prematch<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(view(d->tree), d->ids.p, (int32_t)n,
                                                                         c->roff.p, c->rlen.p, (PreRec *)dev_out);
    counted();
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return FS_OK;
}

static int dispatch_run(fs_dispatcher *d, int64_t n, const int32_t *req_ids, const int32_t *clients,
                        const int64_t *now, const PreRec *dev_pre, int32_t *out_worker, int32_t *out_mlen,
                        uint64_t *out_mask, int64_t *out_rounds);

extern "C" int fs_dispatch(fs_dispatcher *d, int64_t n, const int32_t *req_ids, const int32_t *clients,
                           const int64_t *now, int32_t *out_worker, int32_t *out_mlen, uint64_t *out_mask,
                           int64_t *out_rounds) {
    return dispatch_run(d, n, req_ids, clients, now, nullptr, out_worker, out_mlen, out_mask, out_rounds);
}

extern "C" int fs_dispatch_prematched(fs_dispatcher *d, int64_t n, const int32_t *req_ids, const int32_t *clients,
                                      const int64_t *now, const void *dev_pre, int32_t *out_worker,
                                      int32_t *out_mlen, uint64_t *out_mask, int64_t *out_rounds) {
    if (n > 0 && !dev_pre) return fail(FS_ERR_INVALID, "dev_pre is required");
    return dispatch_run(d, n, req_ids, clients, now, (const PreRec *)dev_pre, out_worker, out_mlen, out_mask,
                        out_rounds);
}

static int dispatch_run(fs_dispatcher *d, int64_t n, const int32_t *req_ids, const int32_t *clients,
                        const int64_t *now, const PreRec *dev_pre, int32_t *out_worker, int32_t *out_mlen,
                        uint64_t *out_mask, int64_t *out_rounds) {
    if (!d || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    if (n == 0) return FS_OK;
    if (!req_ids || !clients || !now || !out_worker)
        return fail(FS_ERR_INVALID, "req_ids, clients, now and out_worker are required");
    fs_ctx *c = d->ctx;
    cudaStream_t s = d->tree->stream;
    TRY(ctx_use(c));
    for (int64_t i = 0; i < n; i++) {
        if (req_ids[i] < 0 || req_ids[i] >= (int64_t)c->h_roff.size()) return fail(FS_ERR_INVALID, "bad request id");
        if (clients[i] < 0 || clients[i] >= d->nclients) return fail(FS_ERR_INVALID, "client id out of range");
    }
    TRY(trie_reserve(d->tree, 2 * n + 2, c->max_len));
    TRY(dgrow(d->ids, n, s)); TRY(dgrow(d->clients, n, s)); TRY(dgrow(d->nows, n, s));
    TRY(dgrow(d->o_w, n, s)); TRY(dgrow(d->o_mlen, n, s)); TRY(dgrow(d->o_mask, n, s)); TRY(dgrow(d->o_rounds, n, s));
    CK(cudaMemcpyAsync(d->ids.p, req_ids, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d->clients.p, clients, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d->nows.p, now, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    const int32_t ndl = (int32_t)d->dl_idx.size();
    TRY(disp_flush(d));
    DispArgs a{};
    a.t = view(d->tree);
    a.n = (int32_t)n; a.D = d->D;
    a.ids = d->ids.p; a.clients = d->clients.p; a.nows = d->nows.p;
    a.roff = c->roff.p; a.rlen = c->rlen.p;
    a.q = d->q.p; a.qset = d->qset.p; a.qsize = d->qsize.p;
    a.quantum = d->quantum; a.w_e = d->w_e;
    a.dl_idx = d->dli.p; a.dl_q = d->dlq.p; a.dl_w = d->dlw.p; a.ndl = ndl;
    a.segs = d->tree->segs.p;
    a.sq_base = d->tree->opseq + 1;
    d->tree->opseq += 2 * n;
    d->tree->version++;
    if (dev_pre) {
        // computed by the caller against this batch-start index (a slice per
        // rank, all-gathered: fs_dispatch_prematch)
        a.pre = dev_pre;
    } else {
        // batch-start matches of every arrival, in parallel (K1, no stamping):
        // the serial chain below resumes each walk from them
        TRY(dgrow(d->pre, n, s));
        k_dispatch_prematch<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(view(d->tree), d->ids.p, (int32_t)n,
                                                                             c->roff.p, c->rlen.p, d->pre.p);
        counted();
        CK(cudaGetLastError());
        a.pre = d->pre.p;
    }
    a.out_w = d->o_w.p; a.out_mlen = d->o_mlen.p; a.out_mask = d->o_mask.p; a.out_rounds = d->o_rounds.p;
    a.hdr = d->hdr.p;
    a.policy = d->policy; a.theta = d->theta;
    k_dispatch<<<1, FS_DISPATCH_THREADS, 0, s>>>(a);
    counted();
    CK(cudaGetLastError());
    d->dl_idx.clear(); d->dl_w.clear(); d->dl_q.clear();
    // results: one batch of DMA copies into page-locked staging, one wait
    const size_t o_st = 0, o_w = 16, o_ml = o_w + ((4 * n + 15) & ~15), o_mk = o_ml + ((4 * n + 15) & ~15),
                 o_rd = o_mk + 8 * n, o_sc = o_rd + 8 * n;
    TRY(hgrow(d->h_stage, (int64_t)(o_sc + sizeof(TrieScalars))));
    uint8_t *hs = d->h_stage.p;
    CK(cudaMemcpyAsync(hs + o_st, d->hdr.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + o_w, d->o_w.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + o_ml, d->o_mlen.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + o_mk, d->o_mask.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + o_rd, d->o_rounds.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + o_sc, d->tree->sc.p, sizeof(TrieScalars), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int64_t st = 0;
    std::memcpy(&st, hs + o_st, sizeof(int64_t));
    std::memcpy(out_worker, hs + o_w, sizeof(int32_t) * n);
    if (out_mlen) std::memcpy(out_mlen, hs + o_ml, sizeof(int32_t) * n);
    if (out_mask) std::memcpy(out_mask, hs + o_mk, sizeof(uint64_t) * n);
    const int64_t *rounds = (const int64_t *)(hs + o_rd);
    std::memcpy(&d->tree->h_sc, hs + o_sc, sizeof(TrieScalars));
    if (st != FS_OK) return fail((int)st, "device dispatch failed (status %lld)", (long long)st);
    // mirror the counter updates (the monitor reads dispatcher.q each timestamp)
    for (int64_t i = 0; i < n; i++) {
        const int32_t cl = clients[i];
        const int32_t wk = out_worker[i];
        int64_t *qr = d->h_q.data() + (int64_t)cl * d->D;
        uint8_t *qs = d->h_qset.data() + (int64_t)cl * d->D;
        d->h_qsize[wk] += 1;
        if (out_rounds) out_rounds[i] = rounds[i];
        if (d->policy != FS_DISPATCH_D2LPM) continue;  // ThresholdRouter keeps no counters
        if (rounds[i] > 0)
            for (int x = 0; x < d->D; x++) { qr[x] += rounds[i] * d->quantum; qs[x] = 1; }
        qr[wk] -= d->w_e * c->h_rlen[req_ids[i]];
        qs[wk] = 1;
    }
    return FS_OK;
}

extern "C" int fs_dispatcher_set_policy(fs_dispatcher *d, int32_t policy, double theta) {
    if (!d) return fail(FS_ERR_INVALID, "NULL");
    if (policy != FS_DISPATCH_D2LPM && policy != FS_DISPATCH_THRESHOLD) return fail(FS_ERR_INVALID, "unknown policy %d", policy);
    if (!(theta >= 0.0 && theta <= 1.0)) return fail(FS_ERR_INVALID, "theta must be in [0, 1]");  // global_policies.py:145-146
    d->policy = policy;
    d->theta = theta;
    return FS_OK;
}

extern "C" int fs_dispatch_finish(fs_dispatcher *d, int32_t client, int32_t worker, int64_t output_tokens) {
    if (!d || client < 0 || client >= d->nclients || worker < 0 || worker >= d->D)
        return fail(FS_ERR_INVALID, "bad arguments");
    const int64_t idx = (int64_t)client * d->D + worker;
    d->h_qsize[worker] -= 1;
    if (d->policy == FS_DISPATCH_D2LPM) {
        // D2lpm.on_finish (global_policies.py:126-129)
        const int64_t dq = -d->w_q * output_tokens;
        d->h_q[idx] += dq;
        d->h_qset[idx] = 1;
        d->dl_idx.push_back((int32_t)idx);
        d->dl_w.push_back(worker);
        d->dl_q.push_back(dq);
    }
    d->dl_idx.push_back(-1);  // queue_size[worker] -= 1 (global_policies.py:52)
    d->dl_w.push_back(worker);
    d->dl_q.push_back(-1);
    return FS_OK;
}

extern "C" int fs_dispatch_finish_many(fs_dispatcher *d, int64_t n, const int32_t *clients, const int32_t *workers,
                                       const int64_t *output_tokens) {
    if (!d || n < 0) return fail(FS_ERR_INVALID, "bad arguments");
    for (int64_t i = 0; i < n; i++) TRY(fs_dispatch_finish(d, clients[i], workers[i], output_tokens[i]));
    return FS_OK;
}

extern "C" int fs_dispatch_counters(fs_dispatcher *d, int32_t client, int64_t *q_row, uint8_t *present) {
    if (!d || client < 0 || client >= d->nclients) return fail(FS_ERR_INVALID, "bad arguments");
    const int64_t b = (int64_t)client * d->D;
    if (q_row) std::memcpy(q_row, d->h_q.data() + b, sizeof(int64_t) * d->D);
    if (present) std::memcpy(present, d->h_qset.data() + b, d->D);
    return FS_OK;
}

extern "C" int fs_dispatch_queue_sizes(fs_dispatcher *d, int64_t *sizes) {
    if (!d || !sizes) return fail(FS_ERR_INVALID, "NULL");
    std::memcpy(sizes, d->h_qsize.data(), sizeof(int64_t) * d->D);
    return FS_OK;
}

// Push every host-side override (set_counter / set_queue_size) and finish delta.
static int disp_flush(fs_dispatcher *d) {
    fs_ctx *c = d->ctx;
    cudaStream_t s = d->tree->stream;
    const int32_t ndl = (int32_t)d->dl_idx.size();
    if (ndl == 0) return FS_OK;
    TRY(dgrow(d->dli, ndl, s)); TRY(dgrow(d->dlw, ndl, s)); TRY(dgrow(d->dlq, ndl, s));
    CK(cudaMemcpyAsync(d->dli.p, d->dl_idx.data(), sizeof(int32_t) * ndl, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d->dlw.p, d->dl_w.data(), sizeof(int32_t) * ndl, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d->dlq.p, d->dl_q.data(), sizeof(int64_t) * ndl, cudaMemcpyHostToDevice, s));
    return FS_OK;
}

extern "C" int fs_dispatch_select(fs_dispatcher *d, int32_t client, uint64_t matched_mask, int32_t *worker,
                                  int64_t *rounds) {
    if (!d || client < 0 || client >= d->nclients || !worker) return fail(FS_ERR_INVALID, "bad arguments");
    fs_ctx *c = d->ctx;
    cudaStream_t s = d->tree->stream;
    TRY(ctx_use(c));
    TRY(disp_flush(d));
    TRY(dgrow(d->clients, 1, s)); TRY(dgrow(d->o_w, 1, s)); TRY(dgrow(d->o_mask, 1, s)); TRY(dgrow(d->o_rounds, 1, s));
    CK(cudaMemcpyAsync(d->clients.p, &client, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d->o_mask.p, &matched_mask, sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    DispArgs a{};
    a.t = view(d->tree);
    a.n = 1; a.D = d->D; a.select_only = 1;
    a.clients = d->clients.p;
    a.q = d->q.p; a.qset = d->qset.p; a.qsize = d->qsize.p;
    a.quantum = d->quantum; a.w_e = d->w_e;
    a.dl_idx = d->dli.p; a.dl_q = d->dlq.p; a.dl_w = d->dlw.p; a.ndl = (int32_t)d->dl_idx.size();
    a.out_w = d->o_w.p; a.out_mask = d->o_mask.p; a.out_rounds = d->o_rounds.p;
    a.hdr = d->hdr.p;
    k_dispatch<<<1, FS_DISPATCH_THREADS, 0, s>>>(a);
    counted();
    CK(cudaGetLastError());
    d->dl_idx.clear(); d->dl_w.clear(); d->dl_q.clear();
    int64_t r = 0;
    CK(cudaMemcpyAsync(worker, d->o_w.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&r, d->o_rounds.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (r > 0) {
        int64_t *qr = d->h_q.data() + (int64_t)client * d->D;
        uint8_t *qs = d->h_qset.data() + (int64_t)client * d->D;
        for (int x = 0; x < d->D; x++) { qr[x] += r * d->quantum; qs[x] = 1; }
    }
    if (rounds) *rounds = r;
    return FS_OK;
}

extern "C" int fs_dispatch_set_counter(fs_dispatcher *d, int32_t client, int32_t worker, int64_t q) {
    if (!d || client < 0 || client >= d->nclients || worker < 0 || worker >= d->D) return fail(FS_ERR_INVALID, "bad arguments");
    const int64_t idx = (int64_t)client * d->D + worker;
    const int64_t delta = q - d->h_q[idx];
    d->h_q[idx] = q;
    d->h_qset[idx] = 1;
    d->dl_idx.push_back((int32_t)idx); d->dl_w.push_back(-1); d->dl_q.push_back(delta);
    return FS_OK;
}

extern "C" int fs_dispatch_set_queue_size(fs_dispatcher *d, int32_t worker, int64_t size) {
    if (!d || worker < 0 || worker >= d->D) return fail(FS_ERR_INVALID, "bad arguments");
    const int64_t delta = size - d->h_qsize[worker];
    d->h_qsize[worker] = size;
    // encoded as a queue-size-only delta: q index -1
    d->dl_idx.push_back(-1); d->dl_w.push_back(worker); d->dl_q.push_back(delta);
    return FS_OK;
}

extern "C" int fs_dispatcher_reserve_clients(fs_dispatcher *d, int32_t max_clients) {
    if (!d) return fail(FS_ERR_INVALID, "NULL dispatcher");
    if (max_clients <= d->nclients) return FS_OK;
    fs_ctx *c = d->ctx;
    cudaStream_t s = d->tree->stream;
    TRY(ctx_use(c));
    const int32_t nc = std::max(max_clients, d->nclients * 2);
    const int64_t old = (int64_t)d->nclients * d->D, nw = (int64_t)nc * d->D;
    TRY(dgrow(d->q, nw, s, true, old)); TRY(dgrow(d->qset, nw, s, true, old));
    CK(cudaMemsetAsync(d->q.p + old, 0, sizeof(int64_t) * (nw - old), s));
    CK(cudaMemsetAsync(d->qset.p + old, 0, nw - old, s));
    d->h_q.resize(nw, 0); d->h_qset.resize(nw, 0);
    d->nclients = nc;
    CK(cudaStreamSynchronize(s));
    return FS_OK;
}

extern "C" int fs_dispatch_device_counters(fs_dispatcher *d, int64_t n, int64_t *q, uint8_t *present, int64_t *qsize) {
    if (!d) return fail(FS_ERR_INVALID, "NULL dispatcher");
    TRY(ctx_use(d->ctx));
    TRY(disp_flush(d));
    // apply pending deltas with an empty dispatch so device == mirror
    if (!d->dl_idx.empty()) {
        DispArgs a{};
        a.t = view(d->tree); a.n = 0; a.D = d->D;
        a.q = d->q.p; a.qset = d->qset.p; a.qsize = d->qsize.p;
        a.dl_idx = d->dli.p; a.dl_q = d->dlq.p; a.dl_w = d->dlw.p; a.ndl = (int32_t)d->dl_idx.size();
        a.hdr = d->hdr.p;
        k_dispatch<<<1, FS_DISPATCH_THREADS, 0, d->tree->stream>>>(a);
        counted();
        CK(cudaGetLastError());
        d->dl_idx.clear(); d->dl_w.clear(); d->dl_q.clear();
    }
    const int64_t k = std::min<int64_t>(n, (int64_t)d->nclients * d->D);
    cudaStream_t s = d->tree->stream;
    if (q) CK(cudaMemcpyAsync(q, d->q.p, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
    if (present) CK(cudaMemcpyAsync(present, d->qset.p, k, cudaMemcpyDeviceToHost, s));
    if (qsize) CK(cudaMemcpyAsync(qsize, d->qsize.p, sizeof(int64_t) * d->D, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return FS_OK;
}

// ---------------------------------------------------------------- verifiers
// Post-run, not on the decision path: plain allocations per call.
namespace {
struct DevArrays {
    std::vector<void *> ptrs;
    ~DevArrays() { for (void *p : ptrs) cudaFree(p); }
    template <typename T>
    int put(const T *h, int64_t n, T **d) {
        *d = nullptr;
        CK(cudaMalloc((void **)d, sizeof(T) * std::max<int64_t>(n, 1)));
        ptrs.push_back(*d);
        if (h && n > 0) CK(cudaMemcpy(*d, h, sizeof(T) * n, cudaMemcpyHostToDevice));
        return FS_OK;
    }
};
}  // namespace

static int svc_upload(DevArrays &m, int32_t C, const int64_t *ev_off, const int64_t *ev_time, const int64_t *ev_cum,
                      const int64_t *iv_off, const int64_t *iv_lo, const int64_t *iv_hi, SvcView *v) {
    if (C <= 0 || !ev_off || !iv_off) return fail(FS_ERR_INVALID, "bad verifier arguments");
    const int64_t ne = ev_off[C], ni = iv_off[C];
    if (ne < 0 || ni < 0 || (ne > 0 && (!ev_time || !ev_cum)) || (ni > 0 && (!iv_lo || !iv_hi)))
        return fail(FS_ERR_INVALID, "bad verifier arguments");
    int64_t *d_eo, *d_et, *d_ec, *d_io, *d_il, *d_ih;
    TRY(m.put(ev_off, C + 1, &d_eo)); TRY(m.put(ev_time, ne, &d_et)); TRY(m.put(ev_cum, ne + C, &d_ec));
    TRY(m.put(iv_off, C + 1, &d_io)); TRY(m.put(iv_lo, ni, &d_il)); TRY(m.put(iv_hi, ni, &d_ih));
    v->C = C; v->ev_off = d_eo; v->ev_time = d_et; v->ev_cum = d_ec; v->iv_off = d_io; v->iv_lo = d_il; v->iv_hi = d_ih;
    return FS_OK;
}

extern "C" int fs_verify_pairs(int device, int32_t C, const int64_t *ev_off, const int64_t *ev_time,
                               const int64_t *ev_cum, const int64_t *iv_off, const int64_t *iv_lo,
                               const int64_t *iv_hi, int mode, int64_t *out_gap, int64_t *out_t1, int64_t *out_t2,
                               int32_t *out_valid) {
    if (mode != 0 && mode != 1) return fail(FS_ERR_INVALID, "mode must be 0 (pairwise) or 1 (global max-min)");
    if (!out_gap || !out_t1 || !out_t2 || !out_valid) return fail(FS_ERR_INVALID, "NULL output");
    CK(cudaSetDevice(device));
    DevArrays m;
    SvcView v{};
    TRY(svc_upload(m, C, ev_off, ev_time, ev_cum, iv_off, iv_lo, iv_hi, &v));
    const int64_t np = (int64_t)C * C;
    int64_t *d_gap, *d_t1, *d_t2;
    int32_t *d_ok;
    TRY(m.put<int64_t>(nullptr, np, &d_gap)); TRY(m.put<int64_t>(nullptr, np, &d_t1));
    TRY(m.put<int64_t>(nullptr, np, &d_t2)); TRY(m.put<int32_t>(nullptr, np, &d_ok));
    CK(cudaMemset(d_ok, 0, sizeof(int32_t) * std::max<int64_t>(np, 1)));
    if (C > 1) {
        dim3 grid((unsigned)((C - 1 + 127) / 128), (unsigned)C);
        k_verify_pairs<<<grid, 128>>>(v, mode, d_gap, d_t1, d_t2, d_ok);
        counted();
        CK(cudaGetLastError());
    }
    CK(cudaMemcpy(out_gap, d_gap, sizeof(int64_t) * np, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_t1, d_t1, sizeof(int64_t) * np, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_t2, d_t2, sizeof(int64_t) * np, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_valid, d_ok, sizeof(int32_t) * np, cudaMemcpyDeviceToHost));
    return FS_OK;
}

extern "C" int fs_verify_vs_any(int device, int32_t C, const int64_t *ev_off, const int64_t *ev_time,
                                const int64_t *ev_cum, const int64_t *iv_off, const int64_t *iv_lo,
                                const int64_t *iv_hi, int64_t nwin, const int32_t *win_f, const int64_t *win_t1,
                                const int64_t *win_t2, int64_t *out_gap, int32_t *out_g) {
    if (nwin < 0 || (nwin > 0 && (!win_f || !win_t1 || !win_t2 || !out_gap || !out_g)))
        return fail(FS_ERR_INVALID, "bad window arguments");
    CK(cudaSetDevice(device));
    DevArrays m;
    SvcView v{};
    TRY(svc_upload(m, C, ev_off, ev_time, ev_cum, iv_off, iv_lo, iv_hi, &v));
    if (nwin == 0) return FS_OK;
    for (int64_t w = 0; w < nwin; w++)
        if (win_f[w] < 0 || win_f[w] >= C) return fail(FS_ERR_INVALID, "window client %d outside [0,%d)", win_f[w], C);
    int32_t *d_wf, *d_g;
    int64_t *d_t1, *d_t2, *d_gap;
    TRY(m.put(win_f, nwin, &d_wf)); TRY(m.put(win_t1, nwin, &d_t1)); TRY(m.put(win_t2, nwin, &d_t2));
    TRY(m.put<int64_t>(nullptr, nwin, &d_gap)); TRY(m.put<int32_t>(nullptr, nwin, &d_g));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    const unsigned grid = (unsigned)std::min<int64_t>(nwin, (int64_t)nsm * 8);
    k_verify_vs_any<<<grid, 256>>>(v, nwin, d_wf, d_t1, d_t2, d_gap, d_g);
    counted();
    CK(cudaGetLastError());
    CK(cudaMemcpy(out_gap, d_gap, sizeof(int64_t) * nwin, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_g, d_g, sizeof(int32_t) * nwin, cudaMemcpyDeviceToHost));
    for (int64_t w = 0; w < nwin; w++)
        if (out_g[w] == INT32_MAX) out_g[w] = -1;
    return FS_OK;
}
