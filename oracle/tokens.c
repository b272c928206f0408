/* TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's token universe
 * for large samples (the hashlib restatement in materialize.py is exact but
 * ~1 us per block in Python).
 *
 *   _token_block(ns, b)   requests.py:89-92   sha256(f"{ns}#{b}") -> 8 big-endian words % 2^31
 *   expand_tokens(ns, n)  requests.py:95-102  blocks 0, 1, ... truncated to n
 *
 * or_expand_segments writes requests given as namespace segments (the layout of
 * paper_2501_14312_b200.trace.Segments) back to back into a flat int32 array.
 * Pinned by tests/test_materialize.py against tests/golden/tokens.json.  Used by
 * bench.py's CPU leg / reference arm to build their samples without the CUDA
 * library.  SHA-256 per FIPS 180-4.  Threads: one per online core (pthreads).
 */
#include <pthread.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

static const uint32_t K[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

static inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void compress(uint32_t h[8], const uint8_t blk[64]) {
    uint32_t w[64];
    for (int i = 0; i < 16; i++)
        w[i] = ((uint32_t)blk[4 * i] << 24) | ((uint32_t)blk[4 * i + 1] << 16) | ((uint32_t)blk[4 * i + 2] << 8) |
               (uint32_t)blk[4 * i + 3];
    for (int i = 16; i < 64; i++) {
        uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
        uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; i++) {
        uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[i] + w[i];
        uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

/* one _token_block: msg = ns ++ "#" ++ decimal(block) */
static void token_block(const uint8_t *ns, int64_t n, uint64_t block, int32_t out[8]) {
    char dig[24];
    int nd = 0;
    char tmp[24];
    uint64_t v = block;
    do { tmp[nd++] = (char)('0' + v % 10); v /= 10; } while (v);
    for (int i = 0; i < nd; i++) dig[i] = tmp[nd - 1 - i];
    const int64_t mlen = n + 1 + nd;
    uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                     0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    const int64_t nchunks = (mlen + 8) / 64 + 1;
    uint8_t blk[64];
    for (int64_t c = 0; c < nchunks; c++) {
        for (int j = 0; j < 64; j++) {
            const int64_t k = c * 64 + j;
            uint8_t byte;
            if (k < n) byte = ns[k];
            else if (k == n) byte = '#';
            else if (k < mlen) byte = (uint8_t)dig[k - n - 1];
            else if (k == mlen) byte = 0x80;
            else byte = 0;
            blk[j] = byte;
        }
        if (c == nchunks - 1) {
            const uint64_t bits = (uint64_t)mlen * 8;
            for (int j = 0; j < 8; j++) blk[56 + j] = (uint8_t)(bits >> (56 - 8 * j));
        }
        compress(h, blk);
    }
    for (int i = 0; i < 8; i++) out[i] = (int32_t)(h[i] & 0x7fffffffu);
}

/* expand_tokens(ns, len) into dst */
static void expand(const uint8_t *ns, int64_t n, int32_t len, int32_t *dst) {
    int32_t t[8];
    for (int64_t b = 0; 8 * b < len; b++) {
        token_block(ns, n, (uint64_t)b, t);
        const int32_t cnt = len - 8 * (int32_t)b < 8 ? len - 8 * (int32_t)b : 8;
        memcpy(dst + 8 * b, t, sizeof(int32_t) * (size_t)cnt);
    }
}

struct job {
    int64_t lo, hi;
    const int64_t *seg_first, *ns_off, *offsets;
    const int32_t *seg_ns, *seg_len, *ns_len;
    const uint8_t *ns_bytes;
    int32_t *out;
};

static void *run_job(void *p) {
    const struct job *j = (const struct job *)p;
    for (int64_t i = j->lo; i < j->hi; i++) {
        int64_t o = j->offsets[i];
        for (int64_t s = j->seg_first[i]; s < j->seg_first[i + 1]; s++) {
            const int32_t k = j->seg_ns[s];
            expand(j->ns_bytes + j->ns_off[k], j->ns_len[k], j->seg_len[s], j->out + o);
            o += j->seg_len[s];
        }
    }
    return 0;
}

/* n requests; request i = segments [seg_first[i], seg_first[i+1]); writes the
 * tokens back to back into out (offsets[i] = start of request i, offsets[n] =
 * total), split over the host's cores with pthreads. */
int64_t or_expand_segments(int64_t n, const int64_t *seg_first, const int32_t *seg_ns, const int32_t *seg_len,
                           const uint8_t *ns_bytes, const int64_t *ns_off, const int32_t *ns_len, int32_t *out,
                           int64_t *offsets) {
    int64_t tot = 0;
    for (int64_t i = 0; i < n; i++) {
        offsets[i] = tot;
        for (int64_t s = seg_first[i]; s < seg_first[i + 1]; s++) tot += seg_len[s];
    }
    offsets[n] = tot;
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if (nt > 64) nt = 64;
    if (n < 64) nt = 1;
    pthread_t th[64];
    struct job jobs[64];
    for (long t = 0; t < nt; t++) {
        jobs[t].lo = n * t / nt;
        jobs[t].hi = n * (t + 1) / nt;
        jobs[t].seg_first = seg_first; jobs[t].ns_off = ns_off; jobs[t].offsets = offsets;
        jobs[t].seg_ns = seg_ns; jobs[t].seg_len = seg_len; jobs[t].ns_len = ns_len;
        jobs[t].ns_bytes = ns_bytes; jobs[t].out = out;
    }
    for (long t = 1; t < nt; t++) pthread_create(&th[t], 0, run_job, &jobs[t]);
    run_job(&jobs[0]);
    for (long t = 1; t < nt; t++) pthread_join(th[t], 0);
    return tot;
}
