// fs_materialize.cuh -- the reference's token universe on the device.
//
// Trace.materialize (requests.py:134-161) builds every request as
//     prefix ++ expand_tokens(f"sfx:{rid}", suffix_len)
// where a prefix is expand_tokens(shared_prefix_id, prefix_len) or, for
// "req:<rid>", a prefix of an earlier request.  expand_tokens
// (requests.py:95-102) concatenates _token_block(namespace, b) for b = 0, 1, ...
// and _token_block (requests.py:89-92) is
//     sha256(f"{namespace}#{b}".encode()) -> eight big-endian 32-bit words % 2^31.
// The host resolves every request into segments, each one a leading slice
// expand_tokens(ns, len) of one namespace (parent-chain prefixes are prefixes
// of the parent's segments), and k_expand writes the segments straight into
// the token arena: one warp per segment, one lane per 8-token block.
#pragma once
#include <stdint.h>

__constant__ uint32_t c_sha_k[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

struct ExpandArgs {
    int32_t *arena;
    const int64_t *seg_dst;   // arena offset of the segment's first token
    const int32_t *seg_len;   // tokens in the segment (a leading slice of the namespace)
    const int32_t *seg_ns;    // namespace index
    const uint8_t *ns_bytes;  // UTF-8 namespace strings, back to back
    const int64_t *ns_off;
    const int32_t *ns_len;
    int64_t nseg;
};

__device__ __forceinline__ uint32_t fs_rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void sha256_compress(uint32_t h[8], const uint32_t m[16]) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; i++) w[i] = m[i];
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
    for (int i = 0; i < 64; i++) {
        uint32_t wi;
        if (i < 16) {
            wi = w[i];
        } else {
            const uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            const uint32_t s0 = fs_rotr(w15, 7) ^ fs_rotr(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = fs_rotr(w2, 17) ^ fs_rotr(w2, 19) ^ (w2 >> 10);
            wi = w[i & 15] + s0 + w[(i - 7) & 15] + s1;
            w[i & 15] = wi;
        }
        const uint32_t S1 = fs_rotr(e, 6) ^ fs_rotr(e, 11) ^ fs_rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = hh + S1 + ch + c_sha_k[i] + wi;
        const uint32_t S0 = fs_rotr(a, 2) ^ fs_rotr(a, 13) ^ fs_rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t t2 = S0 + mj;
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// _token_block(ns, block): sha256 of ns ++ "#" ++ decimal(block), words & 0x7fffffff.
__device__ __forceinline__ void token_block(const uint8_t *ns, int n, uint32_t block, uint32_t out[8]) {
    char dig[10];
    int nd = 0;
    {
        uint32_t v = block;
        char tmp[10];
        do { tmp[nd++] = (char)('0' + v % 10); v /= 10; } while (v);
        for (int i = 0; i < nd; i++) dig[i] = tmp[nd - 1 - i];
    }
    const int mlen = n + 1 + nd;                 // message bytes
    const int nchunks = (mlen + 8) / 64 + 1;     // + 0x80 + 64-bit length
    const uint64_t bits = (uint64_t)mlen * 8;
    uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                     0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    for (int c = 0; c < nchunks; c++) {
        uint32_t m[16];
#pragma unroll
        for (int wd = 0; wd < 16; wd++) {
            uint32_t word = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int k = c * 64 + wd * 4 + j;
                uint32_t byte;
                if (k < n) byte = __ldg(ns + k);
                else if (k == n) byte = '#';
                else if (k < mlen) byte = (uint8_t)dig[k - n - 1];
                else if (k == mlen) byte = 0x80;
                else byte = 0;
                word = (word << 8) | byte;
            }
            m[wd] = word;
        }
        if (c == nchunks - 1) {
            m[14] = (uint32_t)(bits >> 32);
            m[15] = (uint32_t)bits;
        }
        sha256_compress(h, m);
    }
#pragma unroll
    for (int i = 0; i < 8; i++) out[i] = h[i] & 0x7fffffffu;
}

// One warp per segment (grid-stride), lane l computes blocks l, l+32, ...
__global__ void __launch_bounds__(256) k_expand(ExpandArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = warp; s < a.nseg; s += nwarps) {
        const int32_t len = a.seg_len[s];
        const int64_t dst = a.seg_dst[s];
        const int32_t ns = a.seg_ns[s];
        const uint8_t *nsb = a.ns_bytes + a.ns_off[ns];
        const int nlen = a.ns_len[ns];
        const int32_t nblk = (len + 7) >> 3;
        for (int32_t b = lane; b < nblk; b += 32) {
            uint32_t t[8];
            token_block(nsb, nlen, (uint32_t)b, t);
            const int64_t o = dst + 8LL * b;
            const int32_t cnt = min(8, len - 8 * b);
            if (cnt == 8 && (o & 3) == 0) {
                int4 *p = reinterpret_cast<int4 *>(a.arena + o);
                p[0] = make_int4((int)t[0], (int)t[1], (int)t[2], (int)t[3]);
                p[1] = make_int4((int)t[4], (int)t[5], (int)t[6], (int)t[7]);
            } else {
                for (int j = 0; j < cnt; j++) a.arena[o + j] = (int32_t)t[j];
            }
        }
    }
}
