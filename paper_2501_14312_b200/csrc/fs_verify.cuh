// fs_verify.cuh -- the post-run service-gap verifiers of metrics.py on the
// device.  Every window the reference enumerates is enumerated
// here in the same order; the per-pair (or per-window) worst values come back
// to the host, which takes the first maximum in enumeration order, so the
// report (measured value and the window named in `detail`) is the reference's.
//
// Inputs, per client c in sorted-name order (_clients_of, metrics.py:144-145):
//   events  ev_time[ev_off[c] .. ev_off[c+1])  time-ordered service events,
//           ev_cum[ev_off[c] + c ..]           their prefix sums (one extra 0
//                                              per client, so client c's
//                                              cumulative array has n_c + 1
//                                              entries starting at
//                                              ev_off[c] + c)
//   backlog iv_lo/iv_hi[iv_off[c] .. iv_off[c+1])  backlogged_intervals
//           (metrics.py:103-115), sorted and disjoint
#pragma once
#include <cstdint>

struct SvcView {
    int32_t C;
    const int64_t *ev_off, *ev_time, *ev_cum;
    const int64_t *iv_off, *iv_lo, *iv_hi;
};

// ServiceLog.service_in_interval (accounting.py:76-86): units of the events
// with t1 <= time < t2 (two bisect_left over the client's times).
__device__ __forceinline__ int64_t svc_in(const SvcView &v, int32_t c, int64_t t1, int64_t t2) {
    const int64_t b = v.ev_off[c], n = v.ev_off[c + 1] - b;
    const int64_t *tm = v.ev_time + b;
    const int64_t *cum = v.ev_cum + b + c;
    int64_t lo = 0, hi = n;
    while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (tm[m] < t1) lo = m + 1; else hi = m; }
    const int64_t i1 = lo;
    hi = n;
    while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (tm[m] < t2) lo = m + 1; else hi = m; }
    return cum[lo] - cum[i1];
}

// Is [t1, t2) inside one of client c's backlogged intervals?
__device__ __forceinline__ bool svc_backlogged(const SvcView &v, int32_t c, int64_t t1, int64_t t2) {
    const int64_t b = v.iv_off[c], n = v.iv_off[c + 1] - b;
    int64_t lo = 0, hi = n;  // last interval with lo <= t1
    while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (v.iv_lo[b + m] <= t1) lo = m + 1; else hi = m; }
    return lo > 0 && t2 <= v.iv_hi[b + lo - 1];
}

// window_grid(lo, hi, 4) (metrics.py:91-100): window w of the (i < j) bound
// pairs, in order, skipping equal bounds.  Calls fn(t1, t2) per window.
template <typename Fn>
__device__ __forceinline__ void window_grid4(int64_t lo, int64_t hi, Fn fn) {
    int64_t b[5];
#pragma unroll
    for (int i = 0; i < 5; i++) b[i] = lo + (hi - lo) * i / 4;  // non-negative: floor division
#pragma unroll
    for (int i = 0; i < 5; i++)
#pragma unroll
        for (int j = i + 1; j < 5; j++)
            if (b[i] < b[j]) fn(b[i], b[j]);
}

// Pairwise verifiers, one thread per client pair (f = blockIdx.y, g > f):
//   mode 0  verify_service_bound_pairwise (metrics.py:148-174): |W_f - W_g|
//   mode 1  verify_global_max_min (metrics.py:200-237): max - min of W over
//           every client backlogged through the window
// over the windows of intersect_intervals(backlogs f, g) (metrics.py:56-68).
// Out (index f*C + g): the pair's first worst gap and its window; valid = 0
// when the pair has no window.
__global__ void k_verify_pairs(SvcView v, int mode, int64_t *__restrict__ out_gap, int64_t *__restrict__ out_t1,
                               int64_t *__restrict__ out_t2, int32_t *__restrict__ out_valid) {
    const int32_t f = blockIdx.y;
    const int32_t g = f + 1 + (int32_t)(blockIdx.x * blockDim.x + threadIdx.x);
    if (g >= v.C) return;
    int64_t best = -1, bt1 = 0, bt2 = 0;
    int32_t any = 0;
    int64_t i = v.iv_off[f], ie = v.iv_off[f + 1];
    int64_t j = v.iv_off[g], je = v.iv_off[g + 1];
    while (i < ie && j < je) {
        const int64_t lo = max(v.iv_lo[i], v.iv_lo[j]);
        const int64_t hi = min(v.iv_hi[i], v.iv_hi[j]);
        if (lo < hi) {
            window_grid4(lo, hi, [&](int64_t t1, int64_t t2) {
                int64_t gap;
                if (mode == 0) {
                    const int64_t d = svc_in(v, f, t1, t2) - svc_in(v, g, t1, t2);
                    gap = d < 0 ? -d : d;
                } else {
                    int64_t mx = INT64_MIN, mn = INT64_MAX;
                    int32_t members = 0;
                    for (int32_t c = 0; c < v.C; c++) {
                        if (!svc_backlogged(v, c, t1, t2)) continue;
                        const int64_t w = svc_in(v, c, t1, t2);
                        mx = max(mx, w);
                        mn = min(mn, w);
                        members++;
                    }
                    if (members < 2) return;
                    gap = mx - mn;
                }
                if (!any || gap > best) { best = gap; bt1 = t1; bt2 = t2; any = 1; }
            });
        }
        if (v.iv_hi[i] <= v.iv_hi[j]) i++; else j++;
    }
    const int64_t o = (int64_t)f * v.C + g;
    out_gap[o] = best;
    out_t1[o] = bt1;
    out_t2[o] = bt2;
    out_valid[o] = any;
}

// verify_service_bound_vs_nonbacklogged (metrics.py:177-197): one block per
// window (f, t1, t2) of f's backlog grid (enumerated by the host in the
// reference's order); the worst W_g - W_f over g != f, first g on ties.
__global__ void __launch_bounds__(256) k_verify_vs_any(SvcView v, int64_t nwin, const int32_t *__restrict__ wf,
                                                       const int64_t *__restrict__ wt1,
                                                       const int64_t *__restrict__ wt2,
                                                       int64_t *__restrict__ out_gap, int32_t *__restrict__ out_g) {
    __shared__ int64_t sg[256];
    __shared__ int32_t sc[256];
    for (int64_t w = blockIdx.x; w < nwin; w += gridDim.x) {
        const int32_t f = wf[w];
        const int64_t t1 = wt1[w], t2 = wt2[w];
        const int64_t base = svc_in(v, f, t1, t2);
        int64_t best = INT64_MIN;
        int32_t bg = INT32_MAX;
        for (int32_t g = threadIdx.x; g < v.C; g += blockDim.x) {
            if (g == f) continue;
            const int64_t gap = svc_in(v, g, t1, t2) - base;
            if (gap > best) { best = gap; bg = g; }  // g ascending per thread: first g kept
        }
        sg[threadIdx.x] = best;
        sc[threadIdx.x] = bg;
        __syncthreads();
        for (int s = 128; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                const int64_t b2 = sg[threadIdx.x + s];
                const int32_t c2 = sc[threadIdx.x + s];
                if (b2 > sg[threadIdx.x] || (b2 == sg[threadIdx.x] && c2 < sc[threadIdx.x])) {
                    sg[threadIdx.x] = b2;
                    sc[threadIdx.x] = c2;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) { out_gap[w] = sg[0]; out_g[w] = sc[0]; }
        __syncthreads();
    }
}
