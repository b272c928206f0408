"""Post-run service-gap verifiers on the GPU.

Drop-in replacements for three verifiers of the reference's metrics module
(pkg/src/fairsched/metrics.py), same signatures, same BoundReport:

  verify_service_bound_pairwise           metrics.py:148-174  (|W_f - W_g|)
  verify_service_bound_vs_nonbacklogged   metrics.py:177-197  (W_g - W_f)
  verify_global_max_min                   metrics.py:200-237  (max - min)

The reference walks every client pair (or client), every co-backlogged
interval and every window of a 4-division grid in Python -- O(C^2) pairs of
O(log n) service queries at 1000 clients, O(C^3) for the max-min check.  Here
the host builds flat arrays once (per-client service prefix sums, backlogged
intervals, both vectorised with numpy) and the windows are evaluated by
k_verify_pairs / k_verify_vs_any (csrc/fs_verify.cuh); the host then takes
the first maximum in the reference's enumeration order, so `measured` and the
window named in `detail` are the reference's.  plugin.install(verifiers=True)
rebinds the reference's functions (runner.verify_run resolves them through
the module at call time, runner.py:383-440).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import P32, P64, call


@dataclass
class _Report:
    """Field-compatible stand-in for fairsched.metrics.BoundReport (used when
    the reference package is not importable)."""
    theorem: str
    measured: float
    bound: float
    applicable: bool = True
    guaranteed: bool = True
    detail: str = ""


def _report(*args, **kw):
    try:
        from fairsched.metrics import BoundReport
    except ImportError:
        BoundReport = _Report
    return BoundReport(*args, **kw)


def _clients(lifecycle) -> list:
    """_clients_of (metrics.py:144-145)."""
    return sorted({rec["client"] for rec in lifecycle.values() if "client" in rec})


def backlogs(lifecycle, clients, run_end):
    """backlogged_intervals (metrics.py:103-115) of every client, vectorised:
    per client, +1 at each arrival and -1 at its admission (run_end if never
    admitted), deltas summed per time; an interval opens where the running
    count becomes positive and closes where it returns to zero.  Returns
    (iv_off, iv_lo, iv_hi) with client c's intervals at [iv_off[c], iv_off[c+1])."""
    idx = {c: i for i, c in enumerate(clients)}
    cl, arr, adm = [], [], []
    for rec in lifecycle.values():
        c = rec.get("client")
        if c not in idx or "arrival_time" not in rec:
            continue
        a = rec["arrival_time"]
        d = rec.get("admit_time", run_end)
        if d > a:
            cl.append(idx[c]); arr.append(a); adm.append(d)
    nc = len(clients)
    if not cl:
        return np.zeros(nc + 1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)
    cl = np.asarray(cl, np.int64)
    t = np.concatenate([np.asarray(arr, np.int64), np.asarray(adm, np.int64)])
    c2 = np.concatenate([cl, cl])
    d = np.concatenate([np.ones(len(cl), np.int64), -np.ones(len(cl), np.int64)])
    order = np.lexsort((t, c2))
    t, c2, d = t[order], c2[order], d[order]
    # sum the deltas of equal (client, time)
    first = np.ones(len(t), bool)
    first[1:] = (t[1:] != t[:-1]) | (c2[1:] != c2[:-1])
    grp = np.cumsum(first) - 1
    ut, uc = t[first], c2[first]
    ud = np.zeros(len(ut), np.int64)
    np.add.at(ud, grp, d)
    cnt = np.cumsum(ud)  # every client's deltas sum to zero: segments restart at 0
    prev = np.concatenate([[0], cnt[:-1]])
    newc = np.ones(len(ut), bool)
    newc[1:] = uc[1:] != uc[:-1]
    prev[newc] = 0
    opens = (cnt > 0) & (prev <= 0)
    closes = (cnt <= 0) & (prev > 0)
    lo, hi, owner = ut[opens], ut[closes], uc[opens]
    if len(lo) != len(hi) or np.any(uc[closes] != owner):
        raise AssertionError("pending count never returned to zero")
    off = np.zeros(nc + 1, np.int64)
    np.add.at(off, owner + 1, 1)
    return np.cumsum(off), lo.astype(np.int64), hi.astype(np.int64)


def service_arrays(service, clients):
    """Per client: event times and prefix sums of units (accounting.py:35-86)."""
    times, cums, off = [], [], [0]
    for c in clients:
        evs = service._events.get(c, [])
        tt = np.fromiter((e.time for e in evs), np.int64, len(evs))
        uu = np.fromiter((e.units for e in evs), np.int64, len(evs))
        times.append(tt)
        cums.append(np.concatenate([[0], np.cumsum(uu)]).astype(np.int64))
        off.append(off[-1] + len(evs))
    ev_time = np.concatenate(times) if times else np.zeros(0, np.int64)
    ev_cum = np.concatenate(cums) if cums else np.zeros(1, np.int64)
    return np.asarray(off, np.int64), np.ascontiguousarray(ev_time, np.int64), np.ascontiguousarray(ev_cum, np.int64)


class ServiceView:
    """The flat arrays the verifier kernels read, built once per run."""

    def __init__(self, service, lifecycle, run_end, device: int = 0):
        self.clients = _clients(lifecycle)
        self.device = device
        self.ev_off, self.ev_time, self.ev_cum = service_arrays(service, self.clients)
        self.iv_off, self.iv_lo, self.iv_hi = backlogs(lifecycle, self.clients, run_end)

    def _svc_args(self):
        def p(a):
            return a.ctypes.data_as(P64)
        return (self.device, len(self.clients), p(self.ev_off), p(self.ev_time), p(self.ev_cum), p(self.iv_off),
                p(self.iv_lo), p(self.iv_hi))

    def pairs(self, mode: int):
        n = len(self.clients)
        gap = np.zeros(n * n, np.int64)
        t1 = np.zeros(n * n, np.int64)
        t2 = np.zeros(n * n, np.int64)
        ok = np.zeros(n * n, np.int32)
        call("fs_verify_pairs", *self._svc_args(), mode, gap.ctypes.data_as(P64), t1.ctypes.data_as(P64),
             t2.ctypes.data_as(P64), ok.ctypes.data_as(P32))
        return gap, t1, t2, ok

    def intervals(self, c):
        a, b = self.iv_off[c], self.iv_off[c + 1]
        return list(zip(self.iv_lo[a:b].tolist(), self.iv_hi[a:b].tolist()))

    def grid_windows(self):
        """window_grid (metrics.py:91-100) of every backlogged interval, in
        (client, interval, grid) order: (f, t1, t2) arrays."""
        lo, hi = self.iv_lo, self.iv_hi
        nc = len(self.clients)
        f = np.repeat(np.arange(nc, dtype=np.int32), np.diff(self.iv_off))
        b = lo[:, None] + (hi - lo)[:, None] * np.arange(5, dtype=np.int64)[None, :] // 4
        ii, jj = np.triu_indices(5, k=1)  # (0,1), (0,2), ... (3,4): the reference's loop order
        w1, w2 = b[:, ii], b[:, jj]
        keep = w1 < w2
        return (np.ascontiguousarray(np.broadcast_to(f[:, None], w1.shape)[keep], np.int32),
                np.ascontiguousarray(w1[keep]), np.ascontiguousarray(w2[keep]))

    def vs_any(self):
        wf, w1, w2 = self.grid_windows()
        n = len(wf)
        gap = np.zeros(n, np.int64)
        g = np.zeros(n, np.int32)
        call("fs_verify_vs_any", *self._svc_args(), n, wf.ctypes.data_as(P32), w1.ctypes.data_as(P64),
             w2.ctypes.data_as(P64), gap.ctypes.data_as(P64), g.ctypes.data_as(P32))
        return wf, w1, w2, gap, g


def _first_max(values, mask):
    idx = np.flatnonzero(mask)
    if len(idx) == 0:
        return None
    return int(idx[int(np.argmax(values[idx]))])  # argmax: first maximum


def verify_service_bound_pairwise(service, lifecycle, bound, run_end, theorem, guaranteed=True, device=0):
    """metrics.verify_service_bound_pairwise on the GPU."""
    v = ServiceView(service, lifecycle, run_end, device)
    gap, t1, t2, ok = v.pairs(0)
    k = _first_max(gap, ok != 0)
    if k is None:
        return _report(theorem, 0.0, bound, applicable=False, guaranteed=guaranteed,
                       detail="no common backlogged window")
    n = len(v.clients)
    f, g = divmod(k, n)
    return _report(theorem, int(gap[k]), bound, guaranteed=guaranteed,
                   detail=f"{v.clients[f]} vs {v.clients[g]} on [{int(t1[k])},{int(t2[k])})")


def verify_service_bound_vs_nonbacklogged(service, lifecycle, bound, run_end, theorem, guaranteed=True,
                                          device=0):
    """metrics.verify_service_bound_vs_nonbacklogged on the GPU."""
    v = ServiceView(service, lifecycle, run_end, device)
    wf, w1, w2, gap, g = v.vs_any()
    k = _first_max(gap, g >= 0)
    if k is None:
        return _report(theorem, 0.0, bound, applicable=False, guaranteed=guaranteed, detail="no backlogged window")
    return _report(theorem, int(gap[k]), bound, guaranteed=guaranteed,
                   detail=f"{v.clients[int(g[k])]} over backlogged {v.clients[int(wf[k])]} "
                          f"on [{int(w1[k])},{int(w2[k])})")


def verify_global_max_min(service, lifecycle, bound, run_end, theorem, guaranteed=True, device=0):
    """metrics.verify_global_max_min on the GPU."""
    v = ServiceView(service, lifecycle, run_end, device)
    gap, t1, t2, ok = v.pairs(1)
    k = _first_max(gap, ok != 0)
    if k is None:
        return _report(theorem, 0.0, bound, applicable=False, guaranteed=guaranteed,
                       detail="fewer than 2 clients ever co-backlogged")
    a, b = int(t1[k]), int(t2[k])
    members = [c for i, c in enumerate(v.clients) if any(lo <= a and b <= hi for lo, hi in v.intervals(i))]
    return _report(theorem, int(gap[k]), bound, guaranteed=guaranteed, detail=f"clients {members} on [{a},{b})")


REBOUND = ("verify_service_bound_pairwise", "verify_service_bound_vs_nonbacklogged", "verify_global_max_min")
