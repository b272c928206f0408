"""Record the reference's token universe (run in the build container only).

    python tests/golden/make_golden_tokens.py

Imports `fairsched` from /root/reference/pkg/src and writes tokens.json:

* blocks  -- _token_block(ns, b) (requests.py:89-92) for namespaces of every
  SHA-256 padding regime (short, 55/56/63/64-byte boundaries, multi-chunk,
  non-ASCII) and block numbers with 1..7 decimal digits;
* expand  -- expand_tokens(ns, n) (requests.py:95-102) for n = 0..41 and 1000;
* traces  -- generate_trace(...) (workload.py:140-159) for flat and tree
  programs (req:<rid> parent chains), stored as TraceRecords with the
  sha256 of every materialized request (Trace.materialize, requests.py:134-161).

The fixture is committed; /root/reference does not exist on the GPU box.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fairsched.requests import SystemParams, _token_block, expand_tokens  # noqa: E402
from fairsched.workload import ClientProfile, generate_trace  # noqa: E402

NAMESPACES = [
    "", "a", "sfx:r00000001", "pfx:steady", "pfx:flood:3", "req-like:x",
    "x" * 53, "x" * 54, "x" * 55, "x" * 56, "x" * 62, "x" * 63, "x" * 64, "x" * 65, "y" * 119, "z" * 130,
    "sfx:dépôt-κλειδί-鍵", "emoji:\U0001F600" * 5,
]
BLOCKS = [0, 1, 7, 9, 10, 99, 100, 12345, 999999, 1000000, 4194303]


def tok_digest(toks) -> str:
    return hashlib.sha256(json.dumps(list(toks), separators=(",", ":")).encode()).hexdigest()


def main():
    blocks = [[ns, b, list(_token_block(ns, b))] for ns in NAMESPACES for b in BLOCKS]
    expand = [[ns, n, list(expand_tokens(ns, n))] for ns in NAMESPACES[:6] for n in list(range(42)) + [1000]]
    params = SystemParams(L_input=2048, L_output=64, M=8192, D=1)
    traces = []
    for name, profiles in [
        ("flat", [ClientProfile(name="a", rate=40, prefix_len=100, suffix_len=13),
                  ClientProfile(name="b", rate=25, cv=3.0, prefix_len=0, suffix_len=31, prefix_scope="program")]),
        ("tree", [ClientProfile(name="t", rate=10, program="tree", branches=3, depth=3, prefix_len=77, suffix_len=9),
                  ClientProfile(name="u", rate=8, program="tree", branches=2, depth=4, prefix_len=200, suffix_len=40,
                                prefix_scope="program"),
                  ClientProfile(name="f", rate=30, prefix_len=64, suffix_len=5, misbehavior="S2")]),
    ]:
        tr = generate_trace(profiles, params, seed=11, horizon=400_000)
        reqs, outs = tr.materialize()
        traces.append({"name": name,
                       "records": [json.loads(r.to_json()) for r in tr.records],
                       "lens": [len(r.input_tokens) for r in reqs],
                       "digests": [tok_digest(r.input_tokens) for r in reqs],
                       "first_tokens": [list(r.input_tokens[:3]) for r in reqs]})
    with open(os.path.join(HERE, "tokens.json"), "w") as fh:
        json.dump({"blocks": blocks, "expand": expand, "traces": traces}, fh, separators=(",", ":"))
    print("wrote tokens.json:", len(blocks), "blocks,", len(expand), "expansions,",
          [(t["name"], len(t["records"])) for t in traces])


if __name__ == "__main__":
    main()
