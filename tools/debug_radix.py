"""Debug helper: replay one golden radix trace on the GPU DeviceRadixTree and
print the first dump difference."""
import sys
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from replay import load_golden, canon_dump
from paper_2501_14312_b200.radix import DeviceRadixTree, CacheFull
from paper_2501_14312_b200.runtime import get_runtime

idx = int(sys.argv[1])
tr = load_golden("radix_traces.json")["traces"][idx]
cap = tr.get("capacity")
t = DeviceRadixTree(capacity=cap if tr["kind"] == "local" else None, track_workers=tr["kind"] != "local",
                    n_workers=max(tr.get("n_workers", 1), 1), runtime=get_runtime())
pins = {}
for k, op in enumerate(tr["ops"]):
    toks = tuple(op["tokens"])
    kind = op["op"]
    try:
        if kind == "insert":
            t.insert(toks, now=op["now"], worker=op.get("worker"))
        elif kind == "match":
            t.match_prefix(toks, now=op["now"], update_access=op["update"])
        elif kind == "probe":
            t.probe(toks)
        elif kind == "admit":
            m, h = t.admit(toks, now=op["now"])
            pins[op["pin_id"]] = h
        elif kind == "unpin":
            t.unpin(pins.pop(op["pin_id"]))
        elif kind == "evict":
            t.evict_lru(op["needed"])
        elif kind == "lmw":
            t.longest_match_workers(toks, now=op["now"])
        elif kind == "notify":
            t.evict_notify(toks, op["worker"], op["keep_len"], op["notice_time"])
    except CacheFull:
        pass
    got = canon_dump(t.dump())
    if got != op["dump"]:
        print("op", k, op["op"], toks, "now", op.get("now"))
        print("prev ops:", [(o["op"], o["tokens"], o.get("now")) for o in tr["ops"][max(0, k - 4):k]])
        exp = op["dump"]
        for i in range(max(len(got), len(exp))):
            g = got[i] if i < len(got) else None
            e = exp[i] if i < len(exp) else None
            flag = "  " if g == e else "!!"
            print(flag, "got", g, "| exp", e)
        break
else:
    print("trace", idx, "OK")
