"""Random service logs and lifecycles for the verifier tests (the shapes
fairsched.runner produces: ServiceLog events per client, lifecycle records
with client / arrival_time / admit_time)."""
import random


def random_case(fs, seed, n_clients, n_req, horizon=5000, p_unadmitted=0.1, same_time=0.2):
    from fairsched.accounting import CostWeights, ServiceLog

    rng = random.Random(seed)
    names = [f"c{rng.randrange(10 ** 6):06d}" for _ in range(n_clients)]
    life = {}
    events = []
    for k in range(n_req):
        c = rng.choice(names)
        arr = rng.randrange(horizon)
        if rng.random() < same_time and life:
            arr = rng.choice(list(life.values()))["arrival_time"]  # shared timestamps
        rec = {"rid": f"r{k}", "client": c, "arrival_time": arr}
        if rng.random() >= p_unadmitted:
            adm = arr + rng.choice([0, rng.randrange(1, horizon // 4)])
            rec["admit_time"] = adm
            events.append((adm, c, "extend", rng.randrange(1, 300), rng.randrange(300, 600)))
            for s in range(rng.randrange(0, 4)):
                events.append((adm + 1 + s * rng.randrange(1, 50), c, "output", rng.randrange(1, 20), 0))
        life[rec["rid"]] = rec
    if rng.random() < 0.5:
        life["norec"] = {"rid": "norec"}  # records without a client are skipped
    svc = ServiceLog(CostWeights(1, 2))
    for t, c, kind, a, b in sorted(events, key=lambda e: e[0]):
        if kind == "extend":
            svc.add_extend(t, c, a, b)
        else:
            svc.add_output(t, c, a)
    run_end = horizon + horizon // 2
    return svc, life, run_end
