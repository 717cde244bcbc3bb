"""Per-call Engine API latency probe (single update / extract / delete /
bulk_update d=32) at a few heap sizes: host wall time per blocking call.
Run under ncu with --metrics gpu__time_duration.sum to split wall time into
kernel time and launch + synchronize overhead."""
import argparse
import time

import numpy as np

import paper_1908_09378_b200 as P


def run(n_pre, n_calls, dev=0, idle_us=200):
    eng = P.Engine(P.EngineConfig(d=32, debug_assertions=False, key_universe=1 << 21, device=dev))
    eng.set_persistent(idle_us)
    rng = np.random.default_rng(3)
    keys = rng.permutation(1 << 21).astype(np.uint32)
    # prefill with 32-wide batches
    pr = np.arange(32, dtype=np.uint64) + 5000
    for i in range(n_pre // 32):
        eng.bulk_update(values=np.sort(keys[32 * i:32 * (i + 1)]), priorities=pr)
    base = n_pre
    out = {"prefill": n_pre}
    t0 = time.perf_counter()
    for i in range(n_calls):
        eng.update((int(keys[base + i]), int(1000 + i)))
    out["update_us"] = (time.perf_counter() - t0) * 1e6 / n_calls
    base += n_calls
    batches = [np.sort(keys[base + 32 * i:base + 32 * (i + 1)]) for i in range(n_calls)]
    t0 = time.perf_counter()
    for b in batches:
        eng.bulk_update(values=b, priorities=pr)
    out["bulk_update_d32_us"] = (time.perf_counter() - t0) * 1e6 / n_calls
    t0 = time.perf_counter()
    for _ in range(n_calls):
        eng.extract_min()
    out["extract_min_us"] = (time.perf_counter() - t0) * 1e6 / n_calls
    t0 = time.perf_counter()
    for i in range(n_calls):
        eng.delete_value(int(keys[n_pre + n_calls // 2 + i]))
    out["delete_us"] = (time.perf_counter() - t0) * 1e6 / n_calls
    pp = eng.persist_profile()
    if pp["requests"]:
        out["profile"] = pp
    eng.close()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=1000)
    ap.add_argument("--pre", default="0,100000")
    a = ap.parse_args()
    run(0, 64)  # module load / first launches
    import torch
    x = torch.zeros(1, device="cuda")
    for _ in range(100):
        x += 1
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        x += 1
        torch.cuda.synchronize()
    print("floor: torch 1-element kernel + synchronize", (time.perf_counter() - t0) * 1e6 / 2000, "us", flush=True)
    for idle in (200, 0):
        for n_pre in [int(x) for x in a.pre.split(",")]:
            print("api idle_us=%d" % idle, run(n_pre, a.calls, idle_us=idle), flush=True)
