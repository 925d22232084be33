"""Regenerate tests/golden/* from the reference itself (oracle/_ref).

Run here (where /root/reference exists and oracle/_ref was built):
    python tests/golden/gen_golden.py [--big] [--only NAME]

Writes
  digests.json   ciphertext_digest of run_he_mul_bench(seed=7, reps=1)
                 (bench.cpp:49-124) per config, plus the reference's stage
                 times of that single run (informational only)
  s_bench.npz    the S config's seed-7 inputs (c1, c2, evk) and he_mul output
  small_random.npz  random-input he_mul cases at logN=10 over two levels
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import Reference, random_poly  # noqa: E402

CONFIGS = {
    "S": (30, 4, 13),
    "logN13_logQ300": (30, 10, 13),
    "logN14_logQ300": (30, 10, 0),
    "logN15_logQ600": (30, 20, 0),
    "M": (30, 40, 0),
    "X": (30, 80, 0),
}


def main() -> None:
    big = "--big" in sys.argv
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    ref = Reference()
    out = HERE / "digests.json"
    data = json.loads(out.read_text()) if out.exists() else {}
    for name, cfg in CONFIGS.items():
        if (name in ("M", "X") and not big) or (only and name != only):
            continue
        t = time.time()
        dig, ms = ref.run_bench(*cfg, seed=7, reps=1)
        log_n, n, log_q_max = ref.make_params(*cfg)
        data[name] = {"params": list(cfg), "log_n": log_n, "log_q_max": log_q_max,
                      "out_log_q": log_q_max - cfg[0], "digest": f"{dig:016x}",
                      "ref_stage_ms_1thread": ms}
        print(name, f"{dig:016x}", f"{time.time() - t:.1f}s", flush=True)
        out.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    if only:
        return
    # S inputs / outputs
    cfg = CONFIGS["S"]
    inp = ref.bench_inputs(*cfg, seed=7)
    q = inp["log_q_max"]
    st, oa, ob = ref.he_mul(*cfg, q, inp["c1"], inp["c2"], inp["evk"])
    assert st == 0
    np.savez_compressed(HERE / "s_bench.npz", c1ax=inp["c1"][0], c1bx=inp["c1"][1],
                        c2ax=inp["c2"][0], c2bx=inp["c2"][1], evkax=inp["evk"][0],
                        evkbx=inp["evk"][1], outax=oa, outbx=ob, log_q=q)
    # random inputs at logN=10, two levels (arbitrary residues are valid
    # he_mul inputs: SURVEY §8(d) "throughput inputs")
    rng = np.random.default_rng(2024)
    cases = {}
    cfg = (30, 6, 10)
    log_n, n, qmax = ref.make_params(*cfg)
    evk = (random_poly(rng, n, 2 * qmax), random_poly(rng, n, 2 * qmax))
    cases["evkax"], cases["evkbx"] = evk
    for lvl, log_q in enumerate((qmax, qmax - 60)):
        c1 = (random_poly(rng, n, log_q), random_poly(rng, n, log_q))
        c2 = (random_poly(rng, n, log_q), random_poly(rng, n, log_q))
        st, oa, ob = ref.he_mul(*cfg, log_q, c1, c2, evk)
        assert st == 0
        for k, v in (("c1ax", c1[0]), ("c1bx", c1[1]), ("c2ax", c2[0]), ("c2bx", c2[1]),
                     ("outax", oa), ("outbx", ob)):
            cases[f"{k}_{lvl}"] = v
        cases[f"log_q_{lvl}"] = np.array(log_q)
    np.savez_compressed(HERE / "small_random.npz", params=np.array(cfg), **cases)
    print("fixtures written")


if __name__ == "__main__":
    main()
