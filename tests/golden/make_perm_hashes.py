"""Reference permutations at the BASELINE sizes (VERDICT r1 "ordering parity
at scale"): runs the reference's own make_ordering("tree3") -- the UNMODIFIED
patchord library in oracle/_ref -- on each config's seeded points (generated
by the oracle's restatement of the workload generators, pinned bitwise to the
product's) and records sha256 of the forward permutation (int32 LE) plus
its first entries in tests/golden/perm_hashes.json.  Needs /root/reference
(oracle/_ref); C5 (1M x 960) takes ~1 h of single-threaded reference PCA.

    python tests/golden/make_perm_hashes.py c2 [c4 c5 c1]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, Ref  # noqa: E402

CONFIGS = {  # name: (generator, args) -- seed 0 = SEED_POINTS
    "c1": ("c1", (20_000, 49, 64, 1.0, 0)),
    "c2": ("3level", (1_000_000, 49, 0.125, 0)),  # C3 uses the same points
    "c4": ("c1", (4_000_000, 50, 256, 1.0, 0)),
    "c5": ("aniso", (1_000_000, 960, 32, 32, 0)),
}


def points(name):
    orc = Oracle()
    kind, a = CONFIGS[name]
    if kind == "c1":
        return orc.gen_mixture_c1(*a)
    if kind == "3level":
        return orc.gen_mixture_3level(*a)
    return orc.gen_mixture_aniso(*a)


def perm_sha(fwd) -> str:
    return hashlib.sha256(np.ascontiguousarray(fwd, "<i4").tobytes()).hexdigest()


def main():
    out_path = os.path.join(HERE, "perm_hashes.json")
    for name in sys.argv[1:] or ["c1", "c2"]:
        t0 = time.time()
        pts = points(name)
        fwd, ratio = Ref().make_ordering("tree3", pts.astype(np.float64))
        rec = {"sha256": perm_sha(fwd), "n": int(pts.shape[0]), "dim": int(pts.shape[1]),
               "head": [int(v) for v in fwd[:8]], "captured_ratio": ratio,
               "seconds": round(time.time() - t0, 1),
               "how": "oracle/_ref make_ordering('tree3') on the oracle generator's points"}
        # merge under a lock (several configs may run as parallel processes)
        import fcntl
        with open(out_path + ".lock", "w") as lk:
            fcntl.flock(lk, fcntl.LOCK_EX)
            data = {}
            if os.path.exists(out_path):
                with open(out_path) as f:
                    data = json.load(f)
            data[name] = rec
            with open(out_path, "w") as f:
                json.dump(data, f, indent=1, sort_keys=True)
        print(name, rec, flush=True)


if __name__ == "__main__":
    main()
