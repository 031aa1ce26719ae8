"""Per-kernel SASS instruction histograms of the default kernels in
libknnx.so (cuobjdump -sass), the evidence of what each kernel executes:
packed FP32 (FFMA2/FMUL2), MUFU.EX2, shared-memory (LDS/STS), global
(LDG/STG), shuffles and the programmatic-dependent-launch controls.

    python scripts/sass_evidence.py > profiles/r2_sass.md
"""
import collections
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(HERE, "paper_1709_03671_b200", "libknnx.so")
# default kernels (mangled-name fragments) and what they are
KERNELS = [
    ("spmv_tiles_g_kernelILi4ELb1E", "K3 cluster-order SpMV (C2 headline)"),
    ("spmv_orig_kernel", "K2 original-order SpMV"),
    ("gauss_lane_kernelILb1ELi2ELb0ELb0E", "K4 Gaussian recompute, D<=64, tiles"),
    ("gauss_warp_kernelILb1ELi8E", "K4 Gaussian recompute, wide rows, warp per row"),
    ("meanshift_lane_kernelILb0ELi2ELb0ELi4ELi2ELi8E", "K5 mean shift (C3, int32 ids)"),
    ("tsne_group_kernelILb0ELi2ELi8ELb0ELb1ELi6E", "K6 t-SNE, interleaved 8-lane groups (C4)"),
    ("14permute_kernelI5uint4E", "K1 permutation (16-B rows)"),
]
OPS = ["FFMA2", "FMUL2", "FADD2", "FFMA", "FADD", "FMUL", "MUFU.EX2", "MUFU.RCP", "LDG", "STG",
       "LDS", "STS", "LDSM", "SHFL", "BAR", "LDGSTS", "UBLKCP", "UTMALDG", "REDUX", "VOTE",
       "ACQBULK", "CCTL"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    print("# SASS evidence (round 2): instruction histograms of the default kernels\n")
    print("`cuobjdump -sass paper_1709_03671_b200/libknnx.so` (sm_100a), counted per "
          "static instruction; regenerate with `python scripts/sass_evidence.py`.\n")
    print("| kernel | role | " + " | ".join(OPS) + " |")
    print("|---|---|" + "---|" * len(OPS))
    for frag, role in KERNELS:
        body = next((f for f in funcs if f.split("\n", 1)[0].find(frag) >= 0), None)
        if body is None:
            print(f"| `{frag}` | {role} | (not found) |")
            continue
        cnt = collections.Counter()
        for line in body.split("\n"):
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
            if not m:
                continue
            op = m.group(1)
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    cnt[o] += 1
                    break
        print(f"| `{frag}` | {role} | " + " | ".join(str(cnt[o]) for o in OPS) + " |")


if __name__ == "__main__":
    sys.exit(main())
