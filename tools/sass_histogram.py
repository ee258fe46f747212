"""Instruction histogram of the built kernels (cuobjdump -sass of the in-tree
objects): the mnemonics that prove the Blackwell paths -- DMMA (FP64 tensor
MMA), UTMALDG / UTMASTG / UBLKCP / UBLKRED (TMA and bulk copies / reductions),
SYNCS (mbarrier), plus LDS / STG / BAR -- per kernel.

    python tools/sass_histogram.py > profiles/sass_histogram_r02.json
"""
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("DMMA", "DFMA", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "UBLKRED", "SYNCS", "LDS", "LDSM",
        "LDG", "STG", "STS", "BAR", "ATOMG", "REDG", "MEMBAR", "UCGABAR")


def main():
    out = {}
    for obj in ("mf_leaf.cu.o", "mf_fixed.cu.o", "mf_kron.cu.o", "mf_mix.cu.o", "mf_tiny.cu.o", "mf_comm.cu.o"):
        path = os.path.join(ROOT, "paper_2312_12732_b200", "_build", obj)
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        for block in re.split(r"\n\s+Function : ", sass)[1:]:
            name = block.split("\n", 1)[0].strip()
            demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            ops = collections.Counter()
            for line in block.split("\n"):
                m = re.match(r"\s+/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
                if m:
                    ops[m.group(1).split(".")[0]] += 1
            out.setdefault(obj, {})[demangled[:160]] = {k: ops[k] for k in KEYS if ops[k]} | {
                "total": sum(ops.values())}
    print(json.dumps({"what": "SASS instruction counts per kernel (static, cuobjdump -sass of the "
                              "sm_100a objects of libmf.so)", "objects": out}, indent=1))


if __name__ == "__main__":
    main()
