"""SASS census of the hop kernels: per kernel instantiation, the count of the
Blackwell instructions that prove the tensor-core / TMEM / bulk-copy path
(UTCIMMA = tcgen05.mma kind::i8, UTCHMMA = kind::f16, LDTM = tcgen05.ld,
UTCBAR = tcgen05.commit, UBLKCP = cp.async.bulk, SYNCS = mbarrier ops), plus
registers / stack / local memory from the resource usage.  Runs on the CPU
box against the built object (cuobjdump).

    python tools/sass_census.py > profiles/r02_sass_census.json
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJS = [os.path.join(ROOT, "paper_2602_08501_b200", "csrc", "build", o) for o in ("hop_ar.o", "hop_tc.o")]
KEYS = ("UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "SYNCS",
        "USETMAXREG", "IDP", "VIMNMX3", "FMNMX3", "LDL", "STL")


def demangle(name):
    m = re.match(r"_ZN2tc13hop_tc_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)EEEvNS_6ParamsE", name)
    a = re.match(r"_ZN2ar13hop_ar_kernelILi(\d+)ELi(\d+)ELb([01])EEEvNS_6ParamsE", name)
    if a:
        return f"hop_ar_kernel<KB={a.group(1)},NW={a.group(2)},STATS={a.group(3)}>"
    if not m:
        return name
    kb, nw, limbs, mode, cl, pm = map(int, m.groups())
    return f"hop_tc_kernel<KB={kb},NW={nw},LIMBS={limbs},MODE={mode},CL={cl},PM={pm}>"


def census(OBJ):
    sass = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", OBJ], capture_output=True, text=True,
                         check=True).stdout
    usage = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", res):
        usage[m.group(1)] = dict(registers=int(m.group(2)), stack=int(m.group(3)), local=int(m.group(5)))
    out = {}
    for block in re.split(r"\n\s*Function : ", sass)[1:]:
        name = block.split("\n", 1)[0].strip()
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", block)
        counts = {k: 0 for k in KEYS}
        for op in ops:
            if op in counts:
                counts[op] += 1
        out[demangle(name)] = dict(instructions=len(ops), **counts, **usage.get(name, {}))
    return out


def main():
    json.dump({"objects": {os.path.relpath(o, ROOT): census(o) for o in OBJS}}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
