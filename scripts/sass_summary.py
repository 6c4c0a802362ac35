#!/usr/bin/env python3
"""Per-kernel SASS evidence of the built library: Blackwell bulk-copy / TMA and mbarrier instructions, registers,
static shared memory, spills.

  UBLKCP.S.G   cp.async.bulk global -> shared (1-D TMA bulk copy into an mbarrier-tracked stage)
  UBLKCP.G.S   cp.async.bulk shared -> global (bulk store)
  UTMALDG      cp.async.bulk.tensor (2-D/3-D TMA tensor load through a tensor map)
  SYNCS.*      mbarrier arrive / expect-tx / try-wait (the TMA completion protocol)
  LDGSTS       cp.async (Ampere-style, 4/8/16 B)

    python scripts/sass_summary.py [path/to/libcodecsight.so] > profiles/r02_sass.txt
"""
from __future__ import annotations

import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_06036_b200", "libcodecsight.so")
OPS = ("UBLKCP.S.G", "UBLKCP.G.S", "UTMALDG", "UTMASTG", "SYNCS", "LDGSTS", "HMMA", "UTCMMA")


def demangle_short(name: str) -> str:
    m = re.search(r"_cu_[0-9a-f]+\d+(\w+?)(I.*)?E(v|N)", name)
    try:
        out = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        out = name
    out = re.sub(r"\(anonymous namespace\)::", "", out)
    out = re.sub(r"\(.*\)$", "", out)
    return out or (m.group(1) if m else name)


def parse(lib: str = LIB) -> dict:
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True,
                         check=True).stdout
    kernels: dict = {}
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            cur = kernels.setdefault(m.group(1), {op: 0 for op in OPS} | {"instructions": 0})
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if not m:
            continue
        op = m.group(2)
        cur["instructions"] += 1
        for key in OPS:
            if op == key or op.startswith(key + "."):
                cur[key] += 1
    fn = None
    for ln in res.splitlines():
        m = re.match(r"\s*Function (\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", ln)
        if m and fn in kernels:
            kernels[fn].update(reg=int(m.group(1)), stack=int(m.group(2)), smem_static=int(m.group(3)),
                               local=int(m.group(4)))
    return {demangle_short(k): v for k, v in kernels.items()}


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else LIB
    ks = parse(lib)
    cols = ("UBLKCP.S.G", "UBLKCP.G.S", "UTMALDG", "SYNCS", "LDGSTS")
    print(f"# SASS summary of {os.path.relpath(lib, ROOT)} (cuobjdump -sass / --dump-resource-usage, sm_100a)")
    print(f"{'kernel':72s} {'insts':>6s} " + " ".join(f"{c:>10s}" for c in cols) + f" {'reg':>4s} {'smem':>6s} "
          f"{'stack':>5s}")
    for name in sorted(ks):
        v = ks[name]
        print(f"{name[:72]:72s} {v['instructions']:6d} " + " ".join(f"{v[c]:10d}" for c in cols) +
              f" {v.get('reg', -1):4d} {v.get('smem_static', -1):6d} {v.get('stack', -1):5d}")


if __name__ == "__main__":
    main()
