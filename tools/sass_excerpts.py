#!/usr/bin/env python
"""SASS evidence for the hot kernels (no GPU needed): for each kernel, the counts of the
instructions the design relies on and the first lines of its hot loop, from `cuobjdump -sass` of
the in-tree objects (build/cannikin/*.o).

    python tools/sass_excerpts.py > profiles/r02/sass_excerpts.txt

  LDG.E.NA.128 / LDG.E.128  128-bit global loads (K2: L1::no_allocate streaming)
  STG.E.128 / STG.E.NA.128  128-bit stores
  FFMA2                     sm_100's packed fp32x2 FMA (K2's dev::wsum16)
  PREEXIT / ACQBULK         griddepcontrol.launch_dependents / .wait (K2's programmatic launch)
  UBLKCP / SYNCS            cp.async.bulk (TMA bulk copy) and its mbarrier (K2 TMA variant)
  LDGMC / STGMC... (multimem) NVSwitch multicast load-reduce / store (K6)
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "build", "cannikin")
KERNELS = [
    ("K2 LDG (C4: bf16, 8 ranks)", "wsum_local.cu.o",
     "_ZN8cannikin17wsum_local_kernelI13__nv_bfloat16Li8ELi1ELi256EEEvNS_9LocalArgsE"),
    ("K2 LDG (fp32, 2 ranks, U=4)", "wsum_local.cu.o",
     "_ZN8cannikin17wsum_local_kernelIfLi2ELi4ELi256EEEvNS_9LocalArgsE"),
    ("K2 TMA variant (bf16, 8 ranks)", "wsum_local_tma.cu.o", "wsum_local_tma_kernelI13__nv_bfloat16Li8E"),
    ("K3 two-shot pull (bf16, W=2)", "twoshot.cu.o",
     "_ZN8cannikin14twoshot_kernelI13__nv_bfloat16Li2ELi4ELi512EEEvNS_6ArArgsE"),
    ("K3 push (bf16, W=8)", "twoshot.cu.o", "twoshot_push_kernelI13__nv_bfloat16Li8E"),
    ("K3 LL128 (fp32, W=4)", "ll128.cu.o", "_ZN8cannikin12ll128_kernelIfLi4EEEvNS_9LL128ArgsE"),
    ("K3 LL (fp32, W=2)", "ll.cu.o", "_ZN8cannikin9ll_kernelIfLi2EEEvNS_6LLArgsE"),
    ("K6 NVLS (fp32)", "nvls.cu.o", "nvls_kernelIfE"),
]
KEYS = ["LDG.E.NA.128", "LDG.E.128", "LDG.E.STRONG.SYS.128", "LD.E.STRONG.SYS.128", "STG.E.128",
        "STG.E.NA.128", "STG.E.STRONG.SYS.128", "FFMA2", "FFMA", "PREEXIT", "ACQBULK", "UBLKCP",
        "SYNCS", "LDGMC", "STGMC", "MEMBAR", "DADD"]


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs, cur, name = {}, [], None
    for ln in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            if name:
                funcs[name] = cur
            name, cur = m.group(1), []
        elif name and re.match(r"\s+/\*[0-9a-f]{4}\*/", ln):
            cur.append(ln.split(";")[0].strip())
    if name:
        funcs[name] = cur
    return funcs


def main():
    cache = {}
    for title, obj, pat in KERNELS:
        path = os.path.join(OBJ, obj)
        if path not in cache:
            cache[path] = functions(path)
        names = [n for n in cache[path] if pat in n]
        if not names:
            print(f"== {title}: {pat} not found in {obj}\n")
            continue
        code = cache[path][names[0]]
        ops = [re.sub(r"^/\*[0-9a-f]+\*/\s*", "", c) for c in code]
        ops = [re.sub(r"^@!?U?P\w+\s+", "", o) for o in ops]
        counts = {k: sum(1 for o in ops if o.split(" ")[0] == k or o.split(" ")[0].startswith(k + "."))
                  for k in KEYS}
        counts = {k: v for k, v in counts.items() if v}
        print(f"== {title}\n   {names[0]}\n   {len(code)} instructions; key counts: {counts}")
        # first window of the hot loop: from the first 128-bit / multimem load, 28 lines
        first = next((i for i, o in enumerate(ops)
                      if re.match(r"(LDG|LD|LDGMC|UBLKCP)\S*128|LDGMC|UBLKCP", o.split(" ")[0])), None)
        if first is not None:
            for ln in code[first:first + 28]:
                print("   " + ln)
        print()


if __name__ == "__main__":
    sys.exit(main())
