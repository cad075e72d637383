"""Opcode mix of the innermost loops of a kernel in a cuobjdump -sass dump.

usage: python tools/sass_mix.py <dump.sass> <mangled-function-substring>
Prints, per backward branch (loop), the opcode histogram of its body, with
FP64-pipe ops (DADD/DMUL/DFMA/DSETP/DMNMX) totalled.
"""
import re
import sys
from collections import Counter

FP64 = {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX", "DSET"}


def function_lines(path, name):
    out, on = [], False
    for line in open(path):
        if "Function :" in line:
            on = name in line
            continue
        if on:
            out.append(line)
    return out


def parse(lines):
    ins = []
    pat = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
    for ln in lines:
        m = pat.search(ln)
        if not m:
            continue
        addr = int(m.group(1), 16)
        body = m.group(2).strip()
        toks = body.split()
        if toks and (toks[0].startswith("@")):
            toks = toks[1:]
        op = toks[0] if toks else ""
        ins.append((addr, op, body))
    return ins


def main():
    path, name = sys.argv[1], sys.argv[2]
    ins = parse(function_lines(path, name))
    loops = []
    for addr, op, body in ins:
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", body)
            if m and int(m.group(1), 16) < addr:
                loops.append((int(m.group(1), 16), addr))
    for lo, hi in loops:
        c = Counter(op.split(".")[0] for a, op, _ in ins if lo <= a <= hi)
        n = sum(c.values())
        fp64 = sum(v for k, v in c.items() if k in FP64)
        print(f"loop [{lo:#x},{hi:#x}] {n} instrs, FP64-pipe {fp64}")
        print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main()
