"""(History: diagnostic of the config-4 repeatability investigation; the cause turned out to be a missing proxy
fence before the ring refills, not an MMA operand hazard -- DESIGN.md, config 4.)
Static scan of the library's SASS: for every DMMA, how many instructions later is one of its
source operand registers (A, B pairs) overwritten by an instruction that does not depend on the
DMMA's result?  (Diagnostic for the config-4 repeatability investigation: ptxas protects some of these
writes with a read scoreboard on the DMMA and relies on issue distance for others.)  Straight-line distance within a basic block; prints the closest cases per kernel.

    python tools/dmma_war_scan.py [min_distance_to_report=6]
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1406_6923_b200", "libsfw_b200.so")
LIMIT = int(sys.argv[1]) if len(sys.argv) > 1 else 6


def regs(tok, width):
    m = re.match(r"R(\d+)", tok)
    if not m:
        return set()
    r = int(m.group(1))
    return set(range(r, r + width))


def dest_regs(op, args):
    if not args:
        return set()
    width = 1
    if ".128" in op:
        width = 4
    elif ".64" in op or op.startswith(("DMMA", "DADD", "DFMA", "DMUL", "IMAD.WIDE")):
        width = 2
    if op.startswith(("ST", "BRA", "BAR", "SYNCS", "EXIT", "ISETP", "DSETP", "RED", "ATOM", "UBLKCP", "MEMBAR", "NOP")):
        return set()
    return regs(args[0], width)


sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
for fn in re.split(r"\n\s+Function : ", sass)[1:]:
    name = fn.split("\n", 1)[0].strip()
    ins = []
    for ln in fn.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)\s*(.*?);", ln)
        if m:
            ins.append((m.group(1), m.group(2), [a.strip() for a in m.group(3).split(",")]))
    n_dmma, worst = 0, []
    for i, (addr, op, args) in enumerate(ins):
        if not op.startswith("DMMA"):
            continue
        n_dmma += 1
        d = regs(args[0], 2)
        src = (regs(args[1].replace(".reuse", ""), 2) | regs(args[2].replace(".reuse", ""), 2)) - d
        for k in range(1, LIMIT + 1):
            if i + k >= len(ins):
                break
            a2, op2, args2 = ins[i + k]
            if op2.startswith(("BRA", "EXIT", "BAR", "BSYNC")):
                break
            w = dest_regs(op2, args2)
            uses_result = any(regs(a.replace(".reuse", "").lstrip("-|"), 2) & d for a in args2[1:])
            if w & src and not uses_result and not op2.startswith("DMMA"):
                worst.append((k, addr, op + " " + ", ".join(args), a2, op2 + " " + ", ".join(args2)))
                break
    if n_dmma:
        print(f"{name}: {n_dmma} DMMA, {len(worst)} with a source register overwritten within {LIMIT} instructions")
        for k, a, t, a2, t2 in sorted(worst)[:4]:
            print(f"    +{k}: /*{a}*/ {t}  ->  /*{a2}*/ {t2}")
