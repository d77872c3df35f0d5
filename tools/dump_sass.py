"""Write the SASS of the kernels that run on the measured paths to profiles/sass/<name>.sass, with a
summary of the instruction mix (DMMA / UBLKCP / SYNCS / LDS / STS / DFMA counts) in
profiles/sass/SUMMARY.md.   python tools/dump_sass.py"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1406_6923_b200", "libsfw_b200.so")
OUT = os.path.join(ROOT, "profiles", "sass")
KERNELS = {  # file name -> mangled-name pattern
    "k_step_sw_4_7": r"_ZN3sfw9k_step_swILi4ELi7EEEvNS_10StepParamsE",
    "k_ustep_9_2": r"_ZN3sfw7k_ustepILi9ELi2EEEvNS_10StepParamsE",
    "k_wstep_9_2": r"_ZN3sfw7k_wstepILi9ELi2EEEvNS_7WParamsE",
    "k_step_sw4_4_7_2": r"_ZN3sfw10k_step_sw4ILi4ELi7ELi2EEEvNS_10StepParamsE",
    "k_step_mt_9": r"_ZN3sfw9k_step_mtILi9EEEvNS_8MtParamsE",
    "k_pcg2": r"_ZN3sfw6k_pcg2ENS_7PcgArgsE",
    "k_dgemm2_T": r"_ZN3sfw8k_dgemm2ILb1EEEvNS_8GemmArgsE",
    "k_dgemm2_N": r"_ZN3sfw8k_dgemm2ILb0EEEvNS_8GemmArgsE",
    "k_cholqr": r"_ZN3sfw8k_cholqr\w*",
    "k_sfraction": r"_ZN3sfw11k_sfraction\w*",
    "k_stencil": r"_ZN3sfw9k_stencil\w*",
    "k_fdtd_0": r"_ZN3sfw6k_fdtdILi0EEEvNS_8FdParamsE",
}
MNEM = ["DMMA", "UBLKCP", "LDGSTS", "SYNCS", "LDS", "STS", "LDG", "STG", "DFMA", "DADD", "DMUL", "BAR", "SHFL"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    os.makedirs(OUT, exist_ok=True)
    rows = []
    for name, pat in KERNELS.items():
        hit = [f for f in funcs if re.match(pat, f.split("\n", 1)[0].strip())]
        if not hit:
            print("missing", name, file=sys.stderr)
            continue
        # drop the hex encodings (the second line of each instruction and the trailing comment)
        body = "\n".join(re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", ln) for ln in hit[0].splitlines()
                         if not re.match(r"^\s*/\* 0x[0-9a-f]+ \*/\s*$", ln))
        with open(os.path.join(OUT, name + ".sass"), "w") as fh:
            fh.write("Function : " + body + "\n")
        ops = collections.Counter()
        for ln in body.splitlines():
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
            if m:
                ops[m.group(1).split(".")[0]] += 1
        rows.append((name, body.split("\n", 1)[0].strip(), sum(ops.values()), {k: ops.get(k, 0) for k in MNEM}))
    with open(os.path.join(OUT, "SUMMARY.md"), "w") as fh:
        fh.write("# SASS of the measured kernels (cuobjdump -sass paper_1406_6923_b200/libsfw_b200.so)\n\n")
        fh.write("Static instruction counts per kernel (tools/dump_sass.py).  DMMA = FP64 tensor MMA "
                 "(mma.sync.m8n8k4.f64), UBLKCP = TMA bulk copy (cp.async.bulk), SYNCS = mbarrier ops.\n\n")
        fh.write("| file | kernel | instructions | " + " | ".join(MNEM) + " |\n")
        fh.write("|---|---|---|" + "---|" * len(MNEM) + "\n")
        for name, mangled, tot, c in rows:
            fh.write(f"| {name}.sass | `{mangled[:60]}` | {tot} | " + " | ".join(str(c[k]) for k in MNEM) + " |\n")
    print(open(os.path.join(OUT, "SUMMARY.md")).read())


if __name__ == "__main__":
    main()
