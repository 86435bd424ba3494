"""Static SASS instruction counts per kernel of the built library (run here):
    python tools/sass_summary.py [paper_2406_17284_b200/libltl_b200.so] > profiles/sass_summary_r02.txt
The mnemonics that prove the tcgen05 / TMA path: UTCIMMA (tcgen05.mma kind::i8),
UTMALDG / UTMASTG (TMA tensor loads / stores), LDTM / STTM (tcgen05.ld / st),
STSM (stmatrix), UTCBAR (tcgen05.commit)."""
import collections
import re
import subprocess
import sys

KEY = ["UTCIMMA", "UTMALDG", "UTMASTG", "LDTM", "STTM", "STSM", "UTCBAR", "SYNCS", "FENCE", "LDS",
       "STS", "LDG", "STG", "PRMT", "LOP3", "IADD3", "SHF"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2406_17284_b200/libltl_b200.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    print(f"cuobjdump -sass {lib} (sm_100a), static instruction counts per kernel\n")
    for block in re.split(r"\n\s*Function : ", sass)[1:]:
        name = block.split("\n", 1)[0].strip()
        if not re.search(r"ltl_tc_step_kernel|pack_kernel|base_kernel", name):
            continue
        ops = collections.Counter()
        for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", block):
            ops[m.group(1).split(".")[0]] += 1
        total = sum(ops.values())
        print(name[:120])
        print(f"  total {total} SASS instructions; " +
              ", ".join(f"{k} {ops[k]}" for k in KEY if ops[k]))
        print("  top: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(14)))


if __name__ == "__main__":
    main()
