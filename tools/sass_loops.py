#!/usr/bin/env python3
"""Per-loop instruction mix of a kernel's SASS: sass_loops.py file.o <substring of the mangled name> [min_len]
(cuobjdump -sass; loops = backward branches; classes FP64 / move / shuffle / memory / branch / other)."""
import collections
import re
import subprocess
import sys


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    min_len = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0]
        if pat not in name:
            continue
        ins = [(int(m.group(1), 16), m.group(2)) for m in re.finditer(r"/\*([0-9a-f]{4,5})\*/\s+(.*?);", f)]
        print(f"== {name}: {len(ins)} instructions")
        for a, t in ins:
            # loops close with a predicated backward branch (@P BRA / BRA.U UP); returns from out-of-line paths do not
            if not (t.startswith("@") or re.match(r"BRA\.U\s+!?UP", t)):
                continue
            m = re.search(r"BRA\S*\s+(?:\S+,\s*)?0x([0-9a-f]+)", t)
            if not m or "BRA.DIV" in t:
                continue
            tgt = int(m.group(1), 16)
            if tgt >= a or (a - tgt) // 16 < min_len:
                continue
            body = [re.sub(r"^@!?U?P\d+\s+", "", x) for aa, x in ins if tgt <= aa <= a]
            c = collections.Counter(x.split()[0] for x in body)
            cls = collections.Counter()
            for op, v in c.items():
                if op in ("DFMA", "DADD", "DMUL"):
                    cls["fp64"] += v
                elif op.startswith("IMAD.MOV") or op in ("MOV", "CS2R", "UMOV"):
                    cls["move"] += v
                elif op.startswith("SHFL"):
                    cls["shfl"] += v
                elif op.startswith(("LDG", "STG", "LDS", "STS", "CCTL", "LD.", "ST.")):
                    cls["mem"] += v
                elif op.startswith(("BRA", "BSSY", "BSYNC", "WARPSYNC")):
                    cls["branch"] += v
                else:
                    cls["other"] += v
            print(f"  loop {tgt:#x}..{a:#x}: {len(body)} instr  " + "  ".join(f"{k}={v}" for k, v in cls.most_common()))
            print("     " + " ".join(f"{k}:{v}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
