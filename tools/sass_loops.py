"""Opcode histogram of the innermost backward-branch loops of one kernel.

    python tools/sass_loops.py <object.o> <mangled-kernel-name> [min_len]
"""
import collections
import re
import subprocess
import sys


def main():
    obj, fn = sys.argv[1], sys.argv[2]
    min_len = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True,
                          text=True).stdout
    ins = []
    for line in sass.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    for a, t in ins:
        m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or (a - tgt) // 16 < min_len:
            continue
        body = [x for b, x in ins if tgt <= b <= a]
        ops = collections.Counter((x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0]
                                  for x in body)
        print(f"loop {hex(tgt)}..{hex(a)}: {len(body)} instructions")
        print("   " + ", ".join(f"{k} {v}" for k, v in ops.most_common()))


if __name__ == "__main__":
    main()
