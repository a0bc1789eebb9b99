"""Hot SASS runs of one ncu report (measurement scaffolding).

    python tools/ncu_sass_blocks.py REP [per_unit_divisor] [top]

Groups consecutive SASS instructions with equal execution counts (basic-block
like runs) and prints the runs with the most executed warp instructions,
each count divided by `per_unit_divisor` (e.g. warp-tables) with its code.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ie, te, src = h.index("Instructions Executed"), h.index("Thread Instructions Executed"), 1
    runs, cur = [], None
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        n = int(r[ie] or 0)
        if cur is None or n != cur[0]:
            cur = [n, []]
            runs.append(cur)
        cur[1].append((r[0][-5:], r[src].strip(), int(r[te] or 0)))
    total = sum(n * len(c) for n, c in runs) or 1
    print(f"total warp instructions {total} ({total / div:.0f} per unit)")
    for n, code in sorted(runs, key=lambda x: -x[0] * len(x[1]))[:top]:
        act = sum(c[2] for c in code) / max(1, n * len(code))
        print(f"--- {len(code)} instr x {n / div:.2f} per unit = {100 * n * len(code) / total:.1f}% "
              f"(active {act:.1f})")
        for a, s, _ in code:
            print(f"   {a} {s}")


if __name__ == "__main__":
    main()
