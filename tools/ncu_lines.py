"""Per-source-line instruction / stall breakdown of one ncu report.

    python tools/ncu_lines.py gpurun_out/prof_X.ncu-rep [top]

Reads `ncu -i REP --page source --csv --print-source cuda,sass` (the report
must have been captured with --import-source on and the code built with
-lineinfo) and prints the source lines with the most warp instructions,
their thread instructions (divergence) and stall samples.
"""
import csv
import io
import subprocess
import sys


def lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    fname, hdr, res = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] in ("File Name", "File Path"):
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr) or not r[0]:
            continue
        d = dict(zip(hdr, r))
        try:
            ie = int(d.get("Instructions Executed") or 0)
            te = int(d.get("Thread Instructions Executed") or 0)
            ss = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            continue
        if ie or ss:
            res.append((ie, te, ss, fname, r[0], r[1].strip()[:80]))
    return res


def merged(res):
    # a report holding several launches lists every source line once per
    # launch: sum them
    acc = {}
    for ie, te, ss, f, ln, src in res:
        a = acc.setdefault((f, ln), [0, 0, 0, src])
        a[0] += ie
        a[1] += te
        a[2] += ss
    return [(a[0], a[1], a[2], f, ln, a[3]) for (f, ln), a in acc.items()]


def main():
    res = merged(lines(sys.argv[1]))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    ti = sum(r[0] for r in res) or 1
    tt = sum(r[1] for r in res) or 1
    ts = sum(r[2] for r in res) or 1
    print(f"warp inst {ti}, thread inst {tt} (avg active {tt / ti:.1f}), stall samples {ts}")
    for ie, te, ss, f, ln, src in sorted(res, key=lambda r: -r[2])[:top]:
        print(f"{100 * ie / ti:5.1f}% inst {100 * ss / ts:5.1f}% stall act {te / max(ie, 1):4.1f}  "
              f"{f}:{ln}  {src}")


if __name__ == "__main__":
    main()
