"""Hot CUDA source lines of one kernel in an ncu report (warp-stall samples
and executed instructions aggregated per line).

    python tools/ncu_lines.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kname="", top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    path = func = None
    hdr = None
    recs = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or kname not in (func or ""):
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        if len(r) < 8 or r[2] != "-":
            continue
        s = int(r[4] or 0)
        ie = int(float(r[7] or 0))
        if s or ie:
            recs.append((s, ie, path, line, r[1].strip()[:90]))
    tot = sum(x[0] for x in recs) or 1
    toti = sum(x[1] for x in recs) or 1
    for s, ie, p, ln, src in sorted(recs, reverse=True)[:top]:
        print("%5.1f%% %5.1f%%  %s:%d  %s" % (100 * s / tot, 100 * ie / toti, p, ln, src))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 40)
