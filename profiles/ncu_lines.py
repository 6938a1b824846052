"""Per-CUDA-source-line hot spots of an ncu --set full capture (kernels built with -lineinfo,
captured with --import-source on):
    python profiles/ncu_lines.py <report.ncu-rep> [top_n]
Prints the source lines with the most warp-stall samples and executed instructions (with the
share of each), from `ncu --page source --print-source cuda,sass`."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    cur_file, hdr, lines = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            st = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            ins = float(r[hdr["Instructions Executed"]] or 0)
        except (ValueError, KeyError, IndexError):
            continue
        lines.append((cur_file, r[0], r[1][:90], st, ins))
    tst = sum(x[3] for x in lines) or 1
    tin = sum(x[4] for x in lines) or 1
    print(f"{'stall%':>7} {'inst%':>6}  file:line  source")
    for f, ln, src, st, ins in sorted(lines, key=lambda x: -x[3])[:top]:
        print(f"{100 * st / tst:7.2f} {100 * ins / tin:6.2f}  {f}:{ln}  {src}")
    by_file = {}
    for f, _, _, st, ins in lines:
        a = by_file.setdefault(f, [0.0, 0.0])
        a[0] += st
        a[1] += ins
    print("per file:", ", ".join(f"{f} {100 * a[0] / tst:.1f}%/{100 * a[1] / tin:.1f}%" for f, a in
                                 sorted(by_file.items(), key=lambda kv: -kv[1][0])))


if __name__ == "__main__":
    main()
