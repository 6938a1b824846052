"""Summarize an ncu --set full report: key raw metrics + per-source-line hot spots.
usage: python profiles/ncu_summarize.py <report.ncu-rep> [top_n]
       python profiles/ncu_summarize.py --traffic <cfg>=<report.ncu-rep> ... [--source-dir profiles/rNN]
         -> merges {cfg: {kernel, bytes_per_launch, ...}} into profiles/traffic.json (read by bench.py)"""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "derived__memory_l1_wavefronts_shared_excessive", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second"]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    ix = {h: i for i, h in enumerate(hdr)}
    print("kernel:", vals[ix["Kernel Name"]][:100])
    for k in KEYS:
        if k in ix:
            print(f"  {k} = {vals[ix[k]]} {units[ix[k]]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h = srows[1]
    si = {x: i for i, x in enumerate(h)}
    ops = Counter()
    stall = Counter()
    for r in srows[2:]:
        if len(r) < len(h):
            continue
        toks = r[si["Source"]].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        try:
            ops[op.split(".")[0]] += float(r[si["Instructions Executed"]] or 0)
            stall[op.split(".")[0]] += float(r[si["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            pass
    tot = sum(ops.values()) or 1
    tots = sum(stall.values()) or 1
    print("  instruction mix (executed %, stall-sample %):")
    for k, v in ops.most_common(top):
        print(f"    {k:10s} {100 * v / tot:5.1f}%  {100 * stall[k] / tots:5.1f}%")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    agg = Counter()
    for r in srows[2:]:
        if len(r) < len(h):
            continue
        for c in reasons:
            try:
                agg[c] += float(r[si[c]] or 0)
            except ValueError:
                pass
    tr = sum(agg.values()) or 1
    print("  stall reasons:", ", ".join(f"{k[6:]} {100 * v / tr:.0f}%" for k, v in agg.most_common(6)))


def raw_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(v.replace(",", "")) * scale


def to_us(v, unit):
    """ncu prints gpu__time_duration in whatever unit fits (nsecond / usecond / msecond / second)."""
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}[unit]
    return float(v.replace(",", "")) * scale


def to_ghz(v, unit):
    scale = {"hz": 1e-9, "khz": 1e-6, "mhz": 1e-3, "ghz": 1.0, "cycle/second": 1e-9, "cycle/nsecond": 1.0,
             "cycle/usecond": 1e-3}[unit.lower()]
    return float(v.replace(",", "")) * scale


def traffic(args):
    import json
    import os
    src_dir = None
    if "--source-dir" in args:
        i = args.index("--source-dir")
        src_dir = args[i + 1]
        args = args[:i] + args[i + 2:]
    path = os.environ.get("TRAFFIC_JSON") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    try:
        with open(path) as f:
            out = json.load(f)
    except OSError:
        out = {}
    for a in args:
        cfg, rep = a.split("=", 1)
        instances = None  # cfg=report@N: the capture ran N instances (bench.py scales to its count)
        if "@" in rep:
            rep, n = rep.rsplit("@", 1)
            instances = int(n)
        m = raw_metrics(rep)
        rd = to_bytes(*m["dram__bytes_read.sum"])
        wr = to_bytes(*m["dram__bytes_write.sum"])
        dur_us = to_us(*m["gpu__time_duration.sum"])
        wf = float(m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][0].replace(",", ""))
        exc = float(m["derived__memory_l1_wavefronts_shared_excessive"][0].replace(",", ""))
        clk = to_ghz(*m["sm__cycles_elapsed.avg.per_second"])
        # shared memory: one wavefront moves up to 128 B; peak 128 B/clk/SM x 148 SMs
        smem_peak_gbs = 128 * 148 * clk
        out[cfg] = {"kernel": m["Kernel Name"][0][:120], "bytes_per_launch": rd + wr, "read_bytes": rd,
                    "write_bytes": wr, "ncu_duration_us": dur_us,
                    "smem_wavefronts": wf, "smem_excessive_wavefronts": exc,
                    "smem_wavefront_bytes_per_launch": wf * 128, "smem_peak_gbs_at_clock": smem_peak_gbs,
                    "smem_frac_of_peak_under_ncu": (wf / (dur_us * 1e-6)) / (148 * clk * 1e9),
                    "issue_active_pct": float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
                    "bank_conflicts_ld": float(m["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"][0]
                                               .replace(",", "")),
                    "bank_conflicts_st": float(m["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"][0]
                                               .replace(",", "")),
                    "warp_instructions": float(m["smsp__inst_executed.sum"][0].replace(",", "")),
                    "source": os.path.join(src_dir or os.path.dirname(rep), os.path.basename(rep))}
        if instances:
            out[cfg]["instances"] = instances
        print(cfg, out[cfg])
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--traffic":
        traffic(sys.argv[2:])
    else:
        main()
