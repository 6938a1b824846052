"""bench.py -- keys/s of the B200 bank-conflict-free kernels (BASELINE.json metric).

Default workload (BASELINE.json configs[2], the largest configuration that fits one GPU and
one the reference accepts as is): the bank-conflict-free sort, w = 32, n = 4096 uint32 keys
per block-tile (a 32 x 128 machine), 2^20 tiles per GPU = 2^32 keys (16 GiB in + 16 GiB
out), keys generated on the device (the builder-defined uint32 generator).
The reference path is integer_sort_general(view, 2^32) (partition.hpp:436-449), which the
reference arm (`--impl reference`) runs on the same 32 x 128 tiles.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl reference]

Other configs (`--config`): cfg1 (32 x 32 partition), cfg2b (32 x 16 general partition),
cfg4 / cfg4s (permutation), cfg5 (global 8-way partition) and cfg2 (32 x 8 general
partition: a B200 EXTENSION -- the reference rejects that shape, partition.hpp:241-244 --
so its reference arm times 32 x 16 and says so).

A "step" is one pass of the kernel over the whole batch.  value = keys/s over the job
(inputs resident in HBM); e2e = the same metric through the public API with the inputs in
pinned host memory, H2D + kernel + D2H inside the timed region.  Every batch is larger than
the 126 MB L2, so no explicit flush is needed.  After timing, the output is checked at full
size (cfg3: per-tile key sum, sum of squares and XOR against the input, sortedness, and an
exact comparison of sampled tiles against numpy's sort).
Multi-GPU: instances are sharded across ranks (weak scaling, no collective in the data path).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (algorithm, w, m, instances per GPU, flags, description)
    "cfg1": ("partition_general", 32, 32, 1 << 16, 0,
             "w-way partition w=32, n=w^2=1024 uint32 per instance, 65536 instances (reference path: shearsort_rect)"),
    "cfg2": ("partition_general", 32, 8, 1 << 18, 1,
             "general w-way partition w=32, n=256 (n<w^2) per instance, 2^18 instances "
             "[B200 EXTENSION: the reference rejects 32x8; DMM_FLAG_EXT_PARTIAL_GROUPS]"),
    "cfg2b": ("partition_general", 32, 16, 1 << 17, 0,
              "general w-way partition w=32, n=512 (reference-accepted stand-in of cfg2), 2^17 instances"),
    "cfg3": ("integer_sort_general", 32, 128, 1 << 20, 0,
             "bank-conflict-free sort w=32, n=4096 uint32 keys per block-tile (32x128 machine), 2^20 tiles "
             "(reference path: integer_sort_general(view, 2^32))"),
    "cfg1sw": ("partition_short_wide", 32, 1024, 1 << 13, 0,
               "w-way partition at the paper's native mapping w=32, n=32*w^2=32768 uint32 labels per instance "
               "(the Corollary's short-wide machine 32x1024: partition_short_wide), 2^13 instances"),
    "cfg3sw": ("sort_short_wide", 32, 1024, 1 << 15, 0,
               "bank-conflict-free sort w=32, n=32768 uint32 keys per instance (sort_short_wide, Lemma 1 on the "
               "32x1024 machine), 2^15 instances"),
    "cfg5": ("global_partition", 1, 1 << 26, 8, 0,
             "global 8-way partition of 2^32 uint32 keys across 8 GPUs: 2^29 keys per GPU (label = key >> 29), "
             "local stable multisplit + NCCL all-to-all"),
    "cfg4": ("permute", 128, 64, 1 << 18, 0,
             "randomized permutation n=8192 per instance as the reference's accepted 128x64 machine "
             "(it rejects n=8192 at w=32: 32x256 fails m | w), 4 warps per machine, seeded Rng per instance, "
             "2^18 instances"),
    "cfg4s": ("permute", 32, 32, 1 << 18, 0,
              "randomized permutation w=32, n=1024 per instance (one-warp stand-in), seeded Rng per instance, "
              "2^18 instances"),
}
ALG_ID = {"partition_general": 5, "integer_sort_general": 6, "permute": 7, "partition_short_wide": 3,
          "sort_short_wide": 0}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in-process through NVML
    (every 10 ms; forking nvidia-smi from a process with a large CUDA address space stalls
    the launching thread), falling back to nvidia-smi when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None

    def _handle(self, nv):
        # the NVML device of this process's CUDA device (CUDA_VISIBLE_DEVICES may renumber it)
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _run_nvml(self, nv):
        h = self._handle(nv)
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while True:
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            if self._stop.wait(0.01):
                break

    def _run_smi(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
            "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 6:
                    self.samples.append((float(f[0]), float(f[1]),
                                         {n for n, v in zip(self.NAMES, f[2:6]) if v.lower().startswith("active")}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        if os.environ.get("DMM_BENCH_NO_CLOCKS"):  # diagnostics only: no sampling thread
            self.source = None
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            target = lambda: self._run_nvml(nv)  # noqa: E731
            self.source = "nvml"
        except Exception:
            target = self._run_smi
            self.source = "nvidia-smi"
        self._t = threading.Thread(target=target, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))), "samples": len(self.samples),
                "source": getattr(self, "source", None)}


def cpu_baseline(cfg_name: str, seconds: float = 15.0):
    """The reference's own run_algorithm on the host cores (oracle/_ref), bounded sample."""
    from oracle.oracle import Port, Ref
    alg, w, m, count, flags, _ = CONFIGS[cfg_name]
    note = ""
    alg_id = ALG_ID.get(alg)
    kind = {"partition_general": 1, "integer_sort_general": 0, "permute": 2, "partition_short_wide": 1,
            "sort_short_wide": 0}.get(alg)
    if cfg_name == "cfg2":
        # the reference rejects 32 x 8 (balance leftover group, partition.hpp:241-244): time the
        # closest shape it accepts, general partition 32 x 16
        m = 16
        note = "reference rejects 32x8 (ShapeViolation); timed its closest accepted general shape 32x16; "
    if alg == "global_partition":
        # no reference path partitions 2^32 keys (~137 GB of machine cells); its own 8-way partition
        # of one 8 x 65536 instance (partition_short_wide, partition.hpp:178) is the stand-in
        alg, alg_id, kind, w, m = "partition_short_wide", 3, 1, 8, 65536
        note = "8-way partition stand-in: reference partition_short_wide on 8 x 65536 instances; "
    if not Ref.available():
        return None
    ref, port = Ref(), Port()
    import numpy as np
    nthreads = os.cpu_count() or 1
    sample = 64 if w * m <= 4096 else nthreads
    # grow the sample until the run takes ~seconds/4 (bounded)
    while True:
        if kind == 0:
            inst = np.stack([port.gen_sort_u32(w, m, s) for s in range(sample)]).astype(np.uint32)
        else:
            inst = np.stack([port.gen_instance(kind, w, m, s) for s in range(sample)]).astype(np.uint32)
        st, secs, good = ref.cpu_baseline(alg_id, inst, seeds=np.arange(sample, dtype=np.uint64),
                                          domain=1 << 32, nthreads=nthreads)
        if secs * 4 >= seconds or sample >= (1 << 16) or sample * w * m >= (1 << 26):
            break
        sample *= 2
    # the growth runs warmed the host; multi-threaded host timings vary run to run, so take
    # the median of three timed runs of the final sample
    times = [secs]
    for _ in range(2):
        _, t, g2 = ref.cpu_baseline(alg_id, inst, seeds=np.arange(sample, dtype=np.uint64),
                                    domain=1 << 32, nthreads=nthreads)
        times.append(t)
        good = min(good, g2)
    secs = sorted(times)[1]
    keys = sample * w * m
    return {"value": keys / secs, "unit": "keys/s", "cores": nthreads, "kind": "reference",
            "sample": f"{note}{sample} instances of {w}x{m} through run_algorithm({alg}) "
                      f"(strict, auditor on, host_threads=1) on {nthreads} threads, median of 3 "
                      f"runs {secs:.2f} s (range {min(times):.2f}-{max(times):.2f} s), "
                      f"{good}/{sample} correct"}


def smem_line(traffic, ms):
    """Shared-memory side of the roofline: the committed ncu capture's wavefronts per launch
    (x 128 B) over this run's launch time, against 128 B/clk/SM x 148 SMs at the max SM clock;
    plus its bank-conflict count (excessive wavefronts)."""
    if not traffic or "smem_wavefronts" not in traffic:
        return None
    peaks, _ = _peaks()
    peak = 128 * 148 * peaks.get("sm_max_mhz", 1965.0) / 1e3  # GB/s
    achieved = traffic["smem_wavefronts"] * 128 / (ms / 1e3) / 1e9
    return {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "wavefronts_per_launch": traffic["smem_wavefronts"],
            "excessive_wavefronts_per_launch": traffic["smem_excessive_wavefronts"],
            # what actually bounds these kernels: the SM's instruction issue (ncu, same launch)
            "issue_active_pct_of_peak": traffic.get("issue_active_pct"),
            "source": traffic.get("source")}


def measured_traffic(cfg_name: str, count: int = 0):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the config's dominant kernel,
    from the committed ncu --set full capture (profiles/traffic.json, written by
    profiles/ncu_summarize.py --traffic), or None.  A capture of fewer instances than this
    run's `count` (its "instances" field) is scaled linearly to it."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(cfg_name)
    except (OSError, ValueError):
        return None
    if t and count and t.get("instances") and t["instances"] != count:
        t = dict(t)
        f = count / t["instances"]
        for key in ("bytes_per_launch", "read_bytes", "write_bytes", "smem_wavefronts",
                    "smem_excessive_wavefronts", "smem_wavefront_bytes_per_launch", "ncu_duration_us"):
            if key in t:
                t[key] = t[key] * f
        t["scaled_from_instances"] = t["instances"]
    return t


def workload_config(cfg_name: str, world: int = 1, count: int = 0, graph: bool = True, transport: str = "p2p"):
    """The `config` object of the bench line, shared by both arms."""
    alg, w, m, cnt, flags, desc = CONFIGS[cfg_name]
    if count:
        cnt = count
        desc += f" [count overridden: {count}]"
    return {"workload": desc, "name": cfg_name, "algorithm": alg, "w": w, "m": m, "instances_per_gpu": cnt,
            "keys_per_gpu": cnt * w * m, "l2": "inputs >= 2x L2 (no flush needed)",
            "timed_loop": "CUDA graph replay of the one-launch step" if graph and alg != "global_partition"
            else "eager launches",
            "parallelism": (f"instances sharded over {world} GPU(s)" if alg != "global_partition" else
                            f"keys sharded over {world} GPU(s); exchange: " +
                            ("fused into the scatter (stores into the owners' receive buffers, "
                             "CUDA IPC / NVLink peer memory)" if transport == "p2p"
                             else "multisplit + NCCL all-to-all"))}


def verify_sort_full(g, out, count: int, tiles_exact: int = 64) -> dict:
    """Full-size check of a batched sort: per tile, the 64-bit key sum, the 64-bit sum of
    squares and the XOR of the output equal the input's (the multiset survives), every tile is
    ascending, and `tiles_exact` tiles spread over the batch equal numpy's sort exactly."""
    import numpy as np
    import torch
    n = g[0].numel()
    gi, go = g.view(count, n), out.view(count, n)
    ok_sum = ok_xor = ok_sorted = True
    chunk = max(1, (1 << 26) // n)
    for lo in range(0, count, chunk):
        hi = min(count, lo + chunk)
        a = gi[lo:hi].to(torch.int64) & 0xFFFFFFFF
        b = go[lo:hi].to(torch.int64) & 0xFFFFFFFF
        ok_sum &= bool((a.sum(1) == b.sum(1)).all()) and bool(((a * a).sum(1) == (b * b).sum(1)).all())
        ok_sorted &= bool((b[:, 1:] >= b[:, :-1]).all())
        del a, b
        xa, xb = gi[lo:hi], go[lo:hi]
        while xa.shape[1] > 1:
            h = xa.shape[1] // 2
            xa = xa[:, :h] ^ xa[:, h: 2 * h] if xa.shape[1] % 2 == 0 else torch.cat(
                [xa[:, :h] ^ xa[:, h: 2 * h], xa[:, 2 * h:]], 1)
            xb = xb[:, :h] ^ xb[:, h: 2 * h] if xb.shape[1] % 2 == 0 else torch.cat(
                [xb[:, :h] ^ xb[:, h: 2 * h], xb[:, 2 * h:]], 1)
        ok_xor &= bool((xa == xb).all())
    idx = np.unique(np.linspace(0, count - 1, min(count, tiles_exact)).astype(np.int64))
    hin = gi[torch.as_tensor(idx, device=g.device)].cpu().numpy().view(np.uint32)
    hout = go[torch.as_tensor(idx, device=g.device)].cpu().numpy().view(np.uint32)
    ok_exact = bool((np.sort(hin, axis=1) == hout).all())
    return {"tiles": count, "sum_sumsq": ok_sum, "xor": ok_xor, "ascending": ok_sorted,
            "exact_tiles": int(len(idx)), "exact": ok_exact,
            "ok": ok_sum and ok_xor and ok_sorted and ok_exact}


SECONDARY = ["cfg1", "cfg1sw", "cfg2", "cfg2b", "cfg3sw", "cfg4", "cfg4s", "cfg5"]


def run_secondaries(args) -> dict:
    """The default run also measures every other config once (device-resident throughput,
    20-step-style timing with fewer steps, its own correctness check, no e2e / CPU leg), so the
    driver's single default invocation carries evidence for all BASELINE configs.  Each runs in
    its own process (fresh device memory)."""
    res = {}
    for c in SECONDARY:
        cmd = [sys.executable, os.path.abspath(__file__), "--config", c, "--steps", "10", "--warmup", "3",
               "--no-cpu-baseline", "--no-e2e", "--no-secondary"]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
            line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
            res[c] = {"workload": line["config"]["workload"], "value": line["value"], "unit": line["unit"],
                      "ms_per_step": line["ms_per_step"], "steps": line["steps"],
                      "roofline_frac": line["roofline"]["frac"], "correct": line["correct"],
                      "sm_mhz": line["clocks"].get("sm_mhz"), "reasons": line["clocks"].get("reasons"),
                      "gpu_launches": line["gpu_launches"]}
        except Exception as e:  # pragma: no cover
            res[c] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    return res


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    base = cpu_baseline(args.config, seconds=20.0)
    if base is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdmm_ref.so not built"}))
        return 0
    cfg = workload_config(args.config, world=args.gpus)
    same = True
    if args.config == "cfg2":
        # the reference rejects 32 x 8: the line names the shape that was actually timed
        same = False
        cfg.update({"workload": "general w-way partition w=32, n=512 (32x16: the reference's closest accepted "
                                "general shape; it rejects the 32x8 of cfg2)", "m": 16,
                    "keys_per_gpu": cfg["instances_per_gpu"] * 32 * 16})
    if args.config == "cfg5":
        same = False  # no reference path partitions 2^32 keys; its 8 x 65536 stand-in is timed
        cfg["workload"] += " [reference arm: partition_short_wide on 8x65536 instances as the stand-in]"
    line = {"impl": "reference", "metric": "keys/s", "value": base["value"], "unit": "keys/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "dtype": "u32", "data": "synthetic (reference gen_instance)",
            "config": cfg, "same_shape_as_b200_arm": same, "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end (pinned host) leg")
    ap.add_argument("--no-secondary", action="store_true",
                    help="default run only: skip the device-resident lines of the other configs")
    ap.add_argument("--count", type=int, default=0, help="instances per GPU (default: the config's)")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="pipeline chunks of the end-to-end leg")
    ap.add_argument("--no-graph", action="store_true", help="time the eager launch loop instead of graph replay")
    ap.add_argument("--e2e-streams", type=int, default=3, help="CUDA streams of the end-to-end leg")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="cfg5 exchange: fused scatter into peer buffers (p2p) or multisplit + NCCL all-to-all")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1507_01391_b200 as dmm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU over NCCL; DMM_BENCH_BACKEND=gloo runs the same sharded path with
    # several ranks on one GPU (tests/test_gpu_multiproc.py: no kernel waits on another rank)
    backend = os.environ.get("DMM_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def all_reduce(t, op=dist.ReduceOp.SUM):
        # gloo reduces host tensors; NCCL device tensors
        if world == 1:
            return t
        if backend == "nccl":
            dist.all_reduce(t, op=op)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
        return t

    alg, w, m, count, flags, desc = CONFIGS[args.config]
    if args.count:
        count = args.count
        desc += f" [count overridden: {count}]"
    keys_per_gpu = count * w * m
    if alg == "global_partition":
        # 2^29 keys per GPU viewed as `count` x w x m; keys are splitmix64(global index) >> 32
        g = dmm.gen_keys(rank * keys_per_gpu, keys_per_gpu).view(count, w, m)
    else:
        kind = {"partition_general": dmm.KIND_PARTITION, "integer_sort_general": dmm.KIND_SORT_U32,
                "permute": dmm.KIND_PERMUTE, "partition_short_wide": dmm.KIND_PARTITION,
                "sort_short_wide": dmm.KIND_SORT_U32}[alg]
        # rank r owns instances [r*count, (r+1)*count): seeds are disjoint across ranks
        g = dmm.gen_instances(kind, w, m, 1 + rank * count, count)
    out = torch.empty_like(g)
    stream = torch.cuda.current_stream()

    seeds = np.arange(1 + rank * count, 1 + (rank + 1) * count, dtype=np.uint64)
    perm_bufs = {}
    full_check = None

    def step(src, dst):
        if alg == "partition_general":
            return dmm.partition_general(src, flags=flags, out=dst, check=False)
        if alg == "partition_short_wide":
            return dmm.partition_short_wide(src, out=dst, check=False), None
        if alg == "sort_short_wide":
            return dmm.sort_short_wide(src, out=dst), None
        if alg == "permute":
            return dmm.permute_into(src, dst, seeds, perm_bufs)
        if alg == "global_partition":
            if args.transport == "p2p":
                res, _ = global_partition_p2p(src.view(-1), peers[0])
            else:
                res, _ = global_partition(src.view(-1))
            return res, None
        return dmm.integer_sort_general(src, 1 << 32, out=dst, check=False)

    if alg == "global_partition":
        from paper_1507_01391_b200 import distributed as dmm_dist
        from paper_1507_01391_b200.distributed import PeerBuffers, global_partition, global_partition_p2p, p2p_capacity
        # two receive buffers: the end-to-end leg double-buffers consecutive steps
        peers = [PeerBuffers(p2p_capacity(keys_per_gpu, world)) for _ in range(2)] \
            if args.transport == "p2p" else None

    for _ in range(args.warmup):
        step(g, out)
    torch.cuda.synchronize()
    launches_per_step = int(dmm.lib().dmm_last_launch_count())
    if alg == "global_partition" and args.transport == "p2p":
        launches_per_step = dmm_dist.last_launches

    # The step is one kernel launch; it is captured once into a CUDA graph and the timed loop
    # replays it K times, so host-side stalls cannot starve the GPU between steps (measured:
    # the eager loop's step time varied up to 2x run to run on a shared host).  cfg5's step
    # has a host sync (bucket counts) and stays eager.
    graph = None
    if alg != "global_partition" and not args.no_graph:
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            step(g, out)  # settle allocations on the capture stream
        torch.cuda.current_stream().wait_stream(cap)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            _, st_graph = step(g, out)
        torch.cuda.synchronize()
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident throughput -------------------------------------------------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                _, st = step(g, out)
        e1.record(stream)
        torch.cuda.synchronize()
    if graph is not None:
        st = st_graph
    ms = e0.elapsed_time(e1) / args.steps
    barrier()
    t = all_reduce(torch.tensor([ms], device="cuda"), dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # correctness of the timed output (verify_partition_result instance.hpp:249)
    if alg == "partition_general":
        rows = torch.arange(w, device="cuda", dtype=torch.int32).view(1, w, 1)
        ok = bool((out == rows).all()) and int((st.status != 0).sum()) == 0
    elif alg == "partition_short_wide":
        rows = torch.arange(w, device="cuda", dtype=torch.int32).view(1, w, 1)
        ok = bool((out == rows).all())
    elif alg == "permute":
        exp = torch.arange(w * m, device="cuda", dtype=torch.int32).view(1, w, m)
        ok = bool((out == exp).all())
    elif alg == "global_partition":
        # this rank received exactly the keys whose label it owns (8 labels over `world` ranks),
        # in (source rank, source index) order: the receive buffer is filled with a sentinel
        # first, then compared with the stable order of the same keys (world 1: the stable
        # argsort of the local keys; world > 1: per-label key-sum / XOR checksums all-reduced
        # over the ranks' inputs against what this rank received, plus the total count)
        recv = peers[0].local if args.transport == "p2p" else None
        if recv is not None:
            recv.fill_(-1)
        res, _ = step(g, out)
        torch.cuda.synchronize()
        lab = (res.to(torch.int64) & 0xFFFFFFFF) >> 29
        lo, hi = rank * 8 // world, (rank + 1) * 8 // world
        ok = bool(((lab >= lo) & (lab < hi)).all())
        if world == 1:
            src = g.view(-1).to(torch.int64) & 0xFFFFFFFF
            order = torch.argsort(src >> 29, stable=True)
            ok = ok and bool((res.view(-1).to(torch.int64) & 0xFFFFFFFF).equal(src[order]))
            del src, order
        else:
            srcl = g.view(-1).to(torch.int64) & 0xFFFFFFFF
            lab_in = srcl >> 29
            sums = torch.zeros(8, dtype=torch.int64, device="cuda").index_add_(0, lab_in, srcl)
            cnts = torch.bincount(lab_in, minlength=8)
            all_reduce(sums)
            all_reduce(cnts)
            rl = res.view(-1).to(torch.int64) & 0xFFFFFFFF
            got = torch.zeros(8, dtype=torch.int64, device="cuda").index_add_(0, rl >> 29, rl)
            gotc = torch.bincount(rl >> 29, minlength=8)
            ok = ok and bool((got[lo:hi] == sums[lo:hi]).all()) and bool((gotc[lo:hi] == cnts[lo:hi]).all())
            del srcl, lab_in, rl
        n_recv = all_reduce(torch.tensor([res.numel()], device="cuda", dtype=torch.int64))
        ok = ok and int(n_recv.item()) == keys_per_gpu * world
    else:
        full_check = verify_sort_full(g, out, count)
        ok = full_check["ok"]

    e2e_ms = None
    e2e_count = count
    if not args.no_e2e:
        # ---- end to end through the public API (pinned host in/out) -------------------------
        # chunks cycle over 3 streams: H2D of chunk i+1 || kernel of chunk i || D2H of chunk i-1
        from paper_1507_01391_b200.pipeline import run_pipelined
        # pinned host memory: the whole batch at one GPU; with N ranks on one host each rank's
        # end-to-end batch is capped at 16 GiB / N of input (host memory stays 32 GiB in all)
        e2e_count = count
        if world > 1 and alg != "global_partition":
            e2e_count = max(1, min(count, (16 << 30) // (w * m * 4) // world))
        h_in = g[:e2e_count].cpu().pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()

        perm_slot_bufs = {}

        def chunk_fn(din, dout, s, lo):
            if alg == "partition_general":
                dmm.partition_general(din, flags=flags, out=dout, stream=s, check=False)
            elif alg == "partition_short_wide":
                dmm.partition_short_wide(din, out=dout, stream=s, check=False)
            elif alg == "sort_short_wide":
                dmm.sort_short_wide(din, out=dout, stream=s)
            elif alg == "integer_sort_general":
                dmm.integer_sort_general(din, 1 << 32, out=dout, stream=s, check=False)
            elif alg == "permute":
                bufs = perm_slot_bufs.setdefault((s.cuda_stream, din.shape[0]), {})
                if "seeds" not in bufs:
                    bufs["seeds"] = torch.arange(1 + rank * count + lo, 1 + rank * count + lo + din.shape[0],
                                                 dtype=torch.int64, device="cuda")
                dmm.permute_into(din, dout, None, bufs, stream=s)
            else:
                from paper_1507_01391_b200.distributed import global_partition
                res, _ = global_partition(din.view(-1))
                dout.view(-1).copy_(res)

        ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_steps = max(3, args.steps // 4)
        if alg != "global_partition":
            slots = run_pipelined(chunk_fn, h_in, h_out, chunks=args.e2e_chunks, nstreams=args.e2e_streams)  # warm-up
            torch.cuda.synchronize()
            barrier()
            ee0.record(stream)
            for _ in range(e2e_steps):
                run_pipelined(chunk_fn, h_in, h_out, chunks=args.e2e_chunks, slots=slots)
            ee1.record(stream)
        else:
            # the global partition is bucket-major over the whole batch, so a step is not chunked;
            # consecutive steps are double-buffered instead (two streams, two host result buffers):
            # step i's D2H overlaps step i+1's H2D (PCIe is full duplex)
            e2e_streams = [torch.cuda.Stream(), torch.cuda.Stream()]
            d_in = [torch.empty_like(g) for _ in range(2)]
            # a rank receives the keys of its labels from every rank: up to the receive capacity
            cap = peers[0].capacity if args.transport == "p2p" else p2p_capacity(keys_per_gpu, world)
            h_outs = [torch.empty(cap, dtype=torch.int32).pin_memory() for _ in range(2)]
            d2h_keys = []

            def gp_step(i):
                s = e2e_streams[i % 2]
                with torch.cuda.stream(s):
                    d_in[i % 2].copy_(h_in, non_blocking=True)
                    if args.transport == "p2p":
                        res, _ = global_partition_p2p(d_in[i % 2].view(-1), peers[i % 2])
                    else:
                        res, _ = global_partition(d_in[i % 2].view(-1))
                    h_outs[i % 2].view(-1)[: res.numel()].copy_(res, non_blocking=True)
                    d2h_keys.append(res.numel())

            for i in range(2):  # warm-up
                gp_step(i)
            torch.cuda.synchronize()
            barrier()
            ee0.record(stream)
            for s in e2e_streams:
                s.wait_stream(stream)
            for i in range(e2e_steps):
                gp_step(i)
            for s in e2e_streams:
                stream.wait_stream(s)
            ee1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = ee0.elapsed_time(ee1) / e2e_steps
        t = all_reduce(torch.tensor([e2e_ms], device="cuda"), dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        if alg in ("partition_general", "partition_short_wide"):
            rows = torch.arange(w, dtype=torch.int32).view(1, w, 1)
            ok = ok and bool((h_out == rows).all())
        elif alg == "global_partition":
            # the last end-to-end result in host memory: this rank's labels only, bucket-major
            got = h_outs[(e2e_steps - 1) % 2].view(-1)[: res.numel()]
            lab = (got.to(torch.int64) & 0xFFFFFFFF) >> 29
            ok = ok and bool(((lab >= lo) & (lab < hi)).all())
            if world == 1:
                ok = ok and bool((lab[1:] >= lab[:-1]).all())

    # every rank's verdict (its own instances / received keys), and the seed range each rank
    # generated its instances from (disjoint shards)
    ok = bool(all_reduce(torch.tensor([int(ok)], device="cuda"), dist.ReduceOp.MIN).item())
    seed_ranges = [[1 + r * count, (r + 1) * count] for r in range(world)] if alg != "global_partition" else \
        [[r * keys_per_gpu, (r + 1) * keys_per_gpu] for r in range(world)]
    e2e_keys = e2e_count * w * m
    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary and args.config == "cfg3" and not args.count:
        import gc
        g = out = h_in = h_out = slots = None  # noqa: F841  (release the batch before the children run)
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        secondary = run_secondaries(args)
    if rank == 0:
        peaks, peak_kind = _peaks()
        total_keys = keys_per_gpu * world
        value = total_keys / (ms_max / 1e3)
        bytes_per_launch = keys_per_gpu * 8  # algorithmic: one u32 read + one u32 write per key
        traffic = measured_traffic(args.config, count)
        achieved = bytes_per_launch / (ms / 1e3) / 1e9
        line = {
            "metric": "keys/s", "value": value, "unit": "keys/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (reference gen_instance, on device)",
            "config": workload_config(args.config, world, args.count, graph is not None, args.transport),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"],
                         "traffic": (traffic or {}).get("bytes_per_launch"),
                         "traffic_source": (traffic or {}).get("source"),
                         "peak_source": peak_kind + " (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                         else "fallback 6650 GB/s"},
            "smem": smem_line(traffic, ms),
            "e2e": None if e2e_ms is None else {"value": e2e_keys * world / (e2e_ms / 1e3), "unit": "keys/s",
                    "h2d_bytes_per_step": e2e_keys * 4,
                    "d2h_bytes_per_step": (e2e_keys * 4 if alg != "global_partition"
                                           else int(4 * sum(d2h_keys[-e2e_steps:]) / e2e_steps)),
                    "instances_per_gpu": e2e_count},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "correct": ok,
        }
        if full_check is not None:
            line["full_size_check"] = full_check
        if secondary is not None:
            line["secondary"] = secondary
        line["config"]["shards"] = {"backend": backend if world > 1 else None,
                                    ("seed_ranges" if alg != "global_partition" else "key_index_ranges"): seed_ranges}
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N = 1 only
            try:
                line["cpu_baseline"] = cpu_baseline(args.config)
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"error": str(e)}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
