"""Multi-process paths on one B200: the only GPU this build gets is one, so
the world-2 runs put both ranks on cuda:0 with a gloo process group.  No kernel of one rank waits
on another rank's kernel (the fused exchange's ordering is a host barrier after a stream sync),
so co-residency on one GPU is safe.
  * the fused cfg5 exchange across two processes: CUDA IPC receive buffers, every rank's scatter
    writing into its owners' buffers, checked key for key against the all-to-all order;
  * bench.py's sharded paths at world 2: disjoint seed ranges, every rank's result checked,
    max-over-ranks timing, n_gpus = 2 in the line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(nproc, script, *args, env=None, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), script, *args]
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=e)
    if r.returncode != 0:  # keep the whole log (torchrun's tail hides the failing rank's trace)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"torchrun_{os.path.basename(script)}_{_port()}.log"), "w") as f:
            f.write(r.stdout + "\n" + r.stderr)
    return r


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_across_processes(world):
    r = _torchrun(world, os.path.join(ROOT, "tests", "mp_p2p_worker.py"))
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert f"P2P_MULTIPROC ok {world}" in r.stdout


@pytest.mark.parametrize("cfg,count", [("cfg1", 4096), ("cfg3", 512), ("cfg4s", 2048), ("cfg5", 1)])
def test_bench_world2_sharded(cfg, count):
    r = _torchrun(2, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", cfg, "--count", str(count),
                  "--steps", "3", "--warmup", "3", "--no-cpu-baseline", env={"DMM_BENCH_BACKEND": "gloo"})
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["correct"] is True and line["value"] > 0
    sh = line["config"]["shards"]
    assert sh["backend"] == "gloo"
    ranges = sh.get("seed_ranges") or sh.get("key_index_ranges")
    assert len(ranges) == 2 and ranges[0][1] <= ranges[1][0]  # disjoint shards
    per_gpu = line["config"]["keys_per_gpu"]
    # value = keys over all ranks / the max-over-ranks step time
    assert abs(line["value"] - 2 * per_gpu / (line["ms_per_step"] / 1e3)) <= 1e-6 * line["value"]
