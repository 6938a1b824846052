"""Throughput of apply_schedule (offline schedule of one fixed random permutation applied to a
batch of machines) -- algorithmic bytes = 8 per word (read + write), CUDA events, L2 flushed
between launches by the input size (>= 256 MiB)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1507_01391_b200 as dmm  # noqa: E402
from paper_1507_01391_b200 import schedule as S  # noqa: E402

res = []
for W, M, count in [(32, 32, 1 << 16), (32, 64, 1 << 15), (16, 8, 1 << 19), (32, 8, 1 << 18)]:
    rng = np.random.default_rng(1)
    lin = rng.permutation(W * M)
    s = S.offline_schedule(W, M, np.stack([lin // M, lin % M], 1)).upload()
    g = torch.randint(-2 ** 31, 2 ** 31 - 1, (count, W, M), dtype=torch.int32, device="cuda")
    out = torch.empty_like(g)
    for _ in range(3):
        S.apply_schedule(g, s, out=out, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        S.apply_schedule(g, s, out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    words = count * W * M
    res.append({"shape": f"{W}x{M}", "count": count, "ms": round(ms, 4), "G_words_per_s": round(words / ms / 1e6, 2),
                "GB_per_s": round(8 * words / ms / 1e6, 1)})
    print(json.dumps(res[-1]), flush=True)
