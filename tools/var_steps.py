import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1507_01391_b200 as dmm
m = int(sys.argv[1]); count = int(sys.argv[2])
g = dmm.gen_instances(dmm.KIND_PARTITION, 32, m, 1, count)
out = torch.empty_like(g)
for _ in range(5):
    dmm.partition_general(g, out=out, check=False, flags=(dmm.FLAG_EXT_PARTIAL_GROUPS if m == 8 else 0))
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
ev[0].record()
for i in range(40):
    dmm.partition_general(g, out=out, check=False, flags=(dmm.FLAG_EXT_PARTIAL_GROUPS if m == 8 else 0))
    ev[i+1].record()
torch.cuda.synchronize()
t = [ev[i].elapsed_time(ev[i+1]) for i in range(40)]
print(m, 'per-step ms:', ' '.join(f'{x:.3f}' for x in t))
# the bench's exact timed-loop shape: 20 back-to-back steps between two events
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for i in range(20):
    dmm.partition_general(g, out=out, check=False, flags=(dmm.FLAG_EXT_PARTIAL_GROUPS if m == 8 else 0))
e1.record()
torch.cuda.synchronize()
print(m, 'bench-shape loop ms/step:', e0.elapsed_time(e1) / 20)
