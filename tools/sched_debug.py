import faulthandler, sys
faulthandler.dump_traceback_later(40, exit=True)
import torch
import paper_1507_01391_b200 as dmm
from paper_1507_01391_b200 import schedule as S
grid = torch.arange(8, dtype=torch.int32, device="cuda").reshape(1, 4, 2)
keep = torch.full((1, 4, 2), -7, dtype=torch.int32, device="cuda")
cases = [S.Schedule([[S.Move(0, 0, 1, 0), S.Move(0, 1, 2, 0)]]), S.Schedule([[S.Move(0, 0, 1, 0), S.Move(2, 1, 1, 1)]]),
         S.Schedule([[S.Move(0, 0, 1, 0)], [S.Move(0, 2, 1, 0)]]), S.Schedule([[S.Move(i % 4, 0, i % 4, 1) for i in range(5)]])]
for i, bad in enumerate(cases):
    print("case", i, flush=True)
    try:
        S.apply_schedule(grid, bad, out=keep.clone())
        print("no raise", flush=True)
    except Exception as e:
        print("raised", type(e).__name__, e, flush=True)
    torch.cuda.synchronize()
print("done")
