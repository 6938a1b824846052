"""One launch of a bench config's dominant kernel on pre-generated inputs (for ncu A/B runs):
    python tools/one_launch.py cfg1|cfg3
The library is the in-tree build unless DMM_B200_LIB names a variant (paper_1507_01391_b200/_lib.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1507_01391_b200 as dmm  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    if cfg == "cfg1":
        g = dmm.gen_instances(dmm.KIND_PARTITION, 32, 32, 1, 1 << 16)
        dmm.partition_general(g, check=False)
    elif cfg == "cfg3":
        g = dmm.gen_instances(dmm.KIND_SORT_U32, 32, 128, 1, 1 << 18)
        dmm.integer_sort_general(g, 1 << 32, check=False)
    torch.cuda.synchronize()
    print("ok", cfg, os.environ.get("DMM_B200_LIB", "in-tree"))


if __name__ == "__main__":
    main()
