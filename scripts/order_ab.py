"""A/B of the fused block order: `python scripts/order_ab.py old|new [bench args]`
runs bench.py with the KL=4 block first (new, default) or last (old)."""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_06022_b200 import fusion  # noqa: E402

mode = sys.argv[1]
if mode == "old":
    orig = fusion._blocks

    def _blocks(tids, kind="float32"):
        blocks, plain = orig(tids, kind)
        if blocks and blocks[0].kl == fusion.KL_BASE:
            kls = [b.kl for b in blocks[1:]] + [blocks[0].kl]
            out, i = [], 0
            flat = [t for b in blocks for t in b.tasks]
            for kl in kls:
                out.append(fusion.Block(tuple(flat[i:i + kl]), kl))
                i += kl
            blocks = out
        return blocks, plain
    fusion._blocks = _blocks
sys.argv = ["bench.py"] + sys.argv[2:]
runpy.run_path(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"),
               run_name="__main__")
