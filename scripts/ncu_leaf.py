"""C5 leaf scan launches (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_18897_b200.device_ops import LeafScanBatch  # noqa: E402
from paper_2603_18897_b200.synth import long_output_corpus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
c = long_output_corpus(n)
b = LeafScanBatch(c["nodes"], c["bytes"], c["refs"], c["target_off"], c["target_bytes"])
for _ in range(3):
    b.launch()
torch.cuda.synchronize()
