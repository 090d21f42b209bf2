"""torchrun helper for tests/test_gpu_multirank.py: cluster.gpu_mul (the
multi-GPU API) with ranks sharing cuda:0 over gloo; rank 0 prints the digest."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1303_7425_b200 import MulConfig, benchpolys, gpu_mul, io  # noqa: E402

dist.init_process_group("gloo")
torch.cuda.set_device(0)
name, kind = sys.argv[1].split("/")
f, g = benchpolys.CONFIGS[name](float if kind == "float" else int)
p = gpu_mul(f, g, MulConfig(float_ordered=kind == "float"))
if dist.get_rank() == 0:
    print(json.dumps({"n": p.n, "sha256": io.poly_digest(p), "type": type(p).__name__}))
dist.barrier()
dist.destroy_process_group()
