import sys, time, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import bench
from paper_2603_20009_b200 import api, synth
from paper_2603_20009_b200.config import KMeansConfig
from paper_2603_20009_b200.device import to_device_matrix
from paper_2603_20009_b200.hostmath import generate_rotation
dev = torch.device("cuda", 0)
print("c1 before:", bench.run_extra("c1", dev)["ms_per_fit"], flush=True)
x = torch.randn((1_000_000, 1536), device=dev)
r = api.fit_device(x, 1536, KMeansConfig(k=4096, max_iters=10, seed=0), generate_rotation(1536, 0))
torch.cuda.synchronize()
print("c1 after c2-size fit:", bench.run_extra("c1", dev)["ms_per_fit"], flush=True)
del x, r
torch.cuda.empty_cache()
print("c1 after empty_cache:", bench.run_extra("c1", dev)["ms_per_fit"], flush=True)
