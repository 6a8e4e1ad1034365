"""Small end-to-end fits for compute-sanitizer runs (tools/sanitize_small.py covers more)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_20009_b200 as skb  # noqa: E402
from paper_2603_20009_b200.synth import make_blobs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
k = int(sys.argv[3]) if len(sys.argv) > 3 else 64
x = make_blobs(n, d, max(2, k // 2), 0)
res = skb.fit(x, skb.KMeansConfig(k=k, max_iters=4, seed=0))
print("ok", [s.d_prime for s in res.stats], [s.survivors for s in res.stats])
