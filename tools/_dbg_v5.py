import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch, numpy as np
import paper_2505_18875_b200 as svg2
import svg2_synth
from gpu_helpers import random_qkv, to_dev
wl = svg2_synth.WORKLOADS["tiny"]
q, k, v = svg2_synth.generate(wl, heads=range(2))
Q, K, V = to_dev(q), to_dev(k), to_dev(v)
O, pairs, ex = svg2.sparse_attention(Q, K, V, wl.Cq, wl.Ck, 2, wl.top_p, debug=True)
torch.cuda.synchronize()
print("tiny ok", float(O.float().abs().mean()))
