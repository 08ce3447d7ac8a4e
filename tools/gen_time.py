import sys, time; sys.path.insert(0, '.')
import torch
from paper_1202_6158_b200 import gen
torch.cuda.set_device(0)
for k in (3, 5):
    t = time.time(); g, rep = gen.baseline_graph(k); torch.cuda.synchronize()
    print(k, time.time() - t, rep, flush=True)
    del g; torch.cuda.empty_cache()
