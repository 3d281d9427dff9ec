import sys, json, time
sys.path.insert(0, '.')
import torch
import bench, paper_1112_5239_b200 as P
torch.cuda.set_device(0)
r = bench.measure_c1(P, torch, torch.device('cuda'), False)  # no oracle outside tests/bench
print(json.dumps(r))
