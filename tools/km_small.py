"""Small k-means run for compute-sanitizer (GPU box): exercises the k-means++ skip update, the
fp32 screen with a <= 32-column tail tile (k = 40) and the exact fallback."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1509_08863_b200 as sc
import scinputs

n, d, k = 30000, 96, 40
F = torch.from_numpy(scinputs.gaussian_block(11, n, d)).cuda()
lab = torch.empty(n, dtype=torch.int32, device="cuda")
os.environ["SC_KMEANS_SCREEN_MIN"] = "1"
res = sc.sc_kmeans(F, n, d, k, 2, 8, 4, None, lab)
torch.cuda.synchronize()
print("kmeans ok", res)
