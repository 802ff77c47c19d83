import sys
sys.path.insert(0, '.')
from paper_2605_29727_b200 import _lib
import torch
torch.zeros(1, device='cuda')
lib = _lib.lib()
for cl in (1, 2, 4, 8, 12, 16):
    print(cl, [lib.bst_debug_cluster_occupancy_kt(cl, smem) for smem in (150000, 200000, 221000)])
