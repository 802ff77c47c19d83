import sys
sys.path.insert(0, '.')
from paper_2605_29727_b200 import _lib
import torch
torch.zeros(1, device='cuda')
lib = _lib.lib()
for cl in (2, 4, 8, 12, 16):
    for smem in (100000, 150000, 197000):
        print(cl, smem, lib.bst_debug_cluster_occupancy(cl, smem), lib.bst_last_error() if hasattr(lib,'bst_last_error') else '')
