import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_06443_b200 as v
torch.cuda.init()
for g in (4, 5):
    for w in (8, 12, 16):
        print(g, w, [v.lib().vlut_active_clusters(g, w, s) for s in range(1, 9)])
