import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_06339_b200 as P
x = torch.randn(int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 512, 512, device="cuda")
P.svdvals_batched(x); torch.cuda.synchronize()
