import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1602_06589_b200 import configs
from paper_1602_06589_b200.factorized import build_hs_factorized_device
inst = configs.make_instance(sys.argv[1] if len(sys.argv) > 1 else "C2")
for _ in range(3):
    build_hs_factorized_device(inst.spec, inst.tmats)
torch.cuda.synchronize()
