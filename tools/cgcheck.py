import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
torch.cuda.set_device(0)
x = torch.zeros(10, device="cuda:0")
from bench import load_spec
from paper_1802_00330_b200 import bnb
for name in ["broyden_tri6", "katsura6"]:
    e = bnb.engine_for(load_spec(name), 0)
    print(name, e.codegen_active(), flush=True)
