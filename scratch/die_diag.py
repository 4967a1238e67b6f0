import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
t, info = hotpath.die_map(dev)
print(info, "".join(str(int(v)) for v in t.cpu()))
