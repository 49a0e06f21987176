import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_00233_b200.rng import standard_normal
x = standard_normal(0, int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20, np.float32); torch.cuda.synchronize(); print("ok", float(x[0]))
