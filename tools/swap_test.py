import sys, os
sys.path.insert(0, '/root/repo')
import paper_2410_00233_b200.lowrank as L
from paper_2410_00233_b200 import device as D
orig = L._bases
def swapped(cap, mbar, nbar, dtype):
    key = L._bases_key(cap, mbar, nbar, dtype)
    hit = L._BASES.get(key)
    if hit is None:
        q = D.empty((cap, nbar), dtype); s = D.empty((cap, mbar), dtype)
        hit = (s, q); L._BASES[key] = hit
    return hit
L._bases = swapped
sys.argv = ['x', '1024']
exec(open('/root/repo/tools/one_egkb.py').read())
