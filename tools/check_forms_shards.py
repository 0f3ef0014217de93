"""Far-field formulations against each other at large N: the default (fused narrow rows) and
far_rowsum=0 results, and the 8-way pair split against the one-GPU result, at N = 2^22 and 2^24.

    python tools/check_forms_shards.py
"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1501_01652_b200 as fh
from paper_1501_01652_b200 import _lib, _device
from paper_1501_01652_b200.schlomilch import _grid_cache, _grid_lock
def setopt(k,v):
    _lib.check(_lib.load().fhtb_set_option(k,int(v)))
    with _grid_lock: _grid_cache.clear()
for lg in (22, 24):
    n=2**lg
    C = torch.from_numpy(np.random.default_rng(24).standard_normal((1, n))).cuda()
    params = fh.select_params(0, n, 1e-15)
    sc = fh.build_partition(params)
    print(lg, 'M', params.m_terms, sc.blocks)
    res={}
    for rs in (0,2):
        setopt(b"far_rowsum", rs)
        full = fh.schlomilch_fast(params, C)
        tot = torch.zeros_like(full)
        for r in range(8):
            with _device.sharding(r, 8):
                tot += fh.schlomilch_fast(params, C)
        res[rs]=(full,tot)
        d=(tot-full).abs()
        i=int(d.argmax())
        print(' rowsum',rs,'shard-vs-full max', float(d.max()), 'at row', i+1, 'full', float(full.flatten()[i]))
    d=(res[2][0]-res[0][0]).abs(); i=int(d.argmax()); print(' full2 vs full0', float(d.max()), 'row', i+1)
    d=(res[2][1]-res[0][0]).abs(); i=int(d.argmax()); print(' shards2 vs full0', float(d.max()), 'row', i+1)
    print(' tol 2e-15*l1', 2e-15*float(C.abs().sum()))
