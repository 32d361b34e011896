import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2202_11819_b200.dist import ThreadGroup
T0 = time.time()
def log(*a):
    print(f"{time.time()-T0:8.3f}", *a, flush=True)

def case(G, grid, odf, variant, launch, exchange, n):
    def body(rank):
        t = time.time(); ctx = G.create(rank, grid, odf=odf, variant=variant, launch=launch, exchange=exchange)
        tc = time.time() - t; t = time.time()
        ctx.init("hash", seed=3); ti = time.time() - t; t = time.time()
        ctx.iterate(n); tq = time.time() - t; t = time.time()
        ctx.synchronize(); ts = time.time() - t; t = time.time()
        g = ctx.gather_local(); tg = time.time() - t; t = time.time()
        ck = ctx.checksum(); tk = time.time() - t; t = time.time()
        ctx.close(); tx = time.time() - t
        return f"r{rank} create {tc:.3f} init {ti:.3f} iter {tq:.3f} sync {ts:.3f} gather {tg:.3f} ck {tk:.3f} close {tx:.3f}"
    t = time.time()
    out = G.run(body)
    log(variant, launch, exchange, n, f"total {time.time()-t:.3f}")
    for o in out: log("   ", o)

G = ThreadGroup(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
g = (48, 40, 64)
log("start")
case(G, g, 4, "direct", "batched", "p2p", 9)
case(G, g, 4, "direct", "batched", "p2p", 9)
case(G, g, 4, "direct", "batched", "host", 9)
case(G, g, 4, "direct", "persistent", "p2p", 9)
case(G, g, 4, "unfused", "per_block", "p2p", 9)
