import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_08713_b200 as P
import oracle

o = oracle
rng = np.random.default_rng(1)
def run(c,h,w,bd,L,rct,noise=True):
    if noise: a = rng.integers(0, 1<<bd, (c,h,w)).astype(np.int64)
    else:
        yy,xx=np.mgrid[0:h,0:w]; a=np.stack([(xx*7+yy*3+k)%(1<<bd) for k in range(c)]).astype(np.int64)
    ref = o.encode_image(a, bd, L, rct)
    got = P.encode_image(P.RasterImage.from_planes(list(a), bd), levels=L, use_rct=rct)
    print((c,h,w,bd,L,rct), "OK" if got==ref else "FAIL", flush=True)
for args in [(1,64,1024,8,2,False),(1,64,1040,8,2,False),(1,32,1040,8,2,False),(1,80,1040,8,2,False),(1,333,1040,8,2,False),(1,64,1032,8,2,False),(1,64,1280,8,2,False),(1,66,1024,8,2,False),(1,70,1024,8,2,False),(3,333,1040,8,4,True),(1,334,1024,8,2,False),(1,333,1024,8,2,False)]:
    run(*args)
