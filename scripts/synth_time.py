import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, paper_2512_06102_b200 as eb
for (n,h,w) in [(1024,128,128),(1,16384,16384)]:
    b=eb.Batch(n,h,w)
    b.synth_terrain(0); b.sync()
    t0=time.time(); b.synth_terrain(0); b.synth_ignitions(0, 5 if n>1 else 64); b.sync(); dt=time.time()-t0
    print(f"device synth {n}x{h}x{w}: {dt*1e3:.1f} ms", flush=True)
    b.close()
t0=time.time(); t=eb.synth_terrain(0,1024,128,128); print("host synth C1", time.time()-t0)
