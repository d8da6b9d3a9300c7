import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2512_06102_b200 as eb
exec(open('scripts/e2e_probe.py').read().split("print(f\"H2D")[0])  # setup + tm()
L = eb.lib()
def mk():
    b = eb.Batch(N, H, W)
    b.set_terrain(t.fuel_class, t.elevation, t.class_veg, t.class_den, 30.0)
    b.set_wind(t.wind_speed, t.wind_direction)
    return b
def runner(b, hin, streams=None):
    def run():
        b.set_key(0, 0, streams=streams)
        eb._lib.check(L.ebl_batch_run(b.handle, hin.data_ptr(), STEPS, h_out.data_ptr()))
    return run
A = mk(); print("A", tm(runner(A, h_in)))
B = mk(); print("B", tm(runner(B, h_in)))
print("A again", tm(runner(A, h_in)))
h2 = torch.from_numpy(init.copy()).pin_memory()
print("A, new pinned input", tm(runner(A, h2)))
print("A, explicit streams", tm(runner(A, h_in, np.arange(N, dtype=np.uint64))))
hb = eb.host_buffer(init.shape); hb[:] = init
class P:  # data_ptr shim
    def __init__(s, a): s.a = a
    def data_ptr(s): return s.a.ctypes.data
print("A, huge-page input", tm(runner(A, P(hb))))
hb2 = eb.host_buffer(init.shape); hb2[:] = init
print("A, huge-page input #2", tm(runner(A, P(hb2))))
ho = eb.host_buffer(init.shape)
def run_h(b, hin, hout):
    def run():
        b.set_key(0, 0)
        eb._lib.check(L.ebl_batch_run(b.handle, hin.ctypes.data, STEPS, hout.ctypes.data))
    return run
print("A, huge-page in + out", tm(run_h(A, hb, ho)))
B.close()
print("A after B closed", tm(runner(A, h_in)))
