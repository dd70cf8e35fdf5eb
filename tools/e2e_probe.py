# e2e breakdown on C2: pinned D2H bandwidth, generate_into with / without poses.
import ctypes as C, statistics, sys, time
sys.path.insert(0, ".")
import torch
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import scenes

dev = torch.zeros(53 * 2**20 // 8, dtype=torch.float64, device="cuda")
host = torch.empty_like(dev, device="cpu").pin_memory()
for _ in range(3):
    host.copy_(dev, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
print("pinned D2H GB/s %.1f" % (10 * dev.numel() * 8 / (time.perf_counter() - t) / 1e9))
sc = scenes.tabletop_mixed(16384)
eng = pkg.Engine(sc)
P, n = len(sc.placements), 16384
acc = torch.empty((P, n), dtype=torch.int16).pin_memory()
valid = torch.empty(n, dtype=torch.uint8).pin_memory()
poses = torch.empty((P, n, 16), dtype=torch.float64).pin_memory()
A = pkg._capi
full = A.sb_result(C.cast(acc.data_ptr(), C.POINTER(C.c_int16)), C.cast(poses.data_ptr(), C.POINTER(C.c_double)),
                   C.cast(valid.data_ptr(), C.POINTER(C.c_uint8)))
nop = A.sb_result(C.cast(acc.data_ptr(), C.POINTER(C.c_int16)), None, C.cast(valid.data_ptr(), C.POINTER(C.c_uint8)))
for name, res in (("no poses", nop), ("full", full), ("no poses", nop), ("full", full)):
    ms = []
    for _ in range(7):
        torch.cuda.synchronize()
        t = time.perf_counter()
        eng.generate_into(1, res)
        ms.append((time.perf_counter() - t) * 1e3)
    tot, _, _ = eng.last_timing()
    print(name, "wall ms median %.3f min %.3f, device total %.3f" % (statistics.median(ms), min(ms), tot))
for _ in range(3):
    t = time.perf_counter(); eng.generate(1, with_poses=False, download=False); w = (time.perf_counter() - t) * 1e3
    print("no download wall %.3f device %.3f" % (w, eng.last_timing()[0]))
