import time, ctypes as C, sys
sys.path.insert(0, '.')
import paper_1911_06001_b200 as vx
t0 = time.perf_counter(); m = vx.Model.procedural(11, shell=True); t1 = time.perf_counter()
print(f"procedural(11) build+upload {1e3*(t1-t0):.1f} ms")
