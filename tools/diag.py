"""Print the compiled attributes (registers, threads, shared memory) of the hot-path kernels
(te_kernel_attributes); needs a GPU."""
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2205_15346_b200 import te
L = te.load()
for w in range(6):
    r, t, s, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    rc = L.te_kernel_attributes(w, C.byref(r), C.byref(t), C.byref(s), C.byref(d))
    print(w, rc, r.value, t.value, s.value, d.value, L.te_last_error())
