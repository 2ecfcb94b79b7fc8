"""Cycles per batch of the chain warp's fold in isolation (int32 min), C2 masks."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_01938_b200 as pd
inst = pd.generate_sdp(n=1 << 20, k=1024, seed=1, a1_cap=4096)
hi = m32 = 0
for a in inst.offsets:
    if 32 <= a < 64: hi |= 1 << (a - 32)
    elif a < 32: m32 |= 1 << a
print("offsets<64:", [int(a) for a in inst.offsets if a < 64])
L = pd.lib(); L.pipedp_chain_fold_cycles.argtypes = [C.c_uint32, C.c_uint32, C.c_int32, C.POINTER(C.c_double)]
for mode, nm in [(0, "full"), (1, "chain only"), (2, "pre only")]:
    c = C.c_double(); L.pipedp_chain_fold_cycles(hi, m32, mode, C.byref(c)); print(nm, c.value)
for (h, m, nm) in [(0xffffffff, 0xfffffffe, "all offsets<64"), (0, 2, "only offset 1")]:
    c = C.c_double(); L.pipedp_chain_fold_cycles(h, m, 0, C.byref(c)); print(nm, c.value)
