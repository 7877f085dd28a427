import ctypes as C, sys
sys.path.insert(0, ".")
import torch
from paper_2311_04648_b200 import _lib
order = sys.argv[1] if len(sys.argv) > 1 else "lib_first"
if order == "torch_first":
    torch.zeros(1, device="cuda")
ctx = _lib.Context(0, f32_state=True)
ptr = ctx.L.gf_stream(C.c_void_p(ctx.h))
print("ptr", hex(ptr or 0))
es = torch.cuda.ExternalStream(int(ptr), device=torch.device("cuda", 0))
try:
    es.synchronize(); print(order, "sync ok")
except Exception as e:
    print(order, "sync fail", e)
try:
    with torch.cuda.stream(es):
        x = torch.ones(10, device="cuda") * 2
    torch.cuda.synchronize(); print(order, "use ok", float(x.sum()))
except Exception as e:
    print(order, "use fail", e)
ev = torch.cuda.Event()
try:
    ev.record(es); ev.synchronize(); print(order, "event ok")
except Exception as e:
    print(order, "event fail", e)
