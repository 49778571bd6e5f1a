import sys; from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch, ctypes, json
from paper_2510_16028_b200.executor import inject_drift
cudart = ctypes.CDLL("libcudart.so.12") if False else None
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/reps
res={}
for n in (8<<20, 16<<20, 134<<20):
    y=torch.randn(n, device="cuda"); out=torch.empty_like(y)
    b=8.0*n
    res[n]={"inject_copy": round(b/t(lambda: inject_drift(y,0,0,0.0,0))/1e6,0),
            "inject_drift16": round(b/t(lambda: inject_drift(y,1,16,0.0,0))/1e6,0),
            "torch_clone": round(b/t(lambda: y.clone())/1e6,0),
            "copy_into": round(b/t(lambda: out.copy_(y))/1e6,0)}
print(json.dumps(res))
