"""Check that addmm(out_dtype=f32, out=x) accumulates in place (no DtoD copy)."""
import torch
from torch.profiler import profile, ProfilerActivity
x = torch.randn(4096, 4096, device="cuda")
a = torch.randn(4096, 4096, device="cuda").bfloat16()
w = torch.randn(4096, 4096, device="cuda").bfloat16()
ref = x + a.float() @ w.float()
ptr = x.data_ptr()
torch.addmm(x, a, w, out_dtype=torch.float32, out=x)
torch.cuda.synchronize()
print("in-place:", x.data_ptr() == ptr, "max rel err", ((x - ref).abs().max() / ref.abs().max()).item())
with profile(activities=[ProfilerActivity.CUDA]) as p:
    torch.addmm(x, a, w, out_dtype=torch.float32, out=x)
    torch.cuda.synchronize()
print([e.name for e in p.events() if e.device_type.name == "CUDA"][:6])
