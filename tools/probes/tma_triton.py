import torch, triton, triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor
print(triton.__version__, torch.cuda.get_device_name())
@triton.jit
def k(desc, out_ptr, BM: tl.constexpr, BN: tl.constexpr):
    t = desc.load([0, 0])
    offs = tl.arange(0, BM)[:, None] * BN + tl.arange(0, BN)[None, :]
    tl.store(out_ptr + offs, t)
x = torch.arange(64*64, device="cuda", dtype=torch.float32).reshape(64, 64)
d = TensorDescriptor.from_tensor(x, [32, 32])
o = torch.empty(32, 32, device="cuda")
k[(1,)](d, o, 32, 32)
torch.cuda.synchronize()
print("triton host-desc TMA ok", torch.equal(o, x[:32, :32]))
a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
print("cublas", (a @ a).float().abs().sum().item() > 0)
