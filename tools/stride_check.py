import sys
sys.path.insert(0, ".")
import torch
from paper_2506_11449_b200.vit import PackedQKVAttention
B,T,H,hd=8,197,12,64
h=torch.randn(B,T,3,H,hd,device="cuda",dtype=torch.bfloat16,requires_grad=True)
out=PackedQKVAttention.apply(h)
print("out", out.shape, out.stride(), out.is_contiguous())
a=out.transpose(1,2)
print("transposed contiguous?", a.is_contiguous(), a.stride())
r=a.reshape(B,T,H*hd)
print("reshape shares storage:", r.data_ptr()==out.data_ptr())
