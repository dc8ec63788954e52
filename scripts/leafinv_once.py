"""One 64x64 leaf inverse through the C ABI (ncu target / latency check)."""
import sys, ctypes as C, torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import _capi
lib = _capi.load()
torch.manual_seed(0)
A = (torch.randn(64, 64, dtype=torch.float64) + 8 * torch.eye(64, dtype=torch.float64)).cuda()
X = torch.empty_like(A)
sing = C.c_int()
for _ in range(3):
    lib.acr_leaf_inverse(64, C.c_void_p(A.data_ptr()), C.c_void_p(X.data_ptr()), C.byref(sing), None)
torch.cuda.synchronize()
print("err", float((X @ A - torch.eye(64, dtype=torch.float64, device="cuda")).abs().max()))
