"""3xTF32 MN-major B diagnostic: C statistics for CQ_TF32_MNB=1 / 0 and the 1-SM path."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2505_06022_b200 import _native as N  # noqa: E402

N.call("cq_init_device", 0)
m, n, k = 512, 384, 256
g = torch.Generator(device="cuda").manual_seed(8)
a = torch.rand((m, k), device="cuda", generator=g) * 2 - 1
b = torch.rand((k, n), device="cuda", generator=g) * 2 - 1
ref = a.double().cpu().numpy() @ b.double().cpu().numpy()
for env in ({"CQ_TF32_MNB": "1"}, {"CQ_TF32_MNB": "0"}, {"CQ_TF32_2SM": "0"}):
    for kk in ("CQ_TF32_MNB", "CQ_TF32_2SM"):
        os.environ.pop(kk, None)
    os.environ.update(env)
    c = torch.full((m, n), float("nan"), device="cuda")
    torch.cuda.synchronize()
    N.call("cq_sgemm", 0, 0, 1, ctypes.c_void_p(a.data_ptr()), k, ctypes.c_void_p(b.data_ptr()), n,
           ctypes.c_void_p(c.data_ptr()), n, m, n, k)
    N.call("cq_stream_synchronize", 0, 0)
    x = c.cpu().numpy()
    print(env, "zeros", int((x == 0).sum()), "nan", int(np.isnan(x).sum()), "max|c|", float(np.nanmax(np.abs(x))),
          "max err", float(np.nanmax(np.abs(x - ref))), flush=True)
    # which columns / rows are nonzero
    nz = np.abs(x) > 0
    print("   nonzero rows", np.where(nz.any(1))[0][:5], "cols", np.where(nz.any(0))[0][:8], flush=True)
