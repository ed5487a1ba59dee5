import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, ctypes
from paper_2202_07258_b200 import batched as B, _native as nat
from paper_2202_07258_b200.generate import batched_rhs, bump_dictionary
from paper_2202_07258_b200.solvers import auto_step_size
a = bump_dictionary(200, 5000); Y, _ = batched_rhs(a, 100000)
dev = torch.device("cuda")
a_dev = torch.from_numpy(a).to(dev); y_dev = torch.from_numpy(np.ascontiguousarray(Y)).to(dev)
eta = auto_step_size(a, 1.0)
for i in range(3):
    B.solve_batched(a_dev, y_dev, passes=10, rounds=1, gap_tol=1e-6, eta=eta, return_device=True)
torch.cuda.synchronize()
# stage timing (replicates solve_batched)
L = nat.lib()
def T():
    torch.cuda.synchronize(); return time.perf_counter()
for rep in range(2):
    t0 = T()
    m, n = a_dev.shape; K = y_dev.shape[1]; lda = m + (m % 2)
    a2 = torch.zeros((n, lda), dtype=torch.float64, device=dev); a2[:, :m].copy_(a_dev.t())
    y2 = y_dev.t().contiguous().to(dev, torch.float64)
    t1 = T()
    nbytes = L.bx_batched_workspace_bytes(m, n, K); ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    t2 = T()
    h = ctypes.c_void_p(); stream = torch.cuda.current_stream(dev)
    L.bx_batched_create(ctypes.byref(h), m, n, K, a2.data_ptr(), lda, y2.data_ptr(), m, ws.data_ptr(), nbytes, stream.cuda_stream)
    t3 = T()
    out = nat.BatchedOut(); trace = np.zeros((1, 4))
    L.bx_batched_run(h, float(eta), 10, 1, 1, 1e-6, trace.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 1, ctypes.byref(out))
    t4 = T()
    x = torch.empty((K, n), dtype=torch.float64, device=dev); stats = torch.empty((5, K), dtype=torch.float64, device=dev)
    L.bx_batched_get(h, x.data_ptr(), n, stats.data_ptr())
    t5 = T()
    L.bx_batched_destroy(h); st = stats.cpu().numpy()
    t6 = T()
    print("prep %.2f ws %.2f create %.2f run %.2f (kernel %.2f) get %.2f destroy+stats %.2f ms" % tuple(1e3 * v for v in (t1 - t0, t2 - t1, t3 - t2, t4 - t3, out.round_kernel_ms / 1e3, t5 - t4, t6 - t5)))
