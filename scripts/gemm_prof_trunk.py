"""Role wait-time breakdown (QPINN_GEMM_PROF build) of the trunk forward's dual-tanh
tcgen05 layers, aggregated over the 4 GEMM launches of qpinn_trunk_forward (CTA 0 each)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS, train_config  # noqa: E402
from paper_2506_23246_b200 import _native as N  # noqa: E402
from paper_2506_23246_b200.training import Trainer  # noqa: E402

tr = Trainer(train_config(WORKLOADS["config2"]["grid"]), device="cuda", dtype=torch.float32,
             graphs=False)
eng = tr.evaluator.engine
lib = N.lib()
prof = lib.qpinn_gemm_prof
prof.argtypes = [C.c_void_p]
ch, b = eng.chunks[0], eng.bufs[0]
flat = tr.flat.detach()


def fwd():
    N.check(lib.qpinn_trunk_forward(C.byref(eng.desc), eng.dcode, b.R, ch.x.data_ptr(),
                                    ch.y.data_ptr(), ch.t.data_ptr(), flat.data_ptr(),
                                    b.act.data_ptr(), eng.trunk_ws.data_ptr(),
                                    eng.trunk_ws.numel(), N.stream_ptr()), "fwd")


fwd()
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
prof(buf)
for _ in range(10):
    fwd()
torch.cuda.synchronize()
prof(buf)
names = ["A prod wait raw_empty", "B prod wait b_empty", "MMA wait tempty", "MMA wait conv",
         "MMA wait b_full", "conv(w0) wait op_empty", "conv(w0) wait raw_full",
         "epi(w4) wait tfull", "epi(w4) store phase"]
tot = buf[9]
print(f"trunk forward GEMMs: {tot / 10:.0f} CTA-0 cycles per forward (4 launches)")
for i, nm in enumerate(names):
    print(f"   {nm:26s} {buf[i] / tot * 100:6.1f} %")
