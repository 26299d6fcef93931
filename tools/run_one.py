"""Run one codec entry point a few times (for ncu): python tools/run_one.py OP rows cols

OP in: detect, sym, asym, outlier, perchannel, mask, dsym, dasym, doutlier, dperchannel
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200 import _lib  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402

op, rows, cols = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
sp = torch.cuda.current_stream().cuda_stream
x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
x[:, ::97] *= 30
lib = _lib.lib()
specs = {"sym": adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP), "asym": adc.SchemeSpec(adc.Scheme.ASYMMETRIC_GROUP),
         "outlier": adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED),
         "perchannel": adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP, 0), "mask": adc.SchemeSpec(adc.Scheme.BIT_MASK, 0)}
if op == "detect":
    ws_bytes = lib.adc_workspace_bytes(2, rows, cols, 128)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    idx = torch.empty(cols, dtype=torch.int32, device="cuda")
    st = torch.zeros(2, dtype=torch.int32, device="cuda")
    for _ in range(reps):
        lib.adc_detect_outliers(x.data_ptr(), 1, rows, cols, 3.0, cols, idx.data_ptr(), st.data_ptr() + 4,
                                st.data_ptr(), ws.data_ptr(), ws_bytes, sp)
else:
    name = op[1:] if op.startswith("d") and op != "detect" else op
    spec = specs[name]
    if name == "mask":
        x = torch.rand(rows, cols, device="cuda") < 0.9
    s = CodecSlot(rows, cols, spec, x.dtype, torch.uint8 if name == "mask" else torch.bfloat16, k_cap=cols // 8)
    y = torch.empty((rows, cols), dtype=s.out_dtype, device="cuda")
    for _ in range(reps):
        if op.startswith("d"):
            s.compress_ptr(x.data_ptr(), sp)
            s.decompress_ptr(y.data_ptr(), sp)
        else:
            s.compress_ptr(x.data_ptr(), sp)
torch.cuda.synchronize()
