import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests'); sys.path.insert(0,'/root/repo/tests/golden')
import torch
from test_gpu_parity import _bf16_adversarial
from _harness import oracle_run, device_run
xt = _bf16_adversarial(np.random.default_rng(0))
for scheme, group in [(0,16),(0,128),(1,16),(2,128)]:
    want = oracle_run(xt.to(torch.float32).numpy(), scheme, group, 3.0)
    got = device_run(xt, scheme, group, 3.0)
    for k in ("scales","offsets","codes","idx","vals"):
        a, b = got[0][k], want[0][k]
        if a is None or b is None:
            if (a is None) != (b is None): print(scheme, group, k, "none mismatch")
            continue
        d = np.nonzero(a != b)[0]
        if len(d): print(scheme, group, k, len(d), d[:8], a[d[:4]], b[d[:4]])
    dd = np.nonzero(got[1].view(np.uint32) != want[1].view(np.uint32))
    print(scheme, group, "dequant diffs", len(dd[0]), list(zip(dd[0][:5], dd[1][:5])))
    if len(dd[0]):
        r, c = dd[0][0], dd[1][0]
        print("  x", xt[r, c-2:c+3].float().numpy(), "got", got[1][r, c-2:c+3], "want", want[1][r, c-2:c+3])
