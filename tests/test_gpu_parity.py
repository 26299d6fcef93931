"""Parity of the CUDA path (through the C-ABI) with the reference.

Bit-exact on codes, scales, offsets, outlier index sets and outlier values;
bit-exact on the float32 decompression (dequantisation is one
rounding of an exact product, so float32 equality is achievable and tested
bitwise).  Evidence layers:
  * small_golden.npz -- reference outputs of KATs, 240 ragged random cases and
    the adversarial asymmetric tie families;
  * digests.json     -- reference digests of config-1 tensors (5 seeds x 4
    codecs), Llama-shaped 4096^2 and acceptance gates 2 and 9;
  * the oracle       -- on bf16 / f16 inputs, big-magnitude sums (>= 2^29,
    numpy's sequential order matters) and full BASELINE-size tensors.
"""

import numpy as np
import pytest

import cases
from _harness import (assert_matches_golden, device_run, load_digests, load_small, oracle_run,
                      small_inputs)

pytestmark = pytest.mark.gpu

SMALL = load_small()
INPUTS = small_inputs()
DIGESTS = load_digests()


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    torch.cuda.init()
    return torch


@pytest.mark.parametrize("name", sorted(SMALL))
def test_small_golden(torch_cuda, name):
    x, s, g, t = INPUTS[name]
    norm, deq = device_run(x, s, g, t)
    assert_matches_golden(name, SMALL[name], norm, deq)


@pytest.mark.parametrize("key", sorted(k for k in DIGESTS if k.startswith("config1/")))
def test_config1_digest(torch_cuda, key):
    _, s, g, seed = key.split("/")
    scheme, group, seed = int(s[1:]), int(g[1:]), int(seed[4:])
    x = cases.config1_input(scheme, seed)
    norm, deq = device_run(x, scheme, group, 3.0)
    assert not isinstance(norm, str), norm
    assert cases.norm_digest(norm, deq) == DIGESTS[key]


@pytest.mark.parametrize("seed", [0, 1])
def test_llama_digest(torch_cuda, seed):
    x = cases.llama_input(seed)
    for dt in (None, torch_cuda.bfloat16):   # the input is bf16-valued: both dtypes must agree
        norm, deq = device_run(x, cases.OUTL, 128, 3.0, in_dtype=dt)
        assert norm["idx"].size == DIGESTS[f"llama4096/outl/seed{seed}/k"]
        assert cases.norm_digest(norm, deq) == DIGESTS[f"llama4096/outl/seed{seed}"]


def test_gate2_digests(torch_cuda):
    parts = {"sym16": [], "asym16": [], "pc": [], "outl16": [], "mask": []}
    for x, hot, mask in cases.gate2_inputs():
        for key, (arr, s, g) in {
            "sym16": (x, cases.SYM, 16), "asym16": (x, cases.ASYM, 16),
            "pc": (x, cases.SYM, cases.PER_CHANNEL), "outl16": (hot, cases.OUTL, 16),
            "mask": (mask, cases.MASK, 0),
        }.items():
            norm, deq = device_run(arr, s, g, 3.0)
            parts[key].append(cases.norm_digest(norm, deq))
    for key, lst in parts.items():
        assert cases.digest(np.array(lst)) == DIGESTS[f"gate2/{key}"], key


def test_gate9_digest(torch_cuda):
    import paper_2508_00806_b200 as adc
    flagged = [",".join(str(i) for i in adc.detect_outlier_channels(x).cpu().tolist())
               for x in cases.gate9_inputs()]
    assert cases.digest(np.array(flagged)) == DIGESTS["gate9/flagged"]


@pytest.mark.parametrize("dtype_name", ["bfloat16", "float16"])
@pytest.mark.parametrize("scheme,group", [(0, 128), (0, 0), (1, 128), (2, 128), (0, 64), (1, 32)])
def test_half_inputs_vs_oracle(torch_cuda, dtype_name, scheme, group):
    """bf16/f16 activations: the oracle sees the same values as float32."""
    torch = torch_cuda
    dt = getattr(torch, dtype_name)
    rng = np.random.default_rng(11)
    x = rng.normal(size=(512, 1024)).astype(np.float32)
    x[:, rng.choice(1024, 6, replace=False)] *= 40.0
    xt = torch.from_numpy(x).to(dt)
    x_exact = xt.to(torch.float32).numpy()
    want = oracle_run(x_exact, scheme, group, 3.0)
    got = device_run(xt, scheme, group, 3.0)
    assert cases.norm_digest(*got) == cases.norm_digest(*want)


def test_big_sums_sequential_order(torch_cuda):
    """Column |x|-sums >= 2^29: numpy's row order decides rounding (sequential fallback)."""
    rng = np.random.default_rng(3)
    x = (rng.uniform(40000, 65000, size=(16384, 64)) * rng.choice([-1, 1], size=(16384, 64))).astype(np.float32)
    x[:, 5] = 65504.0
    x[:, 9] *= 0.001
    want = oracle_run(x, cases.OUTL, 128, 1.0)
    got = device_run(x, cases.OUTL, 128, 1.0)
    assert cases.norm_digest(*got) == cases.norm_digest(*want)
    import paper_2508_00806_b200 as adc
    from oracle import codec_oracle as orc
    sums = adc.channel_abs_sums(x).cpu().numpy()
    np.testing.assert_array_equal(sums.view(np.uint64),
                                  orc.column_abs_sums(orc.to_f16_matrix(x)).view(np.uint64))


@pytest.mark.parametrize("shape,scheme,group", [
    ((8192, 1024), 2, 128), ((8192, 3072), 0, 0), ((8192, 4096), 2, 128),
    ((16384, 1024), 1, 128), ((4096, 11008), 2, 128), ((32768, 1024), 3, 0)])
def test_baseline_sizes_vs_oracle(torch_cuda, shape, scheme, group):
    """Full configs[1]/[2] tensor sizes, bf16, against the oracle on the same values."""
    torch = torch_cuda
    rng = np.random.default_rng(shape[0] + shape[1] + scheme)
    if scheme == 3:
        x = (rng.random(size=shape) < 0.9).astype(np.uint8)
        xt = torch.from_numpy(x).to(torch.bool)
        want = oracle_run(x, scheme, group, 3.0)
    else:
        x = rng.standard_normal(size=shape, dtype=np.float32)
        if scheme == 1:
            x = np.abs(x) * 3.0
        hot = rng.choice(shape[1], max(1, shape[1] // 100), replace=False)
        x[:, hot] *= 30.0
        xt = torch.from_numpy(x).to(torch.bfloat16)
        want = oracle_run(xt.to(torch.float32).numpy(), scheme, group, 3.0)
    got = device_run(xt, scheme, group, 3.0)
    assert cases.norm_digest(*got) == cases.norm_digest(*want)


@pytest.mark.parametrize("out", ["bfloat16", "float16"])
def test_reduced_precision_outputs(torch_cuda, out):
    """Training-mode outputs are the float32 reconstruction rounded RNE."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.normal(size=(1024, 768)).astype(np.float32)).cuda()
    x[:, 3] *= 60
    for spec in (adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP), adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP, 0),
                 adc.SchemeSpec(adc.Scheme.ASYMMETRIC_GROUP), adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)):
        ct = adc.compress(x, spec)
        f32 = adc.decompress(ct)
        low = adc.decompress(ct, out_dtype=getattr(torch, out))
        assert torch.equal(low, f32.to(getattr(torch, out)))


def test_async_record_matches_parity_record(torch_cuda):
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    rng = np.random.default_rng(9)
    x = torch.from_numpy(rng.normal(size=(2048, 1024)).astype(np.float32)).cuda().to(torch.bfloat16)
    x[:, 17] *= 80
    spec = adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)
    ref = adc.compress(x, spec)
    ct = adc.compress_async(x, spec, k_cap=64)
    out = torch.empty((2048, 1024), dtype=torch.bfloat16, device="cuda")
    adc.decompress_into(ct, out)
    torch.cuda.synchronize()
    assert int(ct.k_dev[1]) == ref.outlier_count
    assert torch.equal(out, adc.decompress(ref).to(torch.bfloat16))
    assert torch.equal(ct.packed_codes, ref.packed_codes)


def test_k_cap_overflow_is_reported(torch_cuda):
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    rng = np.random.default_rng(10)
    x = torch.from_numpy(rng.normal(size=(256, 512)).astype(np.float32)).cuda()
    x[:, :6] *= 100
    ct = adc.compress_async(x, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), k_cap=2)
    from paper_2508_00806_b200.errors import ERR_K_CAP
    err, k = ct.k_dev.cpu().tolist()
    assert k == 6 and (err & ERR_K_CAP)


def test_errors_map_to_reference_types(torch_cuda):
    import paper_2508_00806_b200 as adc
    with pytest.raises(adc.NonFiniteInputError):
        adc.quantize_symmetric(np.array([1.0, np.nan], np.float32))
    with pytest.raises(adc.NonFiniteInputError):
        adc.compress_outlier_separated(np.array([[1.0, 1e6], [2.0, 3.0]], np.float32))
    with pytest.raises(adc.TooManyOutliersError):
        adc.compress_outlier_separated(np.array([[1000.0, 1000.0, 1.0]] * 4, np.float32), threshold=0.1)
    with pytest.raises(adc.NonBinaryMaskError):
        adc.pack_bitmask(np.array([0, 2, 1], np.uint8))
    with pytest.raises(adc.ValidationError):
        adc.quantize_symmetric(np.ones((2, 2, 2), np.float32))
    with pytest.raises(adc.ValidationError):
        adc.quantize_symmetric(np.ones(8, np.float32), group_size=-2)


@pytest.mark.parametrize("spec_args", [(0, 128), (0, 0), (1, 32), (2, 128), (3, 0)])
def test_wire_format_matches_oracle_bytes(torch_cuda, spec_args):
    """serialize(device record) == the oracle's ADC1 bytes; deserialize round-trips."""
    import paper_2508_00806_b200 as adc
    from oracle import codec_oracle as orc
    s, g = spec_args
    rng = np.random.default_rng(6)
    x = rng.normal(size=(16, 256)).astype(np.float32)
    if s == 3:
        x = (x > 0).astype(np.float32)
    if s == 2:
        x[:, 17] *= 90.0
    ct = adc.compress(x, adc.SchemeSpec(adc.Scheme(s), g))
    blob = adc.serialize(ct)
    assert blob == orc.serialize(orc.compress(x, s, g))
    back = adc.deserialize(blob)
    assert adc.serialize(back) == blob
    assert np.array_equal(adc.decompress(back).cpu().numpy(), adc.decompress(ct).cpu().numpy())


def _bf16_adversarial(rng, rows=256, cols=512):
    """bf16-representable values that stress the native bf16 path."""
    import torch
    x = rng.normal(size=(rows, cols)).astype(np.float32)
    x[:, 0:8] *= 1e-6          # tiny values needing f16 subnormal rounding
    x[:, 8:16] = rng.choice([0.0, 2 ** -20, -(2 ** -18), 3 * 2 ** -22], size=(rows, 8))
    x[0:4, :] *= 1e-7          # whole tiny groups (row-major groups of 128)
    x[4:8, :] = np.round(x[4:8, :] * 8) / 8   # exact ties for power-of-two scales
    x[8:12, 100:110] = 65280.0                # largest finite-after-cast bf16
    return torch.from_numpy(x).to(torch.bfloat16)


@pytest.mark.parametrize("scheme,group", [(0, 128), (0, 16), (0, 256), (1, 128), (1, 16), (2, 128), (0, 0)])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_bf16_native_path_adversarial(torch_cuda, scheme, group, seed):
    torch = torch_cuda
    xt = _bf16_adversarial(np.random.default_rng(seed))
    want = oracle_run(xt.to(torch.float32).numpy(), scheme, group, 3.0)
    got = device_run(xt, scheme, group, 3.0)
    assert cases.norm_digest(*got) == cases.norm_digest(*want)


def test_bf16_asym_tie_families(torch_cuda):
    """The Appendix A.5 tie families are bf16-exact: run them natively in bf16."""
    torch = torch_cuda
    for name, x, s, g, t in cases.tie_family_cases():
        xt = torch.from_numpy(x).to(torch.bfloat16)
        want = oracle_run(xt.to(torch.float32).numpy(), s, g, t)
        got = device_run(xt, s, g, t)
        assert cases.norm_digest(*got) == cases.norm_digest(*want), name


def test_bf16_overflow_is_nonfinite(torch_cuda):
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    x = torch.ones(4, 256, dtype=torch.bfloat16)
    x[2, 7] = 65536.0  # rounds to f16 inf (codec.py:167-170)
    for spec in (adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP), adc.SchemeSpec(adc.Scheme.ASYMMETRIC_GROUP),
                 adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP, 0)):
        with pytest.raises(adc.NonFiniteInputError):
            adc.compress(x, spec)


@pytest.mark.parametrize("shape", [(64, 768), (8192, 768), (1000, 1000), (4096, 4096), (2048, 11008),
                                   (333, 1024), (8192, 1024), (3, 20000)])
@pytest.mark.parametrize("dtype_name", ["bfloat16", "float32"])
def test_outlier_separated_wide_shapes(torch_cuda, shape, dtype_name):
    """K4 at layer widths and ragged row counts (full-wave column reduction, heap tree, gather)."""
    torch = torch_cuda
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    x = rng.normal(size=shape).astype(np.float32)
    hot = rng.choice(shape[1], max(1, shape[1] // 64), replace=False)
    x[:, hot] *= rng.uniform(10, 60)
    xt = torch.from_numpy(x).to(getattr(torch, dtype_name))
    want = oracle_run(xt.to(torch.float32).numpy(), cases.OUTL, 128, 3.0)
    got = device_run(xt, cases.OUTL, 128, 3.0)
    assert cases.norm_digest(*got) == cases.norm_digest(*want)


@pytest.mark.parametrize("scheme,group", [(cases.OUTL, 128), (cases.ASYM, 128), (cases.SYM, 0)])
def test_graph_replay_matches_eager(torch_cuda, scheme, group):
    """bench.py times CUDA-graph replays of the codec calls: replays (which
    reuse the self-resetting workspace) must reproduce the eager bytes."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200.slots import CodecSlot
    rows, cols = 2048, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    xs = [torch.randn(rows, cols, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2)]
    for x in xs:
        x[:, ::97] *= 40
    spec = adc.SchemeSpec(adc.Scheme(scheme), group)
    slot = CodecSlot(rows, cols, spec, torch.bfloat16, torch.bfloat16, k_cap=64)
    y = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda")

    def snapshot():
        parts = [slot.codes.clone()]
        parts += [t.clone() for t in (slot.scales, slot.offsets, slot.idx, slot.val) if t is not None]
        parts.append(y.clone())
        return parts

    eager = []
    for x in xs:
        slot.compress_ptr(x.data_ptr(), torch.cuda.current_stream().cuda_stream)
        slot.decompress_ptr(y.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        eager.append(snapshot())
    src = torch.empty_like(xs[0])
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        sp = torch.cuda.current_stream().cuda_stream
        slot.compress_ptr(src.data_ptr(), sp)
        slot.decompress_ptr(y.data_ptr(), sp)
    for rep in range(3):
        for x, want in zip(xs, eager):
            src.copy_(x)
            graph.replay()
            torch.cuda.synchronize()
            got = snapshot()
            for a, b in zip(got, want):
                assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))
    assert int(slot.status[0]) == 0


K4_PATHS = {"two_launch": 0, "single_pass": 1}


def _k4_eligible(shape, group, dtype_name):
    return group == 128 and shape[1] % 128 == 0 and shape[1] <= 16384 and dtype_name in ("bfloat16", "float16")


@pytest.mark.parametrize("path", sorted(K4_PATHS))
@pytest.mark.parametrize("shape,dtype_name,group", [
    ((8192, 1024), "bfloat16", 128), ((8192, 4096), "bfloat16", 128), ((8192, 768), "float32", 128),
    ((4096, 4096), "float16", 128), ((333, 1024), "bfloat16", 64), ((1000, 40), "float32", 8),
    ((64, 4096), "bfloat16", 256), ((16384, 1024), "bfloat16", 128), ((300, 8), "float16", 16),
    ((4096, 11008), "bfloat16", 128), ((2048, 8192), "float16", 32),
    ((7, 512), "bfloat16", 128), ((3, 4096), "float32", 128)])
def test_outlier_paths_match_oracle(torch_cuda, shape, dtype_name, group, path):
    """Every outlier-separated compress path writes the oracle's bytes: the
    two launches (colreduce + quantiser), the single-pass cooperative kernel
    (k4.cu, one launch where eligible) with and without speculation."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200 import _lib
    rng = np.random.default_rng(shape[0] + 3 * shape[1] + group)
    x = rng.normal(size=shape).astype(np.float32)
    hot = rng.choice(shape[1], max(1, shape[1] // 50), replace=False)
    x[:, hot] *= rng.uniform(8, 50)
    xt = torch.from_numpy(x).to(getattr(torch, dtype_name)).cuda()
    want = oracle_run(xt.cpu().to(torch.float32).numpy(), cases.OUTL, group, 3.0)
    spec = adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED, group)
    try:
        _lib.set_option("outlier_path", K4_PATHS[path])
        n0 = _lib.lib().adc_kernel_launches()
        ct = adc.compress(xt, spec)
        torch.cuda.synchronize()
        if path != "two_launch" and _k4_eligible(shape, group, dtype_name):
            assert _lib.lib().adc_kernel_launches() - n0 == 1
        got = device_run(xt, cases.OUTL, group, 3.0)
    finally:
        _lib.set_option("outlier_path", 2)
    assert cases.norm_digest(*got) == cases.norm_digest(*want)
    idx = want[0]["idx"]
    assert ct.outlier_count == (0 if idx is None else len(idx))


@pytest.mark.parametrize("path", ["single_pass", "two_launch"])
@pytest.mark.parametrize("dtype_name,cols,rows", [("bfloat16", 1024, 2048), ("float32", 768, 2048),
                                                  ("float16", 4096, 2048), ("bfloat16", 3072, 2048),
                                                  ("bfloat16", 4096, 16384), ("bfloat16", 11008, 4096),
                                                  ("float16", 896, 777), ("bfloat16", 128, 5000)])
def test_outlier_prediction_hits_and_misses(torch_cuda, dtype_name, cols, rows, path):
    """A slot's workspace carries the previous call's channel set (and the
    double-buffered column accumulator); the single pass quantises with the
    predicted set and re-quantises the groups whose channels changed
    (resident tiles from shared memory, streamed tiles from global memory).  Alternate inputs with different / equal outlier sets
    through ONE slot and check every call against the oracle."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200.slots import CodecSlot
    rng = np.random.default_rng(cols)
    base = rng.normal(size=(rows, cols)).astype(np.float32)
    sets = [rng.choice(cols, 12, replace=False), rng.choice(cols, 7, replace=False), np.array([], int)]
    seq = [0, 0, 1, 1, 0, 2, 2, 1, 0]
    dt = getattr(torch, dtype_name)
    from paper_2508_00806_b200 import _lib
    _lib.set_option("outlier_path", K4_PATHS[path])
    try:
        slot = CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), dt, torch.float32, k_cap=64)
        y = torch.empty(rows, cols, dtype=torch.float32, device="cuda")
        for step, si in enumerate(seq):
            x = base * rng.uniform(0.5, 2.0)
            x[:, sets[si]] *= 40.0
            xt = torch.from_numpy(x).to(dt).cuda()
            sp = torch.cuda.current_stream().cuda_stream
            slot.compress_ptr(xt.data_ptr(), sp)
            slot.decompress_ptr(y.data_ptr(), sp)
            torch.cuda.synchronize()
            want, wdeq = oracle_run(xt.cpu().to(torch.float32).numpy(), cases.OUTL, 128, 3.0)
            k = int(slot.k_status[1])
            got = cases.normalized(slot.scales.cpu().numpy(), None, slot.codes.cpu().numpy(),
                                   slot.idx[:k].cpu().numpy(), slot.val[:k].cpu().numpy(), None)
            for key in ("scales", "codes", "idx", "vals"):
                w, g = want[key], got[key]
                if w is None or w.size == 0:
                    assert g is None or g.size == 0, (step, key)
                else:
                    np.testing.assert_array_equal(g, w, err_msg=f"step {step} {key}")
            np.testing.assert_array_equal(y.cpu().numpy().view(np.uint32), wdeq.view(np.uint32))
            assert int(slot.status[0]) == 0
    finally:
        _lib.set_option("outlier_path", 2)


@pytest.mark.parametrize("rows", [16384, 16384 + 256])
def test_outlier_decompress_sector_patch_large_outputs(torch_cuda, rows):
    """Outputs past L2 take the whole-sector patch instead of the 2-byte
    scatter: f32 (8-element sectors) and bf16 (16-element sectors) outputs
    agree with each other and with a torch reconstruction from the payload."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    cols = 4096
    g = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn(rows, cols, device="cuda", generator=g)
    hot = torch.randperm(cols, generator=g, device="cuda")[:37]
    hot[1] = hot[0] ^ 1  # two flagged channels in one sector
    x[:, hot] *= 40
    x = x.to(torch.bfloat16)
    ct = adc.compress(x, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED))
    y32 = adc.decompress(ct)                       # 256+ MB: patch, 8-element sectors
    y16 = adc.decompress(ct, torch.bfloat16)       # 128+ MB: patch, 16-element sectors
    assert torch.equal(y16.view(torch.int16), y32.to(torch.bfloat16).view(torch.int16))
    # reference reconstruction: dequantise every code, then overwrite the flagged channels
    nib = torch.stack([ct.packed_codes & 0xF, ct.packed_codes >> 4], dim=1).reshape(-1).to(torch.int32)
    code = torch.where(nib >= 8, nib - 16, nib).to(torch.float32).reshape(rows, cols)
    ref = (code.reshape(-1, 128) * ct.scales.to(torch.float32)[:, None]).reshape(rows, cols)
    idx = ct.outlier_indices.to(torch.int64)
    ref[:, idx] = ct.outlier_values.to(torch.float32).T
    assert idx.numel() >= 30
    assert torch.equal(y32.view(torch.int32), ref.view(torch.int32))


@pytest.mark.parametrize("out_name", ["float32", "bfloat16", "float16"])
@pytest.mark.parametrize("shape,group,n_hot,k_cap", [
    ((8192, 1024), 128, 11, 32), ((2048, 4096), 128, 40, 128), ((777, 896), 64, 9, 16),
    ((5000, 128), 128, 3, 8), ((300, 8), 16, 1, 4), ((4096, 1024), 128, 0, 32),
    ((2048, 768), 128, 20, 8), ((64, 4096), 256, 5, 16), ((16384 + 256, 4096), 128, 37, 64)])
def test_outlier_decompress_one_launch_vs_two(torch_cuda, shape, group, n_hot, k_cap, out_name):
    """The one-launch outlier decompress (output tiles dequantised into shared
    memory and overwritten there, every tile size) writes the same bytes as
    the dequantiser + overwrite launches and the oracle: ragged last row block, k = 0, k above
    the slot's capacity (the first k_cap outliers exact), every output dtype,
    and an output past L2 (where the two-launch path takes the sector patch)."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200 import _lib
    from paper_2508_00806_b200.slots import CodecSlot
    rows, cols = shape
    g = torch.Generator(device="cuda").manual_seed(rows + cols + n_hot)
    x = torch.randn(rows, cols, device="cuda", generator=g)
    if n_hot:
        x[:, torch.randperm(cols, generator=g, device="cuda")[:n_hot]] *= 40
    x = x.to(torch.bfloat16)
    out_dt = getattr(torch, out_name)
    slot = CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED, group), torch.bfloat16, out_dt,
                     k_cap=k_cap)
    slot.compress(x)
    outs = {}
    try:
        for mode, tile in ((0, 8192), (2, 4096), (2, 16384), (2, 8192)):
            _lib.set_option("outlier_decompress", mode)
            _lib.set_option("outlier_tile", tile)
            torch.cuda.synchronize()
            n0 = _lib.lib().adc_kernel_launches()
            outs[(mode, tile)] = slot.decompress()
            torch.cuda.synchronize()
            launches = _lib.lib().adc_kernel_launches() - n0
            assert launches == (1 if mode == 2 else 2)
    finally:
        _lib.set_option("outlier_decompress", 2)
        _lib.set_option("outlier_tile", 8192)
    for key, out in outs.items():
        assert torch.equal(outs[(0, 8192)].view(torch.uint8), out.view(torch.uint8)), key
    outs[2] = outs[(2, 8192)]
    if rows * cols <= (1 << 22):
        k_true = int(slot.k_status[1])
        assert k_true == n_hot or n_hot < 3  # (8 columns: z > 3 is unreachable)
        want, wdeq = oracle_run(x.cpu().to(torch.float32).numpy(), cases.OUTL, group, 3.0)
        if k_true <= k_cap:
            ref = torch.from_numpy(wdeq).to(out_dt)
            assert torch.equal(outs[2].cpu().view(torch.uint8), ref.view(torch.uint8))


@pytest.mark.parametrize("smem_cols", [0, 1024, 8192])
@pytest.mark.parametrize("shape", [(2048, 1024), (1024, 4096), (512, 8192), (300, 16384)])
def test_statistics_sums_in_shared_or_global_memory(torch_cuda, shape, smem_cols):
    """The column-statistics tail gives the oracle's flags and outputs whether
    the sums stay in shared memory or go through global memory
    (sum_smem_cols), on the two-launch path."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200 import _lib
    rng = np.random.default_rng(shape[1] + smem_cols)
    x = rng.normal(size=shape).astype(np.float32)
    x[:, rng.choice(shape[1], max(2, shape[1] // 60), replace=False)] *= 25
    xt = torch.from_numpy(x).to(torch.bfloat16)
    want = oracle_run(xt.to(torch.float32).numpy(), cases.OUTL, 128, 3.0)
    try:
        _lib.set_option("sum_smem_cols", smem_cols)
        _lib.set_option("outlier_path", 0)
        got = device_run(xt, cases.OUTL, 128, 3.0)
    finally:
        _lib.set_option("sum_smem_cols", 8192)
        _lib.set_option("outlier_path", 2)
    assert cases.norm_digest(*got) == cases.norm_digest(*want)


@pytest.mark.parametrize("rows8", [0, 1, 2])
@pytest.mark.parametrize("shape", [(8192, 1024), (2048, 3072), (100, 4096), (131072, 64), (40, 256), (8192, 4096), (16384, 3072)])
def test_column_pass_grid_rows8(torch_cuda, shape, rows8):
    """The column pass's grid shape (cr_rows8: at least 8 rows per row lane)
    changes neither the outlier-separated nor the per-channel bytes."""
    torch = torch_cuda
    from paper_2508_00806_b200 import _lib
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    x = rng.normal(size=shape).astype(np.float32)
    x[:, rng.choice(shape[1], max(1, shape[1] // 90), replace=False)] *= 25
    xt = torch.from_numpy(x).to(torch.bfloat16)
    xf = xt.to(torch.float32).numpy()
    try:
        _lib.set_option("outlier_path", 0)
        _lib.set_option("cr_rows8", rows8)
        for scheme, g in [(cases.OUTL, 128), (cases.SYM, 0)]:
            got = device_run(xt, scheme, g, 3.0)
            want = oracle_run(xf, scheme, g, 3.0)
            assert cases.norm_digest(*got) == cases.norm_digest(*want), (scheme, g)
    finally:
        _lib.set_option("cr_rows8", 2)
        _lib.set_option("outlier_path", 2)


@pytest.mark.parametrize("shape", [(777, 13), (64, 1030), (3000, 40)])
def test_outlier_decompress_fallbacks(torch_cuda, shape):
    """Outputs the one-launch tile kernel cannot take -- element counts not a
    multiple of 8, an output pointer off 16-byte alignment -- fall back to the
    dequantiser + overwrite launches with the same bytes."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200.slots import CodecSlot
    rows, cols = shape
    g = torch.Generator(device="cuda").manual_seed(rows * cols)
    x = torch.randn(rows, cols, device="cuda", generator=g)
    x[:, torch.randperm(cols, generator=g, device="cuda")[:3]] *= 60
    x = x.to(torch.bfloat16)
    slot = CodecSlot(rows, cols, adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), torch.bfloat16, torch.bfloat16,
                     k_cap=16)
    slot.compress(x)
    ref = slot.decompress()
    buf = torch.empty(rows * cols + 8, dtype=torch.bfloat16, device="cuda")
    y = buf[1:1 + rows * cols]  # 2-byte offset: not 16-byte aligned
    slot.decompress_ptr(y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(y.view(rows, cols).view(torch.int16), ref.view(torch.int16))
    if rows * cols <= (1 << 20):
        want, wdeq = oracle_run(x.cpu().to(torch.float32).numpy(), cases.OUTL, 128, 3.0)
        assert torch.equal(ref.cpu().view(torch.int16), torch.from_numpy(wdeq).to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("shape,dtype_name", [((512, 1024), "bfloat16"), ((1000, 40), "float32"),
                                              ((257, 4096), "float16")])
def test_outlier_gather_modes_vs_oracle(torch_cuda, shape, dtype_name, monkeypatch):
    """The side-buffer gather by leading CTAs (ADC_GATHER_TAIL=0) and by the
    quantising CTAs after their units (=1) both match the oracle."""
    torch = torch_cuda
    rng = np.random.default_rng(shape[0])
    x = rng.normal(size=shape).astype(np.float32)
    x[:, rng.choice(shape[1], max(2, shape[1] // 50), replace=False)] *= 30
    xt = torch.from_numpy(x).to(getattr(torch, dtype_name))
    want = oracle_run(xt.to(torch.float32).numpy(), cases.OUTL, 128, 3.0)
    assert isinstance(want[0], dict) and want[0]["idx"] is not None and len(want[0]["idx"]) >= 2
    for mode in ("0", "1"):
        monkeypatch.setenv("ADC_GATHER_TAIL", mode)
        got = device_run(xt, cases.OUTL, 128, 3.0)
        assert cases.norm_digest(*got) == cases.norm_digest(*want), mode


def test_outlier_separated_at_2_31_elements(torch_cuda):
    """2^31 elements (4 GB bf16) stays exact on the fast quantiser (the
    channel index of the zeroing step is taken on 8-element units).  The
    input is a [256, 4096] block tiled 2048 times down the rows: a power-of-2
    repetition scales every column sum, the mean and the std exactly, so the
    flagged set, codes, scales and side values are the block's, tiled."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    rows0, cols, reps = 256, 4096, 2048
    g = torch.Generator(device="cuda").manual_seed(31)
    blk = torch.randn(rows0, cols, device="cuda", generator=g)
    hot = torch.randperm(cols, generator=g, device="cuda")[:29]
    blk[:, hot] *= 40
    blk = blk.to(torch.bfloat16)
    spec = adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED)
    small = adc.compress(blk, spec)
    x = blk.repeat(reps, 1)
    assert x.numel() == 1 << 31
    big = adc.compress(x, spec)
    del x
    assert torch.equal(big.outlier_indices, small.outlier_indices)
    assert small.outlier_indices.numel() == 29
    assert torch.equal(big.packed_codes.view(reps, -1), small.packed_codes.view(1, -1).expand(reps, -1))
    assert torch.equal(big.scales.view(reps, -1), small.scales.view(1, -1).expand(reps, -1))
    k = small.outlier_indices.numel()
    assert torch.equal(big.outlier_values.view(k, reps, rows0), small.outlier_values.view(k, 1, rows0).expand(k, reps, rows0))
    y = adc.decompress(big, torch.bfloat16)
    y0 = adc.decompress(small, torch.bfloat16)
    assert torch.equal(y.view(reps, rows0, cols).view(torch.int16), y0.view(1, rows0, cols).expand(reps, rows0, cols).view(torch.int16))


@pytest.mark.parametrize("scheme,group,shape", [
    (cases.SYM, 128, (300, 70)), (cases.ASYM, 128, (256, 768)), (cases.OUTL, 128, (512, 1024)),
    (cases.SYM, 0, (64, 96)), (cases.MASK, 0, (33, 17)), (cases.ASYM, 7, (5, 11)), (cases.OUTL, 64, (1000, 40))])
def test_device_serialize_matches_host_and_oracle_bytes(torch_cuda, scheme, group, shape):
    """adc_serialize assembles the ADC1 bytes on the device: identical to the
    host serializer and to the oracle's (reference-pinned) serializer, for
    parity records and for async records read straight from the slot buffers."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from oracle import codec_oracle as orc
    rng = np.random.default_rng(shape[0] * 3 + group)
    if scheme == cases.MASK:
        x = (rng.random(shape) < 0.7).astype(np.uint8)
    else:
        x = rng.normal(size=shape).astype(np.float32)
        x[:, :: max(1, shape[1] // 9)] *= 30
    spec = adc.SchemeSpec(adc.Scheme(scheme), group)
    ct = adc.compress(x, spec)
    dev_bytes = adc.serialize_device(ct).cpu().numpy().tobytes()
    assert dev_bytes == adc.serialize(ct)
    assert dev_bytes == orc.serialize(orc.compress(x, scheme, group, 3.0))
    if scheme == cases.OUTL:  # async record: (k_cap, rows) buffers and the device k
        act = adc.compress_async(torch.from_numpy(x).cuda(), spec)
        assert adc.serialize_device(act).cpu().numpy().tobytes() == dev_bytes


def test_concurrent_streams_are_reentrant(torch_cuda):
    """adacc.h: calls are reentrant with distinct buffers / workspaces.  Run
    every scheme on four streams at once, repeatedly, and compare with the
    serial results (the cross-CTA counters live in each slot's workspace)."""
    torch = torch_cuda
    import paper_2508_00806_b200 as adc
    from paper_2508_00806_b200.slots import CodecSlot
    g = torch.Generator(device="cuda").manual_seed(11)
    jobs = []
    for spec, shape in [(adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), (4096, 1024)),
                        (adc.SchemeSpec(adc.Scheme.ASYMMETRIC_GROUP), (8192, 1024)),
                        (adc.SchemeSpec(adc.Scheme.SYMMETRIC_GROUP, 0), (4096, 768)),
                        (adc.SchemeSpec(adc.Scheme.OUTLIER_SEPARATED), (2048, 4096))]:
        x = torch.randn(*shape, device="cuda", generator=g)
        x[:, ::77] *= 35
        x = x.to(torch.bfloat16)
        slot = CodecSlot(shape[0], shape[1], spec, torch.bfloat16, torch.float32, k_cap=128)
        y = torch.empty(shape, dtype=torch.float32, device="cuda")
        jobs.append((slot, x, y))

    def snapshot(slot, y):
        parts = [slot.codes.clone(), slot.scales.clone(), y.clone()]
        if slot.idx is not None:
            k = int(slot.k_status[1])
            parts += [slot.idx[:k].clone(), slot.val[:k].clone()]
        return parts

    serial = []
    for slot, x, y in jobs:
        sp = torch.cuda.current_stream().cuda_stream
        slot.compress_ptr(x.data_ptr(), sp)
        slot.decompress_ptr(y.data_ptr(), sp)
        torch.cuda.synchronize()
        serial.append(snapshot(slot, y))
    streams = [torch.cuda.Stream() for _ in jobs]
    for _ in range(5):
        for (slot, x, y), st in zip(jobs, streams):
            with torch.cuda.stream(st):
                for _ in range(3):
                    slot.compress_ptr(x.data_ptr(), st.cuda_stream)
                    slot.decompress_ptr(y.data_ptr(), st.cuda_stream)
        torch.cuda.synchronize()
        for (slot, x, y), want in zip(jobs, serial):
            for a, b in zip(snapshot(slot, y), want):
                assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))
            assert int(slot.status[0]) == 0
