"""One bench step under the CUDA profiler range, for ncu.

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
        dram__bytes_write.sum --csv python tools/ncu_step.py

Builds the same nine GPT-345M block slots as bench.py, warms up, then runs one
compress+decompress step inside cudaProfilerStart/Stop.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2508_00806_b200 as adc  # noqa: E402
from paper_2508_00806_b200.slots import CodecSlot  # noqa: E402
from paper_2508_00806_b200.workload import gpt_block_ops, synth_activation  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ops = gpt_block_ops()
    only = sys.argv[1:]  # optional op names
    xs, slots, outs = [], [], []
    for op in ops:
        if only and op.name not in only:
            continue
        x = synth_activation(op, seed=1, device=dev)
        spec = adc.scheme_for(op.kind)
        k_cap = None
        if spec.scheme is adc.Scheme.OUTLIER_SEPARATED:
            k_cap = max(16, 2 * adc.compress(x, spec).outlier_count)
        s = CodecSlot(op.rows, op.cols, spec, torch.bool if x.dtype == torch.bool else x.dtype,
                      torch.uint8 if x.dtype == torch.bool else torch.bfloat16, k_cap=k_cap, device=dev)
        xs.append(x)
        slots.append(s)
        outs.append(torch.empty((op.rows, op.cols), dtype=s.out_dtype, device=dev))
    sp = torch.cuda.current_stream().cuda_stream

    def step():
        for s, x in zip(slots, xs):
            s.compress_ptr(x.data_ptr(), sp)
        for s, y in reversed(list(zip(slots, outs))):
            s.decompress_ptr(y.data_ptr(), sp)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
