"""Measure integer-pipe peaks on this GPU (writes JSON to stdout)."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_1901_10074_b200 import _native as nat


def measure(kind, blocks=148 * 8, iters=2000):
    lib = nat.load()
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    nat.check(lib.hefv_probe_int(kind, blocks, 10, out.data_ptr(), st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nat.check(lib.hefv_probe_int(kind, blocks, iters, out.data_ptr(), st))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ops = blocks * 256 * iters * 128
    return ops / (ms * 1e-3)


if __name__ == "__main__":
    names = ["imad", "imad_hi", "imad_wide", "iadd3", "shoup_butterfly", "shoup_butterfly64",
             "mad_wide_acc", "dfma", "butterfly_fp64q", "butterfly_mixed"]
    res = {n: measure(k) / 1e12 for k, n in enumerate(names)}
    print(json.dumps({"unit": "Tops/s", **{k: round(v, 3) for k, v in res.items()}}))
