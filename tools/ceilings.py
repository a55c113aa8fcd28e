"""Practical FP32 ceilings on this GPU: cuBLAS SGEMM / cuDNN FP32 conv (TF32 off)
at the BASELINE shapes, to compare the tiled template against library kernels.

  python tools/ceilings.py        prints one JSON line per shape

Not product code: library kernels are the yardstick, not the measured path.
"""

import json

import torch

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
torch.backends.cudnn.benchmark = True


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


def main():
    d = torch.device("cuda")
    out = []
    for n in (512, 1024, 4096):
        a, b = torch.rand(n, n, device=d), torch.rand(n, n, device=d)
        us = timed(lambda: a @ b)
        out.append({"op": f"sgemm {n}^3", "us": us, "tflops": 2 * n ** 3 / us / 1e6})
    a, b = torch.rand(192, 128, 64, device=d), torch.rand(192, 64, 128, device=d)
    us = timed(lambda: torch.bmm(a, b))
    out.append({"op": "bmm TBG", "us": us, "tflops": 2 * 192 * 128 * 128 * 64 / us / 1e6})
    for (h, ci, co) in ((56, 64, 64), (28, 128, 128)):
        x = torch.rand(16, ci, h, h, device=d).to(memory_format=torch.channels_last)
        w = torch.rand(co, ci, 3, 3, device=d).to(memory_format=torch.channels_last)
        us = timed(lambda: torch.nn.functional.conv2d(x, w, padding=1))
        out.append({"op": f"cudnn conv fp32 N16 {h}x{h}x{ci}->{co} 3x3 NHWC", "us": us,
                    "tflops": 2 * 16 * h * h * ci * co * 9 / us / 1e6})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
