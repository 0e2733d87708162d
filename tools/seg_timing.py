"""Time lora_plan_build (the segmenter) for several row counts / key ranges."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2604_07173_b200 import binding as B

def main():
    for (T, nad, E) in [(256, 128, 1), (1024, 512, 8), (8192, 2048, 8), (16384, 64, 8), (16384, 2048, 8)]:
        c = B.make_config([128], [128], [E], 64, nad, None, T, 0)
        s = B.lora_server_create(c)
        rng = np.random.default_rng(0)
        a = torch.from_numpy(rng.integers(0, nad, T).astype(np.int32)).cuda()
        e = torch.from_numpy(rng.integers(0, E, T).astype(np.int32)).cuda()
        p = B.lora_plan_create(s, T)
        for _ in range(5):
            B.lora_plan_build(s, p, a, e if E > 1 else None, T, E)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(50):
            B.lora_plan_build(s, p, a, e if E > 1 else None, T, E)
        ev1.record()
        torch.cuda.synchronize()
        print(f"T={T:6d} K={nad*E:6d}: {ev0.elapsed_time(ev1) / 50 * 1e3:7.1f} us", flush=True)
        B.lora_plan_destroy(p)
        B.lora_server_destroy(s)

main()
