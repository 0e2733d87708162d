"""Prefill-shaped (config 4: Mixtral gate/up/down, 8192 tokens, 4 sequences of
64 adapters) step time at r = 8 / 16 / 32 / 64 / 128 (large segments on the
tcgen05 chain at every rank; RANK_SWEEP_BASE=<config> for other shapes).
Prints one JSON line."""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import lora_inputs as li  # noqa: E402


def main():
    base = os.environ.get("RANK_SWEEP_BASE", "mixtral_prefill")
    import torch
    from paper_2604_07173_b200 import binding as B
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    hbm_peak, _, _ = bench.load_peaks()
    out = {}
    for rk in [int(a) for a in (sys.argv[1:] or ["8", "16", "32", "64", "128"])]:
        c = dataclasses.replace(li.CONFIGS[base], name=f"{base}_r{rk}", rank=rk)
        b = li.make_batch(c)
        slots = list(range(len(c.slots)))
        r = bench.SingleRun(B, torch, c, b, slots, dev, stream)
        t, tot = r.time(10, 3)
        prof = r.profile(3)
        sm = bench.summarise(c, bench.algorithmic(c, b, slots), t, tot, hbm_peak, prof, 3)
        r.destroy()
        out[str(rk)] = {k: sm[k] for k in ("ms_per_step", "tokens_per_s", "step_GBs", "frac_measured", "kernels")}
        print(rk, json.dumps(out[str(rk)]), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
