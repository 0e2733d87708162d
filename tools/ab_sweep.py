#!/usr/bin/env python
"""A/B of run-time switches over batch sizes (config-3 shapes by default):
each variant runs in its own process (switches are read at server create),
step = plan build + gate/up/down apply, CUDA-graph replay, median of 30.

    python tools/ab_sweep.py [--workload mixtral_decode] [--tokens 64,128,256,512,1024] base: v1:LORA_X=1,LORA_Y=2
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(workload, tokens):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import lora_inputs as li
    from bench import SingleRun
    from paper_2604_07173_b200 import binding as B
    base = li.CONFIGS[workload]
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    out = {}
    srv = None
    maxr = max(tokens) * base.top_k
    for n in tokens:
        cfg = li.with_tokens(base, n)
        b = li.make_batch(cfg)
        r = SingleRun(B, torch, cfg, b, list(range(len(cfg.slots))), dev, st, server=srv, max_rows=maxr)
        srv = r.s
        times, _ = r.time(30, 3)
        r.own_server = False
        r.destroy()
        out[n] = round(float(np.median(times)) * 1e3, 1)
    B.lora_server_destroy(srv)
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="mixtral_decode")
    ap.add_argument("--tokens", default="64,128,256,512,1024")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    tokens = [int(v) for v in a.tokens.split(",")]
    if a.child:
        return child(a.workload, tokens)
    res = {}
    for rep in range(2):
        for v in a.variants:
            name, envs = v.split(":", 1)
            env = dict(os.environ)
            for kv in filter(None, envs.split(",")):
                k, val = kv.split("=", 1)
                env[k] = val
            p = subprocess.run([sys.executable, __file__, "--child", "--workload", a.workload, "--tokens", a.tokens],
                               env=env, capture_output=True, text=True, timeout=600)
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
            except Exception:
                d = {"error": p.stderr[-300:]}
            res.setdefault(name, []).append(d)
            print(f"{a.workload} {name:10s} rep {rep}: {d}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
