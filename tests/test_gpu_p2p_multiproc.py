"""The sharded server's push path with two real ranks on ONE GPU.

Two processes, each a rank of a world-2 sharded server on cuda:0, with the
host control plane (lora_server_create_sharded_host over a gloo all-gather):
each rank registers its x / y buffers (lora_shard_register: CUDA IPC, mapped
by the other process); the counts travel through the control areas (device
flags), the owner's shrink kernels read the received x rows from the other
process's x, and the owner's expand epilogue adds the deltas into the other
process's y (red.add).  Checked: fp32 y bit-identical to the
unsharded server on every row when every segment takes the CUDA-core route
(R18; a tcgen05 segment rounds v to bf16, and a unit's rows can be
split between the local and the received plan), every case within the
tolerance of the oracle,
for LoRA Data Parallel with and without replicated adapters and for expert
parallel.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lora_inputs as li

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(y_dtype, two_layers=False):
    sl = (li.Slot("a", 512, 768, 4, 0), li.Slot("b", 768, 512, 4, 1))
    if two_layers:
        sl = sl + (li.Slot("a1", 512, 768, 4, 2), li.Slot("b1", 768, 512, 4, 3))
    return li.Config("mp_p2p", 8, sl, 64, 24, 4, 2, 300, y_dtype)


def _token_range(n_tokens, world, rank, empty_rank):
    """Contiguous token split; with empty_rank >= 0 that rank holds no token
    (its neighbours split its share)."""
    if empty_rank < 0:
        return (n_tokens * rank) // world, (n_tokens * (rank + 1)) // world
    bounds = [0]
    others = [r for r in range(world) if r != empty_rank]
    for r in range(world):
        if r == empty_rank:
            bounds.append(bounds[-1])
        else:
            i = others.index(r)
            bounds.append((n_tokens * (i + 1)) // len(others))
    return bounds[rank], bounds[rank + 1]


def _worker(rank, world, port, out_dir, y_dtype, n_hot, ep, pp=0, empty_rank=-1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if y_dtype == "fp32":
        # CUDA-core route for every segment: the per-row arithmetic then does not depend on how
        # a unit's rows are split between the local and the received plan (bit-exact check)
        os.environ["LORA_SMALL_SEG_MAX"] = "-1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2604_07173_b200 import binding as B

        def allgather(data: bytes) -> bytes:
            t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
            out = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return b"".join(o.numpy().tobytes() for o in out)

        cfg = _cfg(y_dtype, two_layers=pp > 1)
        n_sl = len(cfg.slots)
        calls = [[0, 1], [2, 3]] if pp > 1 else [[0, 1]]   # one sharded apply per layer
        b = li.make_batch(cfg)
        k = b.top_k
        t0, t1 = _token_range(cfg.n_tokens, world, rank, empty_rank)
        r0, r1 = t0 * k, t1 * k
        T = r1 - r0
        Tb = max(T, 1)  # buffers (a rank may hold no row)
        # capacity: every rank's max_rows must cover its own rows, and max_rows * world the rows it may
        # receive (an empty rank still serves the others)
        cap = max(T, (b.n_rows + world - 1) // world) if empty_rank < 0 else b.n_rows
        c = B.make_config([s.h_in for s in cfg.slots], [s.h_out for s in cfg.slots], [4] * n_sl, cfg.rank,
                          cfg.n_adapters, cfg.scale(), cap, 0, n_replicated=n_hot, expert_parallel=ep, pp_stages=pp,
                          slot_layer=[i // 2 for i in range(n_sl)])
        s = B.lora_server_create_sharded_host(c, rank, world, allgather)
        B.lora_server_fill_synthetic(s, cfg.seed)
        xs, ys = [], []
        for i, sl in enumerate(cfg.slots):
            x = torch.zeros((Tb, sl.h_in), dtype=torch.int16, device="cuda")
            B.lora_synth_fill_rows(x, T, sl.h_in, cfg.seed, li.tag_of(li.KIND_X, sl.xbuf), li.shift_x(), r0)
            y = torch.zeros((Tb, sl.h_out), dtype=torch.int16, device="cuda")
            B.lora_synth_fill_rows(y, T, sl.h_out, cfg.seed, li.tag_of(li.KIND_Y0, i), li.shift_y0(), r0)
            if y_dtype == "fp32":
                y = ((y.to(torch.int32) << 16).view(torch.float32)).contiguous()
            xs.append(x)
            ys.append(y)
        ad = torch.from_numpy(b.adapter_ids[r0:r1].copy()).cuda()
        ex = torch.from_numpy(b.expert_ids[r0:r1].copy()).cuda()
        dt = B.LORA_FP32 if y_dtype == "fp32" else B.LORA_BF16
        yy = [y.clone() for y in ys]
        B.lora_shard_register(s, xs + yy, [t.numel() * t.element_size() for t in xs + yy])
        for _ in range(3):  # later calls reuse the registrations; the epoch advances
            for v, v0 in zip(yy, ys):
                v.copy_(v0)
            torch.cuda.synchronize()
            dist.barrier()  # (no rank may overwrite its y while a peer still pushes into it)
            for cl in calls:
                B.lora_apply_sharded(s, cl, [xs[i] for i in cl], ad, ex, [yy[i] for i in cl], dt, T)
            torch.cuda.synchronize()
        assert B.lora_server_check(s) == B.LORA_OK
        for i in range(n_sl):
            np.save(os.path.join(out_dir, f"y{i}_{rank}.npy"), yy[i][:T].cpu().numpy())
        B.lora_server_destroy(s)
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("y_dtype,n_hot,ep,world,pp,empty", [
    ("fp32", 0, False, 2, 0, -1), ("fp32", 3, False, 2, 0, -1), ("bf16", 0, False, 2, 0, -1),
    ("fp32", 0, True, 2, 0, -1), ("fp32", 0, True, 4, 2, -1), ("fp32", 0, False, 3, 0, 1)])
def test_p2p_two_ranks_one_gpu(tmp_path, y_dtype, n_hot, ep, world, pp, empty):
    """(world 4, pp 2: hybrid EP2-PP2 over four processes, one sharded apply
    per layer; each layer's rows are served by its group's two ranks, every
    rank sends.  world 3 with rank 1 holding no row: it still owns adapters,
    serves the others' rows and takes part in every flag exchange.)"""
    from tests import gpu_util as U
    from oracle import oracle as orc
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), y_dtype, n_hot, ep, pp, empty), nprocs=world,
             join=True)
    B = U.binding()
    cfg = _cfg(y_dtype, two_layers=pp > 1)
    b = li.make_batch(cfg)
    T = b.n_rows
    s = U.make_server(B, cfg, small_max=-1 if y_dtype == "fp32" else None)
    try:
        for i in range(len(cfg.slots)):
            got = np.concatenate([np.load(tmp_path / f"y{i}_{r}.npy") for r in range(world)])
            U.assert_parity(torch.from_numpy(got), orc.apply_slot(cfg, i, b), f"p2p 2-rank slot {i}")
            if y_dtype == "fp32":
                # same fp32 delta, added once at the row's home: bit-exact with the unsharded server
                ad, ex = U.ids_dev(b)
                x = U.x_dev(B, cfg, i, T)
                y = U.y0_dev(B, cfg, i, T)
                B.lora_apply(s, i, x, ad, ex, y, B.LORA_FP32, T)
                torch.cuda.synchronize()
                np.testing.assert_array_equal(got.view(np.uint32), y.cpu().numpy().view(np.uint32))
    finally:
        B.lora_server_destroy(s)
