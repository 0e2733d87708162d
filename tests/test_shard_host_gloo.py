"""Sharded LoRA Server host logic on CPU, world size 2 over gloo.

The data path of lora_apply_sharded is NCCL + our kernels (GPU).  What can be
checked without GPUs is everything around it, exercised here through the same
steps the library takes (shard.cu): owner classification (adapters
[0, n_hot) replicated on every rank and processed in place, the rest owned by
rank (a - n_hot) mod G; R19), stable bucketing of the remote rows,
the count exchange (all-gather), the library's own host routine
lora_shard_layout (C-ABI, no GPU needed) for send/receive offsets, the row
exchange in that layout, delta-mode compute on the owner (the oracle stands in
for the GPU kernels here -- test-only), the return exchange and the add at the
origin.  Sharded == unsharded bit-exactly (R18), and the receive
order matches the oracle's dispatch emulation.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lora_inputs as li


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    return li.Config("shard_cpu", 11, (li.Slot("s", 128, 64, 4, 0),), 8, 10, 4, 2, 48, "fp32")


def _worker(rank, world, port, out_dir, n_hot):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_07173_b200 import build
        build.build()
        from paper_2604_07173_b200 import binding as B
        from oracle import oracle as orc

        cfg = _cfg()
        batch = li.make_batch(cfg)
        k, G = batch.top_k, world
        t0, t1 = orc.token_range(cfg.n_tokens, G, rank)
        rows = np.arange(t0 * k, t1 * k)
        a = batch.adapter_ids[rows]
        # 1. classify: in-place rows (owner == me) and stable owner buckets of the rest
        own = orc.owner_of(a, G, n_hot, np.full(a.shape, rank))
        local_idx = np.flatnonzero(own == rank)
        send_idx = np.concatenate([np.flatnonzero(own == d) for d in range(G) if d != rank])
        counts = np.array([(own == d).sum() if d != rank else 0 for d in range(G)], np.int64)
        # 2. count exchange
        allc = [torch.zeros(G, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(allc, torch.from_numpy(counts))
        mat = torch.stack(allc).numpy().reshape(-1)
        so, ro = B.lora_shard_layout(mat.tolist(), G, rank)
        assert so[-1] == len(send_idx) and so[rank + 1] == so[rank] and ro[rank + 1] == ro[rank]
        # 3. dispatch the global row ids (the payload stands for x rows + ids)
        payload = torch.from_numpy(rows[send_idx].astype(np.int64))
        recv = torch.zeros(ro[-1], dtype=torch.int64)
        reqs = []
        for p in range(G):
            if so[p + 1] > so[p] and p != rank:
                reqs.append(dist.isend(payload[so[p]:so[p + 1]].contiguous(), p))
        for p in range(G):
            if ro[p + 1] > ro[p]:
                buf = torch.zeros(ro[p + 1] - ro[p], dtype=torch.int64)
                dist.recv(buf, p)
                recv[ro[p]:ro[p + 1]] = buf
        for r in reqs:
            r.wait()
        got_rows = recv.numpy()
        # receive order == the oracle's dispatch emulation
        disp = orc.shard_dispatch(batch, G, n_hot)[rank]
        np.testing.assert_array_equal(got_rows, disp["rows"])
        np.testing.assert_array_equal(rows[local_idx], disp["local"])
        np.testing.assert_array_equal(mat.reshape(G, G), disp["counts"])
        # 4. owner-side delta (fp64, exact): oracle stands in for the kernels in this CPU test
        x, uor, sor, A, Bw, _ = orc.prepare_slot(cfg, 0, batch, got_rows)
        d = np.zeros((len(got_rows), cfg.slots[0].h_out), np.float32)
        # delta = y0=0 + delta, fp32; the library returns fp32 deltas the same way
        orc.lora_apply_rows(x, uor, sor, A, Bw, d)
        # 5. return deltas in the reverse layout
        dt = torch.from_numpy(d)
        back = torch.zeros((so[-1], d.shape[1]), dtype=torch.float32)
        reqs = []
        for p in range(G):
            if ro[p + 1] > ro[p] and p != rank:
                reqs.append(dist.isend(dt[ro[p]:ro[p + 1]].contiguous(), p))
        for p in range(G):
            if so[p + 1] > so[p]:
                buf = torch.zeros((so[p + 1] - so[p], d.shape[1]), dtype=torch.float32)
                dist.recv(buf, p)
                back[so[p]:so[p + 1]] = buf
        for r in reqs:
            r.wait()
        # 6. add at the origin (one rounding of fp32 y + fp32 delta)
        y = li.bf16_bits_to_f32(li.y0_rows_bits(cfg.seed, 0, rows, cfg.slots[0].h_out)).copy()
        y[send_idx] = y[send_idx] + back.numpy()
        # in-place rows: the same fp32 delta, added once
        if len(local_idx):
            xl, ul, sl, Al, Bl, _ = orc.prepare_slot(cfg, 0, batch, rows[local_idx])
            dl = np.zeros((len(local_idx), cfg.slots[0].h_out), np.float32)
            orc.lora_apply_rows(xl, ul, sl, Al, Bl, dl)
            y[local_idx] = y[local_idx] + dl
        np.save(os.path.join(out_dir, f"y{rank}.npy"), y)
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("n_hot", [0, 3])
def test_sharded_host_logic_world2_gloo(tmp_path, n_hot):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), n_hot), nprocs=world, join=True)
    from oracle import oracle as orc
    cfg = _cfg()
    batch = li.make_batch(cfg)
    y_sharded = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(world)])
    # unsharded, same arithmetic order (fp32 delta, then one fp32 add at the row's home): bit-exact
    d_ref = orc.apply_slot(cfg, 0, batch, y0="zero")
    y0 = li.bf16_bits_to_f32(li.y0_rows_bits(cfg.seed, 0, np.arange(batch.n_rows), cfg.slots[0].h_out))
    touched = batch.adapter_ids >= 0
    y_same = y0.copy()
    y_same[touched] = y0[touched] + d_ref[touched]
    np.testing.assert_array_equal(y_sharded.view(np.uint32), y_same.view(np.uint32))
    # and the oracle's single rounding of (y + delta), within the north-star tolerance
    y_ref = orc.apply_slot(cfg, 0, batch)
    assert np.abs(y_sharded - y_ref).max() <= 1e-2 * np.abs(y_ref).max() + 1e-3


def _p2p_worker(rank, world, port, out_dir, n_hot, ep=False):
    """The P2P transport's address maps (lora_shard_peer_rows, used by
    shard.cu) on emulated peer memory: every rank's send buffer (global row
    ids in send order) and delta buffer (global row ids in receive order) are
    all-gathered; reading them through the row maps must give the oracle's
    receive order on the owner side and each source's own rows back."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_07173_b200 import build
        build.build()
        from paper_2604_07173_b200 import binding as B
        from oracle import oracle as orc

        cfg = _cfg()
        batch = li.make_batch(cfg)
        k, G = batch.top_k, world
        t0, t1 = orc.token_range(cfg.n_tokens, G, rank)
        rows = np.arange(t0 * k, t1 * k)
        a = batch.adapter_ids[rows]
        own = orc.owner_of(a, G, n_hot, np.full(a.shape, rank), batch.expert_ids[rows], ep)
        send_rows = np.concatenate([rows[own == d] for d in range(G) if d != rank] + [np.zeros(0, np.int64)])
        counts = np.array([(own == d).sum() if d != rank else 0 for d in range(G)], np.int64)
        allc = [torch.zeros(G, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(allc, torch.from_numpy(counts))
        mat = torch.stack(allc).numpy().reshape(-1)
        so, ro = B.lora_shard_layout(mat.tolist(), G, rank)
        rb_in, rb_out = B.lora_shard_peer_rows(mat.tolist(), G, rank)
        cap = cfg.n_tokens * k

        def gather_padded(v):
            buf = torch.full((cap,), -7, dtype=torch.int64)
            buf[:len(v)] = torch.from_numpy(np.asarray(v, np.int64))
            out = [torch.zeros(cap, dtype=torch.int64) for _ in range(G)]
            dist.all_gather(out, buf)
            return [o.numpy() for o in out]

        peer_send = gather_padded(send_rows)
        # owner: received row r from source s is row r + rb_in[s] of s's send buffer
        recv = np.array([peer_send[s][r + rb_in[s]] for s in range(G) for r in range(ro[s], ro[s + 1])], np.int64)
        disp = orc.shard_dispatch(batch, G, n_hot, ep)[rank]
        np.testing.assert_array_equal(recv, disp["rows"])
        # owner's delta buffer holds its received rows in receive order
        peer_d = gather_padded(recv)
        back = np.array([peer_d[p][j + rb_out[p]] for p in range(G) for j in range(so[p], so[p + 1])], np.int64)
        np.testing.assert_array_equal(back, send_rows)
        np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([len(recv), len(back)]))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_hot,ep", [(2, 0, False), (3, 0, False), (3, 2, False), (2, 0, True)])
def test_p2p_row_maps_gloo(tmp_path, world, n_hot, ep):
    mp.spawn(_p2p_worker, args=(world, _free_port(), str(tmp_path), n_hot, ep), nprocs=world, join=True)
    tot = sum(int(np.load(tmp_path / f"ok{r}.npy")[0]) for r in range(world))
    assert tot > 0  # rows actually crossed ranks
