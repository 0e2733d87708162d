"""Convenience wrapper over the C-ABI for torch callers (marshalling only)."""
from __future__ import annotations

from typing import Optional, Sequence

import torch

from . import binding as B


def _dtype_code(y: torch.Tensor) -> int:
    if y.dtype == torch.float32:
        return B.LORA_FP32
    if y.dtype in (torch.bfloat16, torch.int16, torch.uint16):
        return B.LORA_BF16
    raise TypeError(f"y must be float32 or bfloat16, got {y.dtype}")


class Plan:
    def __init__(self, server: "LoraServer", max_rows: int):
        self.server = server
        self.handle = B.lora_plan_create(server.handle, max_rows)
        self.max_rows = max_rows

    def build(self, adapter_ids: torch.Tensor, expert_ids: Optional[torch.Tensor], n_experts: int, stream=None):
        T = int(adapter_ids.numel())
        B.lora_plan_build(self.server.handle, self.handle, adapter_ids, expert_ids, T, n_experts, stream)
        return self

    def export(self, stream=None):
        d = self.server.device
        perm = torch.empty(self.max_rows, dtype=torch.int32, device=d)
        off = torch.empty(self.max_rows + 1, dtype=torch.int32, device=d)
        keys = torch.empty(self.max_rows, dtype=torch.int32, device=d)
        nv, ns = B.lora_plan_export(self.server.handle, self.handle, perm, off, keys, stream)
        return perm[:nv].cpu(), off[:ns + 1].cpu(), keys[:ns].cpu()

    def close(self):
        if self.handle:
            B.lora_plan_destroy(self.handle)
            self.handle = None


class LoraServer:
    """One GPU's LoRA Server: weight store for n_slots projections."""

    def __init__(self, h_in: Sequence[int], h_out: Sequence[int], n_experts: Sequence[int], rank: int,
                 n_adapters: int, scale=None, max_rows: int = 4096, device: int = 0, A=None, B_=None,
                 weights_on_device: bool = True):
        self.cfg = B.make_config(h_in, h_out, n_experts, rank, n_adapters, scale, max_rows, device)
        self.handle = B.lora_server_create(self.cfg, A, B_, weights_on_device)
        self.device = torch.device("cuda", device)
        self.h_in, self.h_out, self.n_experts = list(h_in), list(h_out), list(n_experts)
        self.rank, self.n_adapters, self.max_rows = rank, n_adapters, max_rows

    def fill_synthetic(self, seed: int, stream=None):
        B.lora_server_fill_synthetic(self.handle, seed, stream)

    def set_small_seg_max(self, n: int):
        B.lora_server_set_small_seg_max(self.handle, n)

    def plan(self, max_rows: Optional[int] = None) -> Plan:
        return Plan(self, max_rows or self.max_rows)

    def apply(self, slot: int, x: torch.Tensor, adapter_ids: torch.Tensor, expert_ids: Optional[torch.Tensor],
              y: torch.Tensor, stream=None):
        B.lora_apply(self.handle, slot, x, adapter_ids, expert_ids, y, _dtype_code(y), int(adapter_ids.numel()),
                     stream)

    def apply_plan(self, plan: Plan, slot: int, x: torch.Tensor, y: torch.Tensor, stream=None):
        B.lora_apply_plan(self.handle, plan.handle, slot, x, y, _dtype_code(y), stream)

    def apply_multi(self, plan: Plan, slots: Sequence[int], xs, ys, stream=None):
        B.lora_apply_plan_multi(self.handle, plan.handle, list(slots), list(xs), list(ys), _dtype_code(ys[0]), stream)

    def check(self, stream=None) -> int:
        return B.lora_server_check(self.handle, stream)

    def close(self):
        if self.handle:
            B.lora_server_destroy(self.handle)
            self.handle = None
