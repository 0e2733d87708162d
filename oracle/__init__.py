"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py and lora_oracle.c).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never from the product package.
"""
from .oracle import *  # noqa: F401,F403
from .oracle import build, segment, lora_apply_rows, apply_slot, apply_slot_all_rows, unit_tables, shard_dispatch  # noqa: F401
