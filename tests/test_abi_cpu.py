"""CPU-only checks of the C-ABI library: it builds, loads, exports every symbol
declared in include/*.h, the ctypes binding matches the header, and the
host-only entry points behave (argument errors, shard layout)."""
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^(?:const\s+)?\w+\s*\*?\s*(lora_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def B():
    from paper_2604_07173_b200 import build
    build.build()
    from paper_2604_07173_b200 import binding
    return binding


def test_header_declares_the_boundary():
    names = _declared_functions()
    for must in ["lora_server_create", "lora_apply", "lora_server_destroy", "lora_plan_build", "lora_apply_plan",
                 "lora_apply_plan_multi", "lora_apply_sharded", "lora_server_create_sharded"]:
        assert must in names


def test_library_exports_every_declared_symbol(B):
    names = _declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(B.lib, n), f"{n} not exported"
        assert n in B.SIGNATURES, f"{n} has no ctypes signature in binding.py"
    assert set(B.SIGNATURES) == set(names)


def test_sm100a_code_only(B):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_null_handles(B):
    assert "sm_100a" in B.lora_version()
    assert B.lib.lora_server_destroy(None) == B.LORA_OK
    assert B.lib.lora_plan_destroy(None) == B.LORA_OK
    assert B.lib.lora_server_check(None, None) == B.LORA_ERR_INVALID_ARG
    assert isinstance(B.lora_last_error(None), str)


def test_create_rejects_bad_config_without_gpu(B):
    cfg = B.make_config([4096], [4096], [1], 12, 4)          # rank 12 unsupported
    with pytest.raises(B.LoraError) as e:
        B.lora_server_create(cfg)
    assert e.value.status in (B.LORA_ERR_UNSUPPORTED, B.LORA_ERR_CUDA)
    cfg = B.make_config([100], [4096], [1], 16, 4)           # width not a multiple of 64
    with pytest.raises(B.LoraError) as e:
        B.lora_server_create(cfg)
    assert e.value.status in (B.LORA_ERR_UNSUPPORTED, B.LORA_ERR_CUDA)


def test_shard_layout_host_logic(B):
    # counts[src][dst]; receive order is source-rank ascending
    counts = [0, 3, 2,
              1, 0, 4,
              5, 6, 7]
    so, ro = B.lora_shard_layout(counts, 3, 1)
    assert so == [0, 1, 1, 5]          # rank 1 sends 1 row to 0, 0 to 1, 4 to 2
    assert ro == [0, 3, 3, 9]          # rank 1 receives 3 from 0, 0 from itself, 6 from 2
    with pytest.raises(B.LoraError):
        B.lora_shard_layout(counts, 3, 3)
