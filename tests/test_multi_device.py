"""Single-process multi-device res_y (ckb_init_devices + ckb_biv_resultant_multi,
SURVEY §5/§8e): contexts sharing the one GPU of the test box exercise the
sharding, the exchange (peer copies between contexts) and the coefficient-
sharded CRT bit-exactly; NCCL is used when the devices are distinct."""

import json
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.gpu
@pytest.mark.parametrize("devices,exchange,zero_copy", [("0,0", None, True), ("0,0,0", None, True),
                                                        ("0,0,0,0,0,0,0,0", None, True), ("0,0,0", "copy", True),
                                                        ("0,0,0,0", None, False)])
def test_multi_context_resultants_bit_exact(devices, exchange, zero_copy):
    """Default: the exchange folded into the interpolation (every context stores its
    residues straight into the owning context's CRT input) and each context's rows
    written into the page-locked result by its carry kernel; CKB_EXCHANGE=copy: the
    separate peer-copy step; CKB_ZERO_COPY=0: D2H copies of the rows."""
    env = dict(os.environ, CKB_DEVICES=devices)
    env.pop("CKB_GPUS", None)
    env.pop("CKB_EXCHANGE", None)
    env.pop("CKB_ZERO_COPY", None)
    if exchange:
        env["CKB_EXCHANGE"] = exchange
    if not zero_copy:
        env["CKB_ZERO_COPY"] = "0"
    r = subprocess.run([sys.executable, os.path.join(HERE, "helpers", "multi_ctx_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["contexts"] == len(devices.split(",")) and rep["launches"] > 0
    assert rep["nccl"] is False  # one physical device: no NCCL communicators
    assert rep["exchange"] == ("peer-copy" if exchange == "copy" else "peer-store"), rep


def test_multi_abi_declared():
    from paper_1201_1548_b200 import _lib
    lib = _lib.load()
    for name in ("ckb_init_devices", "ckb_devices", "ckb_biv_resultant_multi", "ckb_last_exchange"):
        assert hasattr(lib, name)


def test_bench_gpus_without_enough_devices_exits_nonzero():
    """bench.py --gpus N outside torchrun drives N devices from one process; with
    fewer visible devices it must fail loudly instead of timing one GPU."""
    repo = os.path.dirname(HERE)
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "1"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "CUDA device" in r.stderr
    assert r.stdout.strip() == ""
