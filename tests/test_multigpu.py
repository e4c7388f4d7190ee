"""Multi-GPU pricing on the device (run on one B200 here; the N-GPU cases
skip unless the box has them).

Two paths shard the reference's runParallel chunks (proj/src/pricing.cpp:
268-286) over GPUs with bit-identical results for any GPU count:
  * one process, several GPUs, through the C ABI (cltk_options.devices,
    $CLTK_DEVICES): ncclAllGather of the chunk-partial slices over NVLink
    (a device listed twice shares its GPU and is gathered with device
    copies -- how the sharding logic is tested on one GPU);
  * one process per GPU (distributed.DistributedPricer): here two gloo ranks
    that both price on cuda:0 -- their kernels never wait on each other, the
    collective is the host-side all-gather of the partials slots.
"""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2108_03076_b200 as E
from conftest import ROOT, load_kernel, load_model

pytestmark = pytest.mark.gpu

CASES = [("worst-off", "three", [0, 100], 300_001), ("brc", "three", [0], 40_000),
         ("european-call", "call", [0], 1_000_003)]


@pytest.mark.parametrize("kern,model,days,paths", CASES)
@pytest.mark.parametrize("jit", [False, True])
def test_device_list_is_bitwise_one_gpu(kern, model, days, paths, jit):
    k = load_kernel(kern)
    m = load_model(model)
    one = E.price(k, m, paths, 17, days, jit=jit)
    for devs in ([0], [0, 0], [0, 0, 0], [0] * 8):
        got = E.price(k, m, paths, 17, days, jit=jit, devices=devs)
        assert got == one, devs


def test_device_list_template_batch_bitwise():
    k = load_kernel("worst-off")
    m = load_model("three")
    base = E.kernel_literals(k)
    lits = [[v * (1.0 + 0.01 * i) if v == 0.75 else v for v in base] for i in range(5)]
    one = E.price_template(k, lits, m, 50_000, 3, [0, 50])
    assert E.price_template(k, lits, m, 50_000, 3, [0, 50], devices=[0, 0, 0]) == one


def test_cltk_devices_environment_shards_the_plain_entry_point():
    """$CLTK_DEVICES shards cltk_gpu_price (the entry the reference-side C++
    shim calls) without any code change; the result is the same bits."""
    code = ("import json, sys; sys.path.insert(0, %r); sys.path.insert(0, %r);"
            "import paper_2108_03076_b200 as E; from conftest import load_kernel, load_model;"
            "print(json.dumps(E.price(load_kernel('worst-off'), load_model('three'), 200000, 5,"
            " [0, 30])))" % (ROOT, os.path.join(ROOT, "tests")))
    outs = []
    for env in ("", "0,0", "0,0,0,0"):
        e = dict(os.environ, CLTK_DEVICES=env) if env else {
            k: v for k, v in os.environ.items() if k != "CLTK_DEVICES"}
        r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1] == outs[2]
    e = dict(os.environ, CLTK_DEVICES="0,x")
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode != 0 and "CLTK_DEVICES" in r.stderr


def test_nccl_is_loadable():
    v = E.nccl_version()
    assert v >= 22700, v  # 2.27+ (the system's 2.27.3 or torch's 2.28)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2+ GPUs")
def test_distinct_devices_nccl_allgather_bitwise():
    n = torch.cuda.device_count()
    k = load_kernel("brc")
    m = load_model("three")
    one = E.price(k, m, 200_000, 42, [0])
    assert E.price(k, m, 200_000, 42, [0], devices=list(range(n))) == one
    assert E.price(k, m, 200_000, 42, [0], devices=[1, 0]) == one


def test_device_list_domain_error_lowest_path_wins():
    """A fault in the second shard surfaces as the reference's error once the
    shards' error words merge by MIN (what runGroup and the distributed
    finalize do)."""
    k = E.Kernel(load_kernel("worst-off"))
    m = load_model("three")
    # plan-level: two plans on cuda:0 pricing the two halves, words merged by MIN
    p0 = E.Plan(k, m, [0], fault=True)
    p1 = E.Plan(k, m, [0], fault=True)
    paths = 100_000
    _, nc = p0.chunking(paths)
    s = (nc + 1) // 2
    bufs = [torch.zeros(2 * s * 3, dtype=torch.float64, device="cuda") for _ in range(2)]
    st = torch.cuda.current_stream().cuda_stream
    p1.set_fault(paths - 3, 4)  # in plan 1's slice
    p0.launch(paths, 1, 0, s, bufs[0].data_ptr(), st)
    p1.launch(paths, 1, s, nc, bufs[1].data_ptr(), st)
    w = min(p0.error_word(st), p1.error_word(st))
    assert w >> 24 == paths - 3
    p0.set_error_word(w, st)
    with pytest.raises(E.ContractError, match="invNormalCdf domain error"):
        p0.finalize(paths, 1, bufs[0].data_ptr(), st)


def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _rank(rank, world, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from paper_2108_03076_b200.distributed import DistributedPricer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for name, model, days, paths in CASES:
            for jit in (False, True):
                p = DistributedPricer(E.Kernel(load_kernel(name)), load_model(model), days,
                                      device=0, jit=jit)
                res[(name, jit)] = p.price(paths, 17)
        # a domain error in the LAST rank's shard surfaces on every rank
        p = DistributedPricer(E.Kernel(load_kernel("worst-off")), load_model("three"), [0],
                              device=0, fault=True)
        paths = 100_000
        c0, c1 = p.shard(paths)
        if rank == world - 1:
            p.plan.set_fault(paths - 1, 14)
        try:
            p.price(paths, 17)
            res["fault"] = None
        except E.ContractError as e:
            res["fault"] = (e.code, str(e))
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_pricer_world_bitwise_and_errors(world):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(world, _free_port(), out), nprocs=world, join=True)
    for name, model, days, paths in CASES:
        for jit in (False, True):
            one = E.price(load_kernel(name), load_model(model), paths, 17, days, jit=jit)
            for r in range(world):
                assert out[r][(name, jit)] == one, (name, jit, r)
    for r in range(world):
        assert out[r]["fault"] == (5, "invNormalCdf domain error"), r
