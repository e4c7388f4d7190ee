"""GPU `cltk price` CLI (python -m paper_2108_03076_b200 price), mirroring the
reference CLI's price subcommand (proj/tools/cli.cpp:155-162, 246-259)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import GOLD, ROOT


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2108_03076_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_cli_parse_error_convention(tmp_path):
    bad = tmp_path / "bad.kernel"
    bad.write_text("this is not a kernel\n")
    r = _run("price", str(bad), "--model", os.path.join(GOLD, "models", "call.json"))
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert r.stderr.startswith("error: ")
    assert r.stdout == ""


def test_cli_missing_model_is_eval_error(tmp_path):
    r = _run("price", os.path.join(GOLD, "kernels", "european-call.kernel"), "--model",
             str(tmp_path / "missing.json"))
    assert r.returncode == 5 and r.stderr.startswith("error: ")


@pytest.mark.gpu
def test_cli_prices_like_the_api():
    import paper_2108_03076_b200 as E
    kern = os.path.join(GOLD, "kernels", "worst-off.kernel")
    model = os.path.join(GOLD, "models", "three.json")
    r = _run("price", kern, "--model", model, "--paths", "20000", "--seed", "7", "--at", "0",
             "100", "--threads", "4")
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    want = E.price(E.load_kernel(kern), json.load(open(model)), 20000, 7, [0, 100])
    assert [o["price"] for o in out] == [w["price"] for w in want]
    assert [o["stdError"] for o in out] == [w["std_error"] for w in want]
    assert [o["valuationDay"] for o in out] == [0, 100]
    assert set(out[0]) == {"price", "stdError", "paths", "seed", "valuationDay"}
    r2 = _run("price", kern, "--model", model, "--paths", "20000", "--seed", "7", "--at", "0",
              "100", "--jit", "1")
    assert json.loads(r2.stdout) == out
    # sharded over a device list (one GPU listed twice here): the same bits
    r3 = _run("price", kern, "--model", model, "--paths", "20000", "--seed", "7", "--at", "0",
              "100", "--devices", "0,0")
    assert r3.returncode == 0, r3.stderr
    assert json.loads(r3.stdout) == out
