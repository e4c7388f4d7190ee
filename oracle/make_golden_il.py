"""TEST-FIXTURE GENERATOR (run here, where /root/reference is mounted).
Writes tests/golden/il/<name>.json = {"il": ilToJson(IL), "tenv": ..., "kernel":
kernelToJson(reindex(IL, tenv))} from the UNMODIFIED reference compiled by
oracle/Makefile (oracle/_ref/libcltkref.so): the IL of every golden contract
before and after cutPayoff (proj/src/compile.cpp), so the engine's own reindex
(csrc/reindex.cpp, restating proj/src/kernel.cpp:14-180) can be checked
node for node against the reference's.

    python oracle/make_golden_il.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from make_golden import CONTRACTS  # noqa: E402
from oracle_py import Ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "il")
# extra template environments for the template contract (windows / shifts bound
# to other values give other row layouts)
EXTRA_TENV = {"template-option": [{"t0": 0, "t1": 1}, {"t0": 30, "t1": 400}]}


def main() -> None:
    sys.setrecursionlimit(1_000_000)
    ref = Ref()
    os.makedirs(OUT, exist_ok=True)
    for name, (path, tenv) in CONTRACTS.items():
        src = open(path).read()
        for cut in (True, False):
            if name == "brc" and not cut:
                continue  # the uncut BRC IL is ~1 MB of JSON; the cut one covers it
            il = ref.compile_il(src, cut=cut)
            envs = [tenv] + EXTRA_TENV.get(name, [])
            for i, te in enumerate(envs):
                k = ref.reindex(il, te)
                tag = f"{name}{'' if cut else '_nocut'}{'' if i == 0 else f'_t{i}'}"
                with open(os.path.join(OUT, tag + ".json"), "w") as f:
                    json.dump({"il": il, "tenv": te, "kernel": k}, f, sort_keys=True)
                print(tag, len(json.dumps(il)), "IL bytes,", len(k["rows"]), "rows")


if __name__ == "__main__":
    main()
