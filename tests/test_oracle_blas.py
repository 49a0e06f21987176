"""oracle/blas.py (OpenBLAS x86-64 sdot restated) pinned bit-for-bit against numpy's own
float32 dot product on this host, for both micro-kernels (the other one selected through
OPENBLAS_CORETYPE in a subprocess).  CPU only."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = [1, 7, 31, 32, 33, 63, 64, 65, 95, 96, 100, 127, 1000, 4096, 4099, 65536 + 37]

_PROBE = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
from threadpoolctl import threadpool_info
from oracle import blas
arch = [i for i in threadpool_info() if i.get("internal_api") == "openblas"][0]["architecture"].lower()
kernel = {"skylakex": "openblas-skx", "cooperlake": "openblas-skx", "sapphirerapids": "openblas-skx",
          "haswell": "openblas-hsw", "zen": "openblas-hsw"}.get(arch)
rng = np.random.default_rng(11)
bad = []
for n in %r:
    for t in range(3):
        x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3)).astype(np.float32)
        y = rng.standard_normal(n).astype(np.float32)
        if blas.sdot(x, y, kernel) != x @ y or blas.norm(x, kernel) != float(np.linalg.norm(x)):
            bad.append(n)
print(json.dumps({"arch": arch, "kernel": kernel, "bad": bad}))
"""


@pytest.mark.parametrize("coretype", [None, "Haswell", "SkylakeX"])
def test_sdot_restatement_is_numpys_dot_bitwise(coretype):
    env = dict(os.environ, OPENBLAS_NUM_THREADS="4")
    if coretype:
        env["OPENBLAS_CORETYPE"] = coretype
    out = subprocess.run([sys.executable, "-c", _PROBE % (ROOT, SIZES)], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    if res["kernel"] is None:
        pytest.skip(f"host OpenBLAS kernel {res['arch']} has no restatement")
    assert res["bad"] == [], res
