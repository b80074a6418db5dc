"""VFT1 fixtures written by the REFERENCE writer (src/tensor_io.py:44-55), run here where
/root/reference exists: `python tests/golden/make_vft1.py`. tests/test_vft1.py checks that this
repo's reader returns the same arrays and its writer produces byte-identical files."""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from vfa_lab.tensor_io import DTYPE_F32, DTYPE_F64, write_matrix  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "vft1")
rng = np.random.default_rng(2604)
m = rng.normal(size=(9, 6))
write_matrix(os.path.join(HERE, "m_f64.vft"), m, DTYPE_F64)
write_matrix(os.path.join(HERE, "m_f32.vft"), m, DTYPE_F32)
np.save(os.path.join(HERE, "m.npy"), m)
# a tiny q/k/v dump directory in the layout `vfa-lab run --data` reads (src/cli.py:213-221)
import torch  # noqa: E402

qkv = torch.from_numpy(rng.normal(size=(3, 256, 64))).to(torch.bfloat16).double().numpy()  # bf16 values
for name, x in zip("qkv", qkv):
    write_matrix(os.path.join(HERE, f"{name}.vft"), x, DTYPE_F64)

# reference `run` reports + outputs on that dump (src/cli.py:383-407), for the GPU runner tests
import json  # noqa: E402

from vfa_lab.cli import main as ref_main  # noqa: E402

for variant, extra in (("vfa", []), ("blasst_fa4", ["--lambda", "0.001", "--tau", "2.0"]),
                       ("vsa", ["--lambda", "0.01"])):
    report = os.path.join(HERE, f"ref_run_{variant}.json")
    rc = ref_main(["run", "--data", HERE, "--variant", variant, "--q-block", "128", "--k-block", "64",
                   "--causal", "--report", report, *extra])
    assert rc == 0, rc
