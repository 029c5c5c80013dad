"""Golden TNS1 files written by the REFERENCE's tensor_write (src/core.py:93-117).

Run in the build container (where /root/reference exists):
    python tests/golden/make_tns1.py
Writes tests/golden/tns1_*.bin; the CPU tests check that this package
writes byte-identical files and reads them back exactly.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from moba.core import Tensor, tensor_write  # noqa: E402  (reference, read-only)

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(123)
CASES = {
    "tns1_f32_rank2": rng.standard_normal((7, 5)).astype(np.float32),
    "tns1_f64_rank3": rng.standard_normal((2, 3, 4)),
    "tns1_f64_rank1": rng.standard_normal(9),
}
for name, arr in CASES.items():
    tensor_write(Tensor(arr), os.path.join(HERE, name + ".bin"))
    print("wrote", name, arr.shape, arr.dtype)
