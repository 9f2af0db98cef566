"""Diagnostic: repeat the 3-layer aggregate-first fused step vs the oracle."""
import sys
import os
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from conftest import load_golden, make_g2  # noqa
import test_gpu_fused as T  # noqa
from paper_2601_04707_b200._lib import lib  # noqa

pdl = int(os.environ.get("PDL", "1"))
lib().mq_set_pdl(pdl)
n = int(os.environ.get("REPS", "5"))
gs = load_golden("sampling.npz")
fails = 0
for i in range(n):
    try:
        T._fused_vs_oracle(make_g2(gs), (6, 4, 3), 32, 200, 5, gs["g2/mask10"], windows=4, layer0="af")
    except AssertionError as e:
        fails += 1
        print("FAIL", i, str(e)[:200])
print(f"pdl={pdl} reps={n} fails={fails}")
