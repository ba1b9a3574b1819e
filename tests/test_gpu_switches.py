"""Non-default kernel paths selected by environment switches (read once per
process, so each case runs the relevant tests in a child pytest): the
fallbacks must stay at the same parity bar as the defaults."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    # (env, tests): non-persistent tcgen05 GEMMs (which also restores the concurrent
    # scoring streams); in-kernel fp32 split for the mixed
    # prefill; mma.sync split attention in mixed scoring; one Q tile per CTA for the
    # split tcgen05 attention, two for the bf16 one
    ({"PPOEXP_GEMM_PERSIST": "0"}, "tests/test_gpu_parity.py::test_mixed_scoring_many_rows"),
    ({"PPOEXP_PREFILL_PLANES": "0"}, "tests/test_gpu_parity.py::test_mixed_scoring_many_rows"),
    ({"PPOEXP_ATTN_SPLIT_TC": "0"}, "tests/test_gpu_parity.py::test_mixed_scoring_many_rows"),
    ({"PPOEXP_ATTN_QT": "1"}, "tests/test_gpu_kernels.py::test_attention_prefill_split_tc_vs_fp64"),
    ({"PPOEXP_ATTN_QT": "2"}, "tests/test_gpu_kernels.py::test_attention_prefill_vs_torch"),
    # policy / reference / critic scoring forwards on three concurrent streams
    ({"PPOEXP_SCORE_STREAMS": "1"}, "tests/test_gpu_parity.py::test_mixed_experience_c2_full_depth"),
]


@pytest.mark.parametrize("env,target", CASES, ids=[",".join(f"{k}={v}" for k, v in e.items()) for e, _ in CASES])
def test_switch_paths(env, target):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", target], cwd=ROOT,
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
