"""The alternative attention pipelines (variant 3 = 64-key double-buffered S, variant 4 = P staged in
shared memory) the exp2 split knob and separate (unfused) Q/K/V gathers must give the same results as the default: the attention parity cases of
test_gpu_parity.py re-run in a subprocess with the switch set (the library reads it once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = "varblock_attention_parity or online_softmax_rescale or p1_equals_dense or fused_stagewise"


@pytest.mark.parametrize("env", [{"SVG2_ATTN_VARIANT": "3"}, {"SVG2_ATTN_VARIANT": "4"}, {"SVG2_EXP_POLY": "0"},
                                 {"SVG2_FUSE_GATHER": "0"}],
                         ids=["variant3", "variant4", "mufu_only_exp", "separate_gathers"])
def test_attention_variant_parity(env):
    full_env = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", CASES,
                        os.path.join(HERE, "test_gpu_parity.py")], env=full_env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
