"""Forward progress of the cross-CTA waits (the invariants at stake are the
table / refcount audit, which a hung or torn round would violate).

Stage 1's fused fill sums the counts every earlier work item published, and segmentation's
decoupled look-back waits on earlier tiles. Both take their work from atomic tickets, so a
waiter only ever waits on items already claimed by running CTAs. The regression case is the
round-1 hang: Stage-1 thread-block clusters forced to 8 CTAs per current step (more clusters
launched than can be co-resident: 8-CTA clusters must fit inside one GPC) with the fused fill,
in LAST and RANGE rounds. Environment knobs are read once per process, so each case runs in a
child process under a timeout; the child runs the full oracle parity check.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CHILD = os.path.join(HERE, "_progress_child.py")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("cluster,case", [(8, "last_many"), (8, "range"), (4, "range"), (8, "last_long_step")])
def test_forced_clusters_make_progress(cluster, case):
    env = dict(os.environ, MEMSHARE_S1_CLUSTER=str(cluster))
    r = subprocess.run([sys.executable, CHILD, case], env=env, cwd=os.path.dirname(HERE), timeout=300,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ok" in r.stdout


def test_segmentation_and_stage1_under_a_competing_persistent_kernel():
    """All but 8 SMs are held by another stream's spinning kernel while the round runs: with
    a static CTA -> item map the look-back / prefix waits would depend on CTAs that cannot be
    scheduled; with tickets the round completes and matches the oracle."""
    r = subprocess.run([sys.executable, CHILD, "contended"], env=dict(os.environ, CUDA_MODULE_LOADING="EAGER"),
                       cwd=os.path.dirname(HERE),
                       timeout=300, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ok" in r.stdout
