"""Several pools in one process, driven from several host threads at once (e.g. two engine replicas sharing a GPU):
each pool's bytes, tables and counters must equal its own oracle's.  The binding's ctypes calls release the GIL, so
the library's calls of different pools really run concurrently (its only process-wide state is the per-device cache
of the TMA kernels' shared-memory attribute, kernels.cu).  Header contract: one pool = one writer."""
import threading

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import BytesStore, OraclePool  # noqa: E402
from workloads import content  # noqa: E402
from workloads.replay import Replayer  # noqa: E402
from workloads.scripts import fuzz_script  # noqa: E402

from test_gpu_parity import compare_full, compare_live_host, dev_pool  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _drive(tid, mode, seed, errors):
    try:
        L, H, D, N, S, T = 6, 4, 128, 48, 24, 16
        pool0 = content.pool_bytes(seed, L, N, T, H, D)
        o = OraclePool(N, S, n_classes=2, max_agents=1024, store=BytesStore(pool0, S))
        c = dev_pool(L, H, D, N, S, mode, ncls=2, seed=seed, staging=3 * 2 * L * T * H * D * 2)
        ro, rc = Replayer(o), Replayer(c)
        ops = fuzz_script(700 + seed, n_ops=240, n_agents=4, n_classes=2, N=N, max_alloc=6, gradual=True,
                          retire=True, lags=(1, 2))
        for i, op in enumerate(ops):
            a, b = ro.step(op), rc.step(op)
            assert a == b, (tid, i, op, a, b)
            if op[0] in ("offload", "offload_batch") and a[0] == 0:
                compare_live_host(o, c, f"thread {tid} op {i}")
            if op[0] == "sync":
                compare_full(o, c, f"thread {tid} op {i}")
        c.sync()
        compare_full(o, c, f"thread {tid} end")
        c.close()
    except BaseException as e:  # noqa: BLE001 - reported by the main thread
        errors.append((tid, repr(e)))


@pytest.mark.parametrize("modes", [("staged", "staged_tma", "direct_default", "auto"),
                                   ("staged_tma4", "staged_tma4", "staged_tma4", "staged_tma4")])
def test_pools_on_concurrent_threads(modes):
    errors = []
    th = [threading.Thread(target=_drive, args=(t, m, t + 1, errors)) for t, m in enumerate(modes)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a pool thread hung"
    assert not errors, errors
