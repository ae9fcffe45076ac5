"""Host concurrency of the binding and the C ABI: two host threads factor and sweep different
matrices at the same time on their own CUDA streams (one context per thread; the POTRF panel
stream of the device is shared and its enqueue serialised). Every result must be bitwise equal
to the same call made alone (the kernels are deterministic), and the caller's current device is
left as it was."""
import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch(cuda_device):
    import torch as t
    return t


def run_one(torch, g, seed, stream=None):
    import paper_2405_14892_b200 as mvn
    cfg = W.small_config(f"thr{g}", g, 400, 2, base="B")
    inp = W.make_inputs(cfg)
    order, a, _ = mvn.mvn_marginal_order(inp.mu, np.full(cfg.n, cfg.sigma2 + cfg.nugget), cfg.u)
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
    with ctx:
        T = mvn.mvn_cov_matern(torch.from_numpy(np.ascontiguousarray(inp.xy[order])).cuda(), cfg.sigma2, cfg.beta,
                               cfg.nu, cfg.nugget)
        info = mvn.mvn_potrf(T, cfg.n)
        M, S = mvn.mvn_sov_prefix(T, cfg.n, torch.from_numpy(a).cuda(), cfg.N, cfg.R, seed)
        torch.cuda.current_stream().synchronize()
    return info, T.cpu().numpy(), M.cpu().numpy(), S.cpu().numpy()


def test_two_threads_bitwise_equal_to_alone(torch):
    ref = {g: run_one(torch, g, 7) for g in (40, 47)}
    out = {}
    errs = []

    def worker(g):
        try:
            for _ in range(3):
                out[g] = run_one(torch, g, 7, torch.cuda.Stream())
        except Exception as e:      # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(g,)) for g in (40, 47)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for g in (40, 47):
        assert out[g][0] == ref[g][0] == -1
        for x, y in zip(out[g][1:], ref[g][1:]):
            assert np.array_equal(x, y)
    assert torch.cuda.current_device() == 0


def test_thread_contexts_are_freed(torch):
    """A thread's contexts go with its thread-local storage (mvn_destroy frees their workspace)."""
    import gc
    import paper_2405_14892_b200 as mvn
    gc.collect()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    seen = []

    def worker():
        c = mvn.Context.get(0)
        seen.append(c.h.value)
        run_one(torch, 47, 7, torch.cuda.Stream())

    for _ in range(3):
        t = threading.Thread(target=worker)
        t.start()
        t.join()
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free1, _ = torch.cuda.mem_get_info()
    assert len(seen) == 3
    assert free0 - free1 < (256 << 20), (free0, free1)    # no per-thread workspace left behind
