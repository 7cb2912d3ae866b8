"""GPU: the reference's parexec contract (test_parexec.py:29-99) against the
device objective and the device top-k, the scratch-ordering guarantee of
qpm_fitness_bits vs the host plugin path, and engine state guards.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import torch

    torch.cuda.set_device(0)
    import paper_2511_01255_b200 as pkg

    return pkg


def pattern_objective(q, n=16, mode="fast"):
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    return q.make_objective(spec, q.MismatchTable({1404.0: q.PhaseMismatchPair(0.3, 0.7)}), 1.0, n, mode=mode)


def signs_matrix(rows, n, seed=0):
    return O.random_population_matrix(rows, n, seed=seed)


class TestEvaluateBatch:
    def test_worker_counts_give_identical_results(self, q):
        obj = pattern_objective(q)
        items = signs_matrix(500, 16)
        ref = q.evaluate_batch(q.BatchJob(items=items, workers=1), obj)
        for workers in (2, 8, 64):
            assert np.array_equal(ref, q.evaluate_batch(q.BatchJob(items=items, workers=workers), obj))

    def test_chunk_size_does_not_change_results(self, q):
        obj = pattern_objective(q)
        items = signs_matrix(100, 16)
        ref = q.evaluate_batch(q.BatchJob(items=items, workers=1, chunk_size=100), obj)
        for chunk in (1, 7, 64):
            assert np.array_equal(ref, q.evaluate_batch(q.BatchJob(items=items, workers=3, chunk_size=chunk), obj))

    def test_single_item_equals_direct_call(self, q):
        obj = pattern_objective(q)
        items = signs_matrix(1, 16)
        assert q.evaluate_batch(q.BatchJob(items=items, workers=1), obj)[0] == obj(items[0])

    def test_repeat_evaluation_identical_and_exact_mode_bit_exact(self, q):
        obj = pattern_objective(q, 300, mode="exact")
        items = signs_matrix(64, 300, seed=4)
        a = q.evaluate_batch(q.BatchJob(items=items, workers=2), obj)
        b = q.evaluate_batch(q.BatchJob(items=items, workers=2), obj)
        assert np.array_equal(a, b)
        t = obj.tables[0]
        P = O.Problem("thg", t.e1[None], t.b[None], np.array([t.w]), np.array([t.hconst]), t.normalization)
        assert np.array_equal(a, O.evaluate_block(P, items))

    def test_failure_carries_item_index(self, q):
        """A row the device objective rejects (wrong length inside a list batch) is located."""
        obj = pattern_objective(q)
        items = [signs_matrix(1, 16, seed=i)[0] for i in range(10)]
        items[6] = np.ones(5, dtype=np.int8)
        with pytest.raises(q.BatchEvaluationError) as info:
            q.evaluate_batch(q.BatchJob(items=items, workers=4, chunk_size=3), obj)
        assert info.value.item_index == 6


class TestReduceBest:
    def test_basic_and_ties(self, q):
        assert q.reduce_best([3.0, 1.0, 2.0], 1) == [0]
        assert q.reduce_best([5.0, 5.0, 5.0], 2) == [0, 1]

    def test_matches_sort_oracle_large(self, q):
        vals = np.random.default_rng(99).random(100_000)
        want = sorted(range(len(vals)), key=lambda i: (-vals[i], i))
        for k in (4, 9, 33, 64):
            assert q.reduce_best(vals, k, workers=4, chunk_size=1000) == want[:k]

    def test_workers_chunks_invariant_with_ties(self, q):
        vals = np.random.default_rng(5).integers(0, 50, size=777).astype(float)
        want = [int(i) for i in np.lexsort((np.arange(vals.size), -vals))]
        for k in (1, 8, 10, 64):
            ref = q.reduce_best(vals, k, workers=1)
            assert ref == want[:k]
            for workers, chunk in ((2, 10), (4, 333), (8, 1)):
                assert q.reduce_best(vals, k, workers=workers, chunk_size=chunk) == ref

    def test_all_equal_and_k_equals_n(self, q):
        assert q.reduce_best(np.zeros(40), 40) == list(range(40))
        v = np.array([1.0, -np.inf, np.inf, 0.0, -0.0, 2.0])
        assert q.reduce_best(v, 6) == [int(i) for i in np.lexsort((np.arange(6), -v))]


def test_fitness_bits_ordered_with_host_path(q):
    """qpm_fitness_bits (caller's stream) and evaluate_block (the problem's host
    stream) share the problem's scratch; interleaved calls, including ones that
    grow it, give the serial values (the two paths were unordered)."""
    import torch

    obj = pattern_objective(q, 4000)
    signs = signs_matrix(512, 4000, seed=2)
    want = obj.evaluate_block(signs)
    bits = torch.zeros((512, obj.row_words), dtype=torch.int32, device="cuda")
    packed = np.packbits((signs < 0).astype(np.uint8), axis=1, bitorder="little")
    pad = np.zeros((512, obj.row_words * 4), dtype=np.uint8)
    pad[:, :packed.shape[1]] = packed
    bits.copy_(torch.from_numpy(pad.view(np.int32)))
    s = torch.cuda.Stream()
    for rows in (64, 512, 128, 512):
        out = torch.empty(rows, dtype=torch.float64, device="cuda")
        obj.evaluate_bits(bits[:rows], out, stream=s)
        host = obj.evaluate_block(signs[:rows // 2])
        s.synchronize()
        assert np.array_equal(out.cpu().numpy(), want[:rows])
        assert np.array_equal(host, want[:rows // 2])


def test_engine_init_twice_rejected(q):
    obj = pattern_objective(q, 64)
    eng = q.Engine(obj, "hybrid", pop_size=8, generations=3, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                   sch=q.Schedules())
    eng.init()
    from paper_2511_01255_b200._native import QpmError

    with pytest.raises(QpmError, match="twice"):
        eng.init()
    eng.step(3)
    assert eng.trace().shape == (4, 5)


def test_prepare_then_step_equals_plain_step(q):
    """prepare(n) only captures graphs: the run is the same as without it."""
    obj = pattern_objective(q, 700)
    out = []
    for prep in (False, True):
        eng = q.Engine(obj, "hybrid", pop_size=40, generations=25, seed=5, de=q.DEParams(), gwo=q.GWOParams(),
                       sch=q.Schedules())
        eng.init()
        eng.step(3)
        if prep:
            eng.prepare(22)
        eng.step(22)
        out.append(eng.trace())
    assert np.array_equal(out[0], out[1])
