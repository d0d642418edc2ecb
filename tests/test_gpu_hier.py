"""The G-rank reducer (paper_2208_14228_b200.hier) on one B200 with G simulated ranks.

Each simulated rank has its own slots, replica and stream; cross-rank reads
and writes go through raw pointers exactly as peer/IPC pointers would.  The
result must equal the single-GPU reducer bit for bit, and every replica must
be identical -- for the hierarchical RankTree(2) and the owner-computes
parity variants (Sequential, rotated Tree(2)).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def adversarial(E, n, seed, dtype):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (E, n)) * 10.0 ** rng.integers(-12, 13, (E, n))).astype(dtype)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("E,G", [(8, 2), (8, 4), (8, 8), (16, 4), (64, 8), (32, 2)])
@pytest.mark.parametrize("variant", ["rank_tree2", "sequential", "tree2_rotated"])
def test_group_reducer_equals_single_gpu(oracle, dtype, E, G, variant):
    from paper_2208_14228_b200.hier import GroupReducer, RankBuffers

    n = 40_003
    grads = adversarial(E, n, 100 + E + G, dtype)
    p0 = adversarial(1, n, 7, dtype)[0]
    v0 = adversarial(1, n, 8, dtype)[0]
    rot = None
    if variant == "tree2_rotated":
        rot = oracle.rotation_table(oracle.buckets_initial(n, 64), E, n)
    fan = "seq" if variant == "sequential" else "tree2"
    want_p, want_v = oracle.reduce_update(grads, rot, fan, p0, v0, 0.02, 0.9)
    E_loc = E // G
    ranks = []
    for g in range(G):
        ranks.append(RankBuffers(torch.from_numpy(grads[g * E_loc:(g + 1) * E_loc].copy()).cuda(),
                                 torch.from_numpy(p0.copy()).cuda(), torch.from_numpy(v0.copy()).cuda(),
                                 torch.cuda.Stream()))
    red = GroupReducer(ranks, E, variant, None if rot is None else torch.from_numpy(rot).cuda(), 0.02, 0.9)
    red.step()
    torch.cuda.synchronize()
    red.check()
    for r in ranks:
        assert np.array_equal(r.param.cpu().numpy().view(np.uint8), want_p.view(np.uint8))
        assert np.array_equal(r.vel.cpu().numpy().view(np.uint8), want_v.view(np.uint8))


def test_group_reducer_repeated_steps_stay_identical(oracle):
    from paper_2208_14228_b200.hier import GroupReducer, RankBuffers

    E, G, n = 16, 4, 10_000
    grads = adversarial(E, n, 3, np.float32)
    p = adversarial(1, n, 4, np.float32)[0]
    v = np.zeros(n, np.float32)
    ranks = [RankBuffers(torch.from_numpy(grads[g * 4:(g + 1) * 4].copy()).cuda(), torch.from_numpy(p.copy()).cuda(),
                         torch.from_numpy(v.copy()).cuda(), torch.cuda.Stream()) for g in range(G)]
    red = GroupReducer(ranks, E, "rank_tree2", None, 0.1, 0.9)
    for _ in range(5):
        red.step()
        p, v = oracle.reduce_update(grads, None, "tree2", p, v, 0.1, 0.9)
    torch.cuda.synchronize()
    for r in ranks:
        assert np.array_equal(r.param.cpu().numpy(), p) and np.array_equal(r.vel.cpu().numpy(), v)


@pytest.mark.parametrize("variant", ["rank_tree2", "sequential"])
def test_group_reducer_non_finite_leaves_every_replica(variant):
    """A non-finite synchronized gradient in ONE rank's shard: no rank commits its shard (the shard
    status words are exchanged before the update), every replica keeps its bytes, every rank raises."""
    from paper_2208_14228_b200.errors import NumericError
    from paper_2208_14228_b200.hier import GroupReducer, RankBuffers

    E, G, n = 8, 4, 10_000
    grads = adversarial(E, n, 12, np.float32)
    grads[5, 9_001] = np.inf  # lands in the last rank's parameter shard
    p = adversarial(1, n, 13, np.float32)[0]
    v = adversarial(1, n, 14, np.float32)[0]
    ranks = [RankBuffers(torch.from_numpy(grads[g * 2:(g + 1) * 2].copy()).cuda(), torch.from_numpy(p.copy()).cuda(),
                         torch.from_numpy(v.copy()).cuda(), torch.cuda.Stream()) for g in range(G)]
    red = GroupReducer(ranks, E, variant, None, 0.1, 0.9)
    red.step()
    torch.cuda.synchronize()
    for r in ranks:
        assert np.array_equal(r.param.cpu().numpy(), p) and np.array_equal(r.vel.cpu().numpy(), v)
    for f in red.flags:
        assert f.status()[0] == 5
    with pytest.raises(NumericError):
        red.check()
