"""Multi-rank row-slab path on CPU (gloo, world_size 2): each rank assembles
its slab (here with the CPU oracle standing in for the device), the slab
summaries are gathered through the package's verification collective, and
the combination equals the single-rank matrix."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, config, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.checkers import Oracle
    from paper_1905_05417_b200 import distributed as D
    from paper_1905_05417_b200 import problem as P
    prob = P.baseline_config(config)
    r, w, _ = D.env_rank()
    b = D.slab_for_rank(prob, r, w)  # functions [f_begin, f_end): cut inside a thickness row
    ns = prob.n_s
    t0, t1 = b["f_begin"] // ns, -(-b["f_end"] // ns)
    trp, tcols, tvals = Oracle().assemble(prob, "fast", t0, t1)
    a, e = 3 * (b["f_begin"] - t0 * ns), 3 * (b["f_end"] - t0 * ns)
    rp, cols, vals = trp[a:e + 1] - trp[a], tcols[trp[a]:trp[e]], tvals[trp[a]:trp[e]]
    assert rp[0] == 0 and int(rp[-1]) == b["nnz_end"] - b["nnz_begin"]
    s = D.slab_summary(torch.from_numpy(rp), torch.from_numpy(cols), torch.from_numpy(vals),
                       b["row_begin"], b["nnz_begin"])
    # the per-rank oracle comparison of one sampled thickness row (here of the
    # oracle's own slab: exactly 0)
    from oracle.checkers import slab_oracle_delta
    s = D.with_field(s, "oracle_rel_dk", slab_oracle_delta(prob, b["f_begin"], b["f_end"], torch.from_numpy(rp),
                                                            torch.from_numpy(cols), torch.from_numpy(vals)))
    assert float(s[D.FIELD_INDEX["oracle_rel_dk"]]) == 0.0
    parts = D.gather_summaries(s)
    full = D.gather_csr(torch.from_numpy(rp), torch.from_numpy(cols), torch.from_numpy(vals), dst=0)
    if rank == 0:
        q.put((D.combine_summaries(parts), tuple(t.numpy() for t in full)))
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("config", ["C1", "C2"])
def test_two_rank_slabs_reproduce_full_matrix(config, oracle):
    from paper_1905_05417_b200 import distributed as D
    from paper_1905_05417_b200 import problem as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, config, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    prob = P.baseline_config(config)
    rp, cols, vals = oracle.assemble(prob, "fast")
    full = D.combine_summaries([D.slab_summary(torch.from_numpy(rp), torch.from_numpy(cols),
                                               torch.from_numpy(vals))])
    assert got["rows"] == full["rows"] == prob.dim
    assert got["nnz"] == full["nnz"] == P.sizes(prob)["nnz"]
    assert got["fro_sq"] == pytest.approx(full["fro_sq"], rel=1e-13)
    assert got["checksum"] == pytest.approx(full["checksum"], rel=1e-12)
    assert got["max_abs"] == full["max_abs"]
    assert got["pattern_hash"] == full["pattern_hash"]
    assert got["oracle_rel_dk"] == 0.0
    # the full-slab gather reassembles the single-rank matrix exactly
    assert np.array_equal(gathered[0], rp) and np.array_equal(gathered[1], cols)
    assert np.array_equal(gathered[2], vals)


def test_pattern_hash_is_additive_and_sensitive(oracle):
    """The slab pattern hashes sum (mod p) to the full matrix's for any cut,
    and a single moved column or shifted row offset changes the hash."""
    from paper_1905_05417_b200 import distributed as D
    from paper_1905_05417_b200 import problem as P
    import paper_1905_05417_b200 as lf
    prob = P.baseline_config("C1")
    rp, cols, _ = oracle.assemble(prob, "fast")
    rp_t, c_t = torch.from_numpy(rp), torch.from_numpy(cols)
    full = D.pattern_hash(rp_t, c_t)
    for parts in (2, 3):
        tot = 0
        for k in range(parts):
            b = lf.slab_bounds(prob, parts, k)
            r0, r1 = b["row_begin"], b["row_end"]
            z0, z1 = int(rp[r0]), int(rp[r1])
            tot += D.pattern_hash(torch.from_numpy(rp[r0:r1 + 1] - z0), c_t[z0:z1], r0, z0, chunk=1000)
        assert tot % D.HASH_P == full
    bad = c_t.clone()
    bad[12345] += 1
    assert D.pattern_hash(rp_t, bad) != full
    bad_rp = rp_t.clone()
    bad_rp[77] += 1
    assert D.pattern_hash(bad_rp, c_t) != full
