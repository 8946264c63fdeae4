"""N>1 path on CPU: two gloo ranks run bench.py's sharding/aggregation logic
(rank_shard + sum_checksums + max-over-ranks timing) with the oracle standing
in for the per-rank kernel, and the stitched result must equal the
single-process transform of the whole stream.  No collective is on the data
path: only scalars (checksums, timings) cross ranks."""
from __future__ import annotations

import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    from paper_1403_7295_b200 import paes

    O = oracle.Oracle()
    d = bench.Dist(world, backend="gloo")
    sh = bench.rank_shard(total, world, rank, paes.plan_chunks)
    key = O.sweep(3, 16)
    pt = O.counter_fill(3, sh["offset"], sh["raw_len"])
    ct = O.encrypt_chunk(pt, sh["is_final"], key) if sh["raw_len"] or sh["is_final"] else b""
    assert len(ct) == sh["padded_len"]
    cs = O.checksum(ct[: len(ct) - len(ct) % 8], sh["offset"] // 8)
    total_cs = bench.sum_checksums(d, cs)
    t_max = d.reduce(float(rank + 1), "max")
    n_all = d.reduce(int(sh["raw_len"]), "sum")
    per_rank = d.gather(float(10 * rank + 1))  # bench.py's per-rank fields
    with open(os.path.join(out_dir, f"r{rank}.bin"), "wb") as f:
        f.write(ct)
    with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
        f.write(f"{total_cs} {t_max} {n_all} {','.join(str(x) for x in per_rank)}")
    d.barrier()
    d.close()


@pytest.mark.parametrize("total", [1 << 20, (1 << 20) + 8, 4096 * 3 + 16])
def test_two_rank_shards_stitch_to_whole(tmp_path, total, orc):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), total, str(tmp_path)), nprocs=world, join=True)
    key = orc.sweep(3, 16)
    whole = orc.encrypt_chunk(orc.counter_fill(3, 0, total), True, key)
    stitched = b"".join((tmp_path / f"r{r}.bin").read_bytes() for r in range(world))
    assert stitched == whole  # output offsets == input offsets: no assemble step
    want_cs = orc.checksum(whole[: len(whole) - len(whole) % 8], 0)
    for r in range(world):
        cs, tmax, n_all, per_rank = (tmp_path / f"r{r}.txt").read_text().split()
        assert [float(x) for x in per_rank.split(",")] == [1.0, 11.0]
        assert int(cs) == want_cs
        assert float(tmax) == 2.0
        assert int(n_all) == total
