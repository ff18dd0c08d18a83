"""Host logic of bench.py (no GPU): the rank -> source-range split of weak and strong scaling."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def test_strong_scaling_partitions_the_instance():
    for name in ("100M_x_100k", "powerlaw", "tiny"):
        for world in (1, 2, 3, 4, 8):
            ranges = [bench.shard_range(name, world, r, "strong") for r in range(world)]
            full = ranges[0][0]
            assert all(cfg == full for cfg, _, _ in ranges)           # one instance for every rank
            assert ranges[0][1] == 0 and ranges[-1][2] == full.num_sources
            for (_, a0, a1), (_, b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0 and a0 < a1                            # contiguous, disjoint, nonempty
            sizes = [s1 - s0 for _, s0, s1 in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_weak_scaling_grows_the_instance():
    for name in ("1M_x_10k", "tiny"):
        base = bench.shard_range(name, 1, 0, "weak")[0]
        for world in (2, 4, 8):
            ranges = [bench.shard_range(name, world, r, "weak") for r in range(world)]
            full = ranges[0][0]
            assert full.num_sources == world * base.num_sources and full.seed == base.seed
            assert [(s0, s1) for _, s0, s1 in ranges] == [(r * base.num_sources, (r + 1) * base.num_sources)
                                                          for r in range(world)]


def test_default_workload_is_the_metric_config():
    # BASELINE.json configs[2] carries the metric's 1/2/4/8-GPU numbers; strong scaling by default
    assert bench.WORKLOAD == "100M_x_100k"
    assert bench.WORKLOADS[bench.WORKLOAD][0] == 2 and bench.WORKLOADS[bench.WORKLOAD][5] == "strong"
