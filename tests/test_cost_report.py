"""CPU: the executed-plan cost algebra and the compare report schema."""
from paper_2110_09524_b200 import cost


def test_measured_from_counters_matches_closed_forms():
    V, E, h, f = 7, 31, 2, 4
    c = [0] * 10
    c[0], c[1] = E, V  # K2
    c[6], c[7] = E, V  # K4f
    c[8], c[9] = V, 1  # LP rows
    m = cost.measured_from_counters(c, h, f)
    assert m["flops"] == cost.gat_executed_flops(V, E, h, f) == 4 * V * f * h + 2 * E * h
    assert m["io_units"] == cost.gat_executed_io(V, E, h, f)


def test_compare_report_schema_and_spec_examples():
    rep = cost.compare_report(3, 3, 1, 2, {"max_in": 2, "mean_in": 1.0})
    assert set(rep) == {"version", "config", "graph", "results"}
    assert [r["opt"] for r in rep["results"]] == ["none", "reorg", "reorg+fusion", "all"]
    for r in rep["results"]:
        assert {"opt", "mapping", "flops", "io_units", "peak_mem_units", "wall_ms", "checks"} <= set(r)
    # SPEC.md:287-289 (G3, f = 2, h = 1)
    assert [r["flops"] for r in rep["results"]] == [39, 30, 30, 30]
    assert rep["results"][0]["io_units"] == 45 and rep["results"][2]["io_units"] == 33
    # memory: fusion+recompute keeps no per-edge state: strictly less
    # whenever |E| > |V| (criterion 10)
    assert rep["results"][3]["peak_mem_units"] <= rep["results"][2]["peak_mem_units"]
    big = cost.compare_report(3, 6, 1, 2, {})
    assert big["results"][3]["peak_mem_units"] < big["results"][2]["peak_mem_units"]
    gap = lambda r: r["results"][2]["peak_mem_units"] - r["results"][3]["peak_mem_units"]  # noqa: E731
    assert gap(big) - gap(rep) == 2 * (6 - 3) * 1  # the gap grows by 2 h per added edge
