"""The reference CLI's bench suites on the B200 engine (paper_2411_15332_b200.bench_modes;
qcsim_cli.cpp:84-239): rows, counters and statuses as the reference reports
them; the rh-signs counters equal the reference's own rh_mvm statistics."""
import numpy as np
import pytest


def test_table2_counts_equal_reference_rh_stats():
    """CPU: the Table-2 sign counts the suite asserts equal the compiled reference's RhMvmStats."""
    from oracle.oracle_py import Reference
    from paper_2411_15332_b200 import bench_modes as B
    from paper_2411_15332_b200 import qcsim as Q
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    for n in range(2, 9):
        x = np.random.default_rng(n).standard_normal(1 << n) + 0j
        for m in (Q.SignMethod.nonopt, Q.SignMethod.quarter, Q.SignMethod.block, Q.SignMethod.logarithm):
            if m == Q.SignMethod.block:
                continue  # ref_rh_mvm runs block with the optimal size: checked below
            _, sc, mc = Reference.rh_mvm(n, x, m.name)
            assert sc == B.table2_count(m, n, 1) and mc == 4 * (1 << (n - 1)) ** 2
        _, sc, _ = Reference.rh_mvm(n, x, "block")
        assert sc == B.table2_count(Q.SignMethod.block, n, B.optimal_block_size(n))


@pytest.mark.gpu
def test_suites_on_device():
    from paper_2411_15332_b200 import bench_modes as B
    from paper_2411_15332_b200 import qcsim as Q
    rows = B.run_suite("rh-signs", [4, 12, 20], [])
    assert len(rows) == 12 and all(r.status == "ok" for r in rows)
    assert [r.engine for r in rows[:4]] == ["rh:nonopt", "rh:quarter", "rh:block", "rh:logarithm"]
    assert rows[0].sign_count == 4 ** 4 and rows[3].sign_count == 8 * 3
    eng = [Q.Engine.dense, Q.Engine.dax, Q.Engine.das]
    mtp = B.run_suite("mtp", [4, 8, 14], eng)
    assert [r.status for r in mtp] == ["ok"] * 6 + ["capacity-error", "ok", "ok"]
    assert mtp[1].memory_bytes == 24 * 16 and mtp[0].memory_bytes == 16 * 256
    mvm = B.run_suite("mvm", [10], eng)
    assert [r.multiply_count for r in mvm] == [1 << 20, 1 << 10, 1 << 10]
    gr = B.run_suite("grover", [8, 12], [Q.Engine.rh_dax, Q.Engine.dax])
    assert all(r.status == "ok" for r in gr) and gr[0].note == f"argmax={(1 << 8) // 3}"
    qn = B.run_suite("qnn", [4], [Q.Engine.rh_dax])
    assert qn[0].status == "ok" and qn[0].n == 4 + 2 + 1
    csv = B.render_bench(rows + mtp)
    assert csv.splitlines()[0] == "suite,n,engine,seconds,memory_bytes,sign_count,multiply_count,status,note"
