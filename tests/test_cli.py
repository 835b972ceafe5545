"""CLI parity (fpmm_cli.cpp): plan output, CSV schema v1, crossover table."""
import io

import pytest

from paper_2601_07508_b200 import cli


def test_plan_and_usage(capsys):
    assert cli.main(["plan", "--bits", "37"]) == 0
    assert "variant=(1,3)" in capsys.readouterr().out
    assert cli.main(["plan", "--bits", "53"]) == 1
    assert cli.main(["frobnicate"]) == 2


def test_preset_dims():
    assert cli.preset_dims("square", 1.0) == (10016, 10016, 10016)
    assert cli.preset_dims("unbalanced", 1.0) == (10923, 32768, 32)
    assert cli.preset_dims("square", 0.1) == (992, 992, 992)  # llround(1001.6/32)*32


def test_crossover_from_csv(tmp_path):
    rows = []
    for bits in range(20, 30):
        for (u, v), g in (((1, 1), 100 - 5 * max(0, bits - 24)), ((1, 2), 60)):
            rows.append(dict(schema_version=1, scenario="square", m=8, k=8, n=8, bits=bits, p=0, u=u, v=v,
                             concat="none", kernel="b200", runs=1, t_avg_s=1.0, eff_gflops=float(g),
                             status="ok" if (u, v) == (1, 2) or bits <= 26 else "infeasible", **{"lambda": 1}))
    path = tmp_path / "b.csv"
    with open(path, "w") as f:
        cli.write_csv(rows, f)
    head = open(path).readline().strip()
    assert head == ",".join(cli.HEADER)
    table = cli.crossover_table(cli.read_csv(str(path)))
    assert table == [[(1, 1), 20, 26], [(1, 2), 27, 29]]
    with pytest.raises(cli.Error):
        cli.crossover_table([r for r in cli.read_csv(str(path)) if r["bits"] != 23])


@pytest.mark.gpu
def test_bench_csv_on_gpu(tmp_path):
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--dims", "256,256,256", "--bits", "20", "26", "27", "--variant", "1,1", "1,2",
                     "--runs", "2", "--out", str(out), "--extended"]) == 0
    lines = open(out).read().strip().split("\n")
    assert lines[0].startswith(",".join(cli.HEADER))
    body = [l.split(",") for l in lines[1:]]
    assert len(body) == 6
    status = {(int(r[5]), int(r[7]), int(r[8])): r[15] for r in body}
    assert status[(27, 1, 1)] == "infeasible" and status[(26, 1, 1)] == "ok"
    assert cli.main(["bench", "--scenario", "unbalanced", "--scale", "0.05", "--bits", "40", "--runs", "1",
                     "--out", str(tmp_path / "u.csv")]) == 0


def test_check_verifier_catches_wrong_products():
    """cli.verify_product (the check suite's verifier: exact Freivalds trials
    plus sampled exact entries) accepts the oracle's C and rejects C with one
    corrupted entry or an entry outside [0, p)."""
    import numpy as np

    import oracle as O
    from paper_2601_07508_b200 import cli
    p, A, B = O.seeded_inputs(40, 70, 30, 48)
    C = O.exact_mod_gemm(A, B, p)
    assert cli.verify_product(A, B, C, p, 2, 4, 7) is None
    bad = C.copy()
    bad[13, 17] = (bad[13, 17] + 1) % p
    assert cli.verify_product(A, B, bad, p, 2, 4, 7) is not None
    bad = C.copy()
    bad[0, 0] = float(p)
    assert "outside" in cli.verify_product(A, B, bad, p, 2, 4, 7)
    assert cli.verify_product(np.zeros((0, 5)), np.zeros((5, 3)), np.zeros((0, 3)), p, 2, 4, 7) is None


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,extra", [("b200", []), ("b200-dmma-exact", ["--checked"]), ("b200-rns", ["--op", "workspace"])])
def test_check_suite_on_gpu(capsys, kernel, extra):
    """`check` (driver.cpp:37-140): the standard suite's shapes at a subset of
    bitsizes passes on every engine; one line per case, then the summary."""
    from paper_2601_07508_b200 import cli
    rc = cli.main(["check", "--bits", "5", "26", "39", "52", "--seeds", "1", "--kernel", kernel] + extra)
    out = capsys.readouterr().out
    assert rc == 0, out
    assert "FAIL" not in out and "check: " in out and " 0 failed" in out
    assert out.count("PASS") >= 12


def test_check_argument_errors(capsys):
    """check's argument handling needs no GPU: dims over the oracle cap fail
    with exit code 1 (driver.cpp:44-46), a malformed --dims with 1, usage errors
    with 2 (fpmm_cli.cpp:14-16)."""
    assert cli.main(["check", "--dims", "513,4,4"]) == 1
    assert "oracle cap" in capsys.readouterr().err
    assert cli.main(["check", "--dims", "4,4"]) == 1
    assert cli.main(["check", "--op", "nonsense"]) == 2
