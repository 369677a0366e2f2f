"""filterkit-bench compatibility (paper_2212_09005_b200.bench vs the
reference CLI, /root/reference/pkg/src/filterkit/bench.py): flags, exit
codes, CSV schema, and -- on the GPU -- every filter/op, with load factors
and FPRs equal to the oracle's on the same key stream."""

import numpy as np
import pytest

from paper_2212_09005_b200 import bench as cli

REF_FIELDS = ["filter", "api", "op", "log_slots", "load_factor", "threads", "dist", "seed", "wall_seconds",
              "ops_per_sec", "fpr", "bits_per_item"]


def test_csv_schema_matches_reference():
    assert cli.CSV_FIELDS == REF_FIELDS


def test_csv_roundtrip(tmp_path):
    p = tmp_path / "runs.csv"
    recs = [cli.MetricsRecord("tcf", "point", "fpr", 16, 0.9, 1, "uniform", 0, 0.5, 2e6, 4.4e-4, 17.8),
            cli.MetricsRecord("gqf", "bulk", "insert", 18, 0.31, 4, "zipf", 3, 0.25, 1e7)]
    cli.write_csv(str(p), recs[:1])
    cli.write_csv(str(p), recs[1:])  # append: no second header
    lines = p.read_text().splitlines()
    assert lines[0] == ",".join(REF_FIELDS) and len(lines) == 3
    assert lines[2].endswith(",,")  # None -> empty cells
    assert cli.read_csv(str(p)) == recs


@pytest.mark.parametrize("argv", [
    ["--filter", "gqf", "--op", "insert", "--load", "0"],
    ["--filter", "gqf", "--op", "insert", "--load", "1.5"],
    ["--filter", "tcf", "--op", "insert", "--threads", "0"],
    ["--filter", "tcf", "--op", "insert", "--mode", "mapreduce"],
    ["--filter", "gqf", "--op", "insert", "--no-backing"],
    ["--filter", "tcf", "--op", "insert", "--dist", "kmer"],
    ["--filter", "tcf", "--api", "bulk", "--op", "insert"],
    ["--filter", "tcf-bulk", "--api", "point", "--op", "insert"],
    ["--filter", "tcf", "--op", "insert", "--log-slots", "3"],
])
def test_parameter_errors_exit_1(argv, capsys):
    assert cli.main(argv + ["--repeats", "1"]) == 1
    assert "parameter error" in capsys.readouterr().err


def test_usage_errors_exit_1():
    with pytest.raises(SystemExit) as e:
        cli.main(["--filter", "bloom", "--op", "insert"])
    assert e.value.code == 1
    with pytest.raises(SystemExit) as e:
        cli.main(["--filter", "tcf"])
    assert e.value.code == 1


# -- on the device --------------------------------------------------------------------

def _oracle_tcf(oracle, log_slots, keys, seed=0):
    from paper_2212_09005_b200 import TcfParams
    p = TcfParams(num_blocks=(1 << log_slots) // 16, seed=seed)
    o = oracle.OracleTcf(p.num_blocks, 16, 16, np.uint16, p.backing_slots, p.cut_slots, p.probe_limit, seed)
    o.insert_many(keys)
    return o


@pytest.mark.gpu
def test_tcf_fpr_matches_oracle(oracle, tmp_path):
    from paper_2212_09005_b200.workloads import TAG_FPR, WorkloadSpec, counter_stream, gen_keys
    csvp = str(tmp_path / "r.csv")
    assert cli.main(["--filter", "tcf", "--op", "fpr", "--log-slots", "16", "--repeats", "2", "--csv", csvp]) == 0
    recs = cli.read_csv(csvp)
    assert len(recs) == 2 and recs[0].fpr == recs[1].fpr
    keys = gen_keys(WorkloadSpec("uniform", n=int(0.9 * (1 << 16)), seed=0))
    o = _oracle_tcf(oracle, 16, keys)
    exp_fpr = float(o.query_many(counter_stream(1, TAG_FPR, cli.FPR_QUERIES)).sum()) / cli.FPR_QUERIES
    exp_load = float((o.blocks > 1).sum()) / len(o.blocks)
    assert recs[0].fpr == exp_fpr
    assert recs[0].load_factor == round(exp_load, 6)
    assert recs[0].bits_per_item == round((len(o.blocks) + len(o.backing)) * 16 / len(keys), 4)


@pytest.mark.gpu
def test_tcf_fill_to_failure_matches_oracle(oracle, tmp_path):
    from paper_2212_09005_b200.workloads import WorkloadSpec, gen_keys
    csvp = str(tmp_path / "r.csv")
    assert cli.main(["--filter", "tcf", "--op", "fill-to-failure", "--log-slots", "12", "--no-backing",
                     "--repeats", "1", "--csv", csvp]) == 0
    rec = cli.read_csv(csvp)[0]
    from paper_2212_09005_b200 import TcfParams
    p = TcfParams(num_blocks=(1 << 12) // 16, backing_fraction=0.0)
    keys = gen_keys(WorkloadSpec("uniform", n=int(p.main_slots * 1.05) + cli.FILL_CHUNK, seed=0))
    o = oracle.OracleTcf(p.num_blocks, 16, 16, np.uint16, 0, p.cut_slots, p.probe_limit, 0)
    done = 0
    for lo in range(0, len(keys), cli.FILL_CHUNK):
        codes = o.insert_many(keys[lo:lo + cli.FILL_CHUNK])
        bad = np.flatnonzero(codes == 3)
        if len(bad):
            done += int(bad[0])
            break
        done += len(codes)
    assert rec.load_factor == round(done / p.main_slots, 6)


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ["--filter", "tcf", "--op", "insert", "--log-slots", "16"],
    ["--filter", "tcf", "--op", "query", "--log-slots", "16", "--threads", "4"],
    ["--filter", "tcf", "--op", "delete", "--log-slots", "16", "--group-width", "4"],
    ["--filter", "tcf-bulk", "--op", "insert", "--log-slots", "16"],
    ["--filter", "tcf-bulk", "--op", "fpr", "--log-slots", "16", "--batches", "4"],
    ["--filter", "tcf-bulk", "--op", "delete", "--log-slots", "16"],
    ["--filter", "gqf", "--op", "insert", "--log-slots", "16", "--dist", "zipf", "--mode", "mapreduce"],
    ["--filter", "gqf", "--api", "bulk", "--op", "count", "--log-slots", "16", "--dist", "ur-count"],
    ["--filter", "gqf", "--op", "delete", "--log-slots", "16"],
    ["--filter", "gqf", "--api", "bulk", "--op", "fill-to-failure", "--log-slots", "12"],
])
def test_every_filter_and_op_runs_and_validates(argv, tmp_path):
    csvp = str(tmp_path / "r.csv")
    assert cli.main(argv + ["--repeats", "1", "--csv", csvp]) == 0
    rec = cli.read_csv(csvp)[0]
    assert rec.ops_per_sec > 0 and 0 < rec.load_factor <= 1.0


@pytest.mark.gpu
def test_gqf_mapreduce_load_matches_oracle(oracle, tmp_path):
    from paper_2212_09005_b200 import GqfParams
    from paper_2212_09005_b200.workloads import WorkloadSpec, gen_keys
    csvp = str(tmp_path / "r.csv")
    assert cli.main(["--filter", "gqf", "--op", "insert", "--log-slots", "16", "--dist", "zipf",
                     "--mode", "mapreduce", "--repeats", "1", "--csv", csvp]) == 0
    rec = cli.read_csv(csvp)[0]
    keys = gen_keys(WorkloadSpec("zipf", n=int(0.9 * (1 << 16)), seed=0))
    uniq, counts = np.unique(keys, return_counts=True)
    p = GqfParams(q=16, r=8)
    o = oracle.OracleGqf(16, 8, 0, p.max_occupied)
    o.bulk_insert(uniq, counts.astype(np.uint64))
    assert rec.load_factor == round(int(o.stats[0]) / (1 << 16), 6)
