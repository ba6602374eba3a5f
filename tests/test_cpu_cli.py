"""The bench front end's host logic (paper_2412_10287_b200/cli.py), mirroring
the reference's CLI tests (test_cli.py:161-167 parse errors, :101-117 CSV
schema).  No device work."""

import csv
import io

import pytest

from paper_2412_10287_b200 import cli


def test_workload_parse_errors():
    with pytest.raises(cli.WorkloadFormatError):
        cli.parse_workload(io.StringIO("only\tthree\tfields\n"))
    with pytest.raises(cli.WorkloadFormatError):
        cli.parse_workload(io.StringIO("q\tboth\t3\ta\n"))
    with pytest.raises(cli.WorkloadFormatError) as ei:
        cli.parse_workload(io.StringIO("q\tssr\t3\ta\nq\tssr\t3\tb\n"))
    assert ei.value.line_no == 2


def test_workload_parse_comments_and_blank_lines():
    es = cli.parse_workload(io.StringIO("# header\n\nq1\tssr\t3\ta* b\r\nq2\tsdr\t5\tb\n"))
    assert [(e.id, e.mode, e.endpoint, e.pattern) for e in es] == [("q1", "ssr", "3", "a* b"),
                                                                    ("q2", "sdr", "5", "b")]


def test_csv_schema_plain_and_extended():
    rows = [{"id": "q1", "mode": "ssr", "algorithm": "hybrid", "result_count": 1, "iterations": 3,
             "time_ms": 0.12345, "status": "ok", "gteps": 1.5, "levels": 3, "te": 10, "bytes_alg": 100,
             "roofline_frac": 0.0001, "ngpu": 1, "cpu_ms": "", "cpu_cores": ""}]
    out = io.StringIO()
    cli.write_csv(rows, out)
    got = list(csv.reader(io.StringIO(out.getvalue())))
    assert got[0] == cli.BENCH_HEADER == ["id", "mode", "algorithm", "result_count", "iterations", "time_ms",
                                          "status"]
    assert got[1] == ["q1", "ssr", "hybrid", "1", "3", "0.123", "ok"]
    out = io.StringIO()
    cli.write_csv(rows, out, extended=True)
    got = list(csv.reader(io.StringIO(out.getvalue())))
    assert got[0] == cli.EXT_HEADER and got[0][:7] == cli.BENCH_HEADER
    assert got[1][7:] == ["1.500", "3", "10", "100", "0.0001", "1", "", ""]


def test_automaton_lookup_from_config_json(tmp_path):
    import json
    import os

    here = os.path.dirname(os.path.abspath(cli.__file__))
    d = json.load(open(os.path.join(here, "data", "config_automata.json")))
    p = tmp_path / "a.json"
    p.write_text(json.dumps(d["cfg3"]))
    comp = cli.automaton_compiler(str(p))
    n = comp("^a (b|c)* d")
    assert n.nstates == 3
    with pytest.raises(KeyError):
        comp("a )b")
