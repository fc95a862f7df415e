"""The bench CSV contract (reference cli.py:47-55, 213-325): header, kernel
list and append semantics on CPU; on the GPU every count column of a row
equals the reference's own cmd_bench row for the same (kernel, n, bits,
variant) - only the timing columns differ (GPU vs CPU)."""

from __future__ import annotations

import csv

import pytest

import oracle
from paper_2209_01290_b200 import benchcsv


def _ref_cli():
    ref = oracle.reference()
    if ref is None:
        pytest.skip("reference (oracle/_ref) not built")
    import nttmul.cli as cli

    return cli


def test_header_and_kernels_match_reference():
    cli = _ref_cli()
    assert benchcsv.CSV_HEADER == cli.CSV_HEADER
    assert benchcsv.BENCH_KERNELS == cli.BENCH_KERNELS


def test_write_row_appends_with_one_header(tmp_path, capsys):
    path = tmp_path / "b.csv"
    row = ("ntt", 4096, 60, "proposed", 2, 1.0, 1.5, 1.5, 24576, 49152, 0, 4095)
    benchcsv.write_row(row, str(path))
    benchcsv.write_row(row, str(path))
    rows = list(csv.reader(open(path)))
    assert rows[0] == list(benchcsv.CSV_HEADER) and len(rows) == 3
    benchcsv.write_row(row)
    out = capsys.readouterr().out.splitlines()
    assert out[0] == ",".join(benchcsv.CSV_HEADER) and out[1].startswith("ntt,4096,60")


def _ref_row(cli, kernel, n, bits, variant, reps):
    if kernel.startswith(("reduce", "barrett")):
        q, v, r, times, ctr = cli._bench_reduction(kernel, bits, reps, 1, 0)
        n = 1
    else:
        q, v, r, times, ctr = cli._bench_transform(kernel, n, bits, reps, 1, 1, 0, variant)
    return (kernel, n, bits, v, r, ctr.modmul, ctr.modadd_sub, ctr.half_scalings,
            ctr.twiddle_loads)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,n,bits,variant", [
    ("ntt", 4096, 60, "proposed"), ("intt", 4096, 60, "proposed"),
    ("ntt-radix4", 1024, 50, "classical"), ("ntt-2d", 1024, 40, "proposed"),
    ("polymul", 2048, 60, "dhem"), ("polymul-fused", 65536, 60, "proposed"),
    ("batch-ntt", 4096, 60, "proposed"), ("barrett-proposed", 1, 60, "proposed"),
    ("reduce-builtin", 1, 62, "builtin"), ("barrett-dhem", 1, 59, "dhem"),
])
def test_rows_match_reference_counts(kernel, n, bits, variant):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cli = _ref_cli()
    reps = 8192 if kernel.startswith(("reduce", "barrett")) else 2
    ours = benchcsv.bench_row(kernel, n, bits, reps, 1, 1, 0, variant)
    assert len(ours) == len(benchcsv.CSV_HEADER)
    assert ours[5] <= ours[6] and ours[5] <= ours[7] and ours[5] > 0
    want = _ref_row(cli, kernel, n, bits, variant, reps)
    assert ours[:5] + ours[8:] == want
