"""The benchmark CLI (reference cli.py / bench.py schema) on the device."""

import pytest

pytestmark = pytest.mark.gpu


def test_cli_bench_csv(tmp_path, capsys):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_04644_b200.cli import CSV_HEADER, main

    path = tmp_path / "out.csv"
    for op in ("helmholtz", "mass", "bwdtrans"):
        rc = main(["bench", "--op", op, "--shape", "hex,tet", "--order", "2..3", "--nelem", "64",
                   "--geometry", "deformed", "--reps", "3", "--csv", str(path)])
        assert rc == 0
        lines = path.read_text().splitlines()
        assert lines[0] == CSV_HEADER and len(lines) == 5
        for ln in lines[1:]:
            f = ln.split(",")
            assert f[0] == op and f[3] == "sumfac_top" and float(f[9]) > 0

