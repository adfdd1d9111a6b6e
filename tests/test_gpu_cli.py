"""`online` command on the GPU plan (paper_2510_04825_b200.cli) against the
reference's own `subapsnap online` on the same offline artifacts.

The reference's `offline` command writes the artifacts for two of its packaged
experiments (fig1-tridiag: lupp selector, p-dependent rhs; heat2d: leverage
selector); both `online` commands then read them and write results.csv.  The
method and parameter columns must be identical, the relative residuals agree
to 3 significant digits (above 1e-12; both below it otherwise), and the
output_error column is empty as in the reference.  Skipped without the
baseline/_ref install."""
import csv
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
pytestmark = pytest.mark.gpu


def _rows(path):
    with open(path) as fh:
        return list(csv.reader(fh))


@pytest.mark.parametrize("config", ["fig1-tridiag", "heat2d"])
def test_cli_online_matches_reference(config):
    if not (REF / "subapsnap" / "__init__.py").exists():
        pytest.skip("baseline/_ref (reference install) absent")
    env = dict(os.environ, PYTHONPATH=f"{REF}:{ROOT}")
    with tempfile.TemporaryDirectory() as tmp:
        art, out_ref, out_gpu = Path(tmp) / "art", Path(tmp) / "ref", Path(tmp) / "gpu"
        for cmd in (["-m", "subapsnap.cli", "offline", config, "--artifacts", str(art)],
                    ["-m", "subapsnap.cli", "online", config, "--artifacts", str(art), "--out", str(out_ref)],
                    ["-m", "paper_2510_04825_b200.cli", "online", config, "--artifacts", str(art), "--out",
                     str(out_gpu)]):
            r = subprocess.run([sys.executable, *cmd], cwd=ROOT, env=env, capture_output=True, text=True,
                               timeout=900)
            assert r.returncode == 0, (cmd, r.stdout[-2000:], r.stderr[-3000:])
        want, got = _rows(out_ref / "results.csv"), _rows(out_gpu / "results.csv")
    assert got[0] == want[0] and len(got) == len(want) > 1
    for g, w in zip(got[1:], want[1:]):
        assert g[:2] == w[:2] and g[3] == w[3] == ""
        a, b = float(g[2]), float(w[2])
        if max(a, b) > 1e-12:
            assert a == pytest.approx(b, rel=5e-4), (g, w)
        else:
            assert a <= 1e-12 and b <= 1e-12
