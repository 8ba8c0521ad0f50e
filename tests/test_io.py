"""CPU tests of the data-file layer around the device filter:
time-series CSV and samples files written by the REFERENCE (tests/golden/io,
make_io_golden.py) are read and re-written byte for byte, and the LOCF input
provider returns the reference's values (timeseries.py:79-210,
sampleio.py:39-137)."""

import os

import numpy as np
import pytest

from paper_1306_3277_b200 import LORENZ96, WINDKESSEL
from paper_1306_3277_b200.errors import DataFormatError, MissingInputError
from paper_1306_3277_b200.sampleio import read_run_output, write_run_output
from paper_1306_3277_b200.timeseries import (InputProvider, TimeSeries, read_timeseries, role_arrays,
                                             variables, write_timeseries)
from tests.conftest import GOLDEN

IO = os.path.join(GOLDEN, "io")


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name,model,roles", [("wk_input.csv", WINDKESSEL, ("input",)),
                                              ("wk_obs.csv", WINDKESSEL, ("obs",)),
                                              ("l96_obs.csv", LORENZ96, ("obs",))])
def test_timeseries_round_trip_is_byte_identical(name, model, roles, tmp_path):
    ts = read_timeseries(os.path.join(IO, name), model, roles=roles)
    out = tmp_path / name
    write_timeseries(out, ts, model)
    assert _bytes(out) == _bytes(os.path.join(IO, name))


def test_role_arrays_masks_and_layout():
    t, v, m = role_arrays(read_timeseries(os.path.join(IO, "l96_obs.csv"), LORENZ96), LORENZ96, "obs")
    assert v.shape == (20, 8) and m.shape == (20, 8)
    assert not m[0].any() and m[1, :4].all() and not m[1, 4:].any()  # slots 0-3 every other step
    t, v, m = role_arrays(read_timeseries(os.path.join(IO, "wk_obs.csv"), WINDKESSEL), WINDKESSEL, "obs")
    assert m.sum() == 39 and not m[7, 0]


def test_input_provider_matches_reference():
    g = np.load(os.path.join(IO, "wk_input_at.npz"))
    prov = InputProvider(WINDKESSEL, read_timeseries(os.path.join(IO, "wk_input.csv"), WINDKESSEL, ("input",)))
    got = np.array([prov.at(t) for t in g["t"]])
    np.testing.assert_array_equal(got, g["v"])
    with pytest.raises(MissingInputError):
        prov.at(-0.5)


def test_input_provider_forward_fills_masked_cells():
    ts = TimeSeries(times=np.array([0.0, 1.0, 2.0])).add("F", np.array([np.nan, 3.0, np.nan]))
    prov = InputProvider(WINDKESSEL, ts)
    with pytest.raises(MissingInputError):
        prov.at(0.5)  # slot not yet present
    assert prov.at(1.0)[0] == 3.0 and prov.at(2.5)[0] == 3.0


@pytest.mark.parametrize("name", ["l96_mh_samples.txt", "wk_smc_samples.txt"])
def test_samples_file_round_trip_is_byte_identical(name, tmp_path):
    out = read_run_output(os.path.join(IO, name))
    assert out.records and out.param_labels
    p = tmp_path / name
    write_run_output(p, out)
    assert _bytes(p) == _bytes(os.path.join(IO, name))


def test_variable_layouts_agree_across_model_objects():
    from tests.test_cpu_generic import _desc as _lowered

    for spec, name in ((LORENZ96, "Lorenz96"), (WINDKESSEL, "Windkessel")):
        a = variables(spec)
        d = _lowered(name)
        if "vars" in d:
            assert a == variables(d)
        for role in ("param", "state", "obs", "input"):
            labels = [lab for v in sorted((v for v in a.values() if v.role == role), key=lambda v: v.offset)
                      for lab in v.labels()]
            assert labels == spec.slot_labels(role)


def test_data_format_errors(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("time,q\n0.0,1.0\n")
    with pytest.raises(DataFormatError):
        read_timeseries(p, WINDKESSEL)
    p.write_text("time,Pa\n1.0,1.0\n0.5,2.0\n")
    with pytest.raises(DataFormatError):
        read_timeseries(p, WINDKESSEL)
    p.write_text("time,Pa\n0.0,1.0\n")
    with pytest.raises(DataFormatError):
        read_timeseries(p, WINDKESSEL, roles=("input",))
    p.write_text("time,x\n0.0,1.0\n")
    with pytest.raises(DataFormatError):
        read_timeseries(p, LORENZ96)  # vector variable without an index
