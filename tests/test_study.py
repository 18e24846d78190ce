"""Study harness: the reference's run_study / run_bundle_study / write_csv
contract (include/bddc/study.hpp, src/study.cpp:40-217) on the GPU path."""
import io

import numpy as np
import pytest

from conftest import golden
from paper_2410_14786_b200 import Problem
from paper_2410_14786_b200.study import (KCSV_HEADER, ExperimentConfig, StudyRow, parse_study_mode,
                                         run_bundle_study, run_study, write_csv)


def test_header_and_row_format():
    rows = [StudyRow("compare", 3, 9, 121, 16, 0.25, 0.0125, 5, 1.2345678901234567e-9, 12.5, "", True),
            StudyRow("compare", 3, 9, 121, 0, 0.0, 0.5, 20, 3e-9, None, "not converged, x\ny", False)]
    out = io.StringIO()
    write_csv(rows, out)
    lines = out.getvalue().splitlines()
    assert lines[0] == KCSV_HEADER == ("mode,k,n_subdomains,global_dofs,coarse_dim,setup_seconds,"
                                       "solve_seconds,iterations,final_relative_residual,"
                                       "condition_estimate,error")
    assert lines[1] == "compare,3,9,121,16,0.250000,0.012500,5,1.2345678901234566e-09,12.5,"
    assert lines[2] == "compare,3,9,121,0,0.000000,0.500000,20,3e-09,,not converged; x;y"


def test_config_validation_and_modes():
    with pytest.raises(ValueError, match="k list is empty"):
        ExperimentConfig(k_list=[]).validate()
    with pytest.raises(ValueError, match="every k must be at least 2"):
        ExperimentConfig(k_list=[2, 1]).validate()
    with pytest.raises(ValueError, match="tolerance must be positive"):
        ExperimentConfig(k_list=[2], tolerance=0.0).validate()
    with pytest.raises(ValueError, match="cells must be at least 2"):
        ExperimentConfig(k_list=[2], cells=1).validate()
    assert [parse_study_mode(m) for m in ("weak", "strong", "compare", "single")]
    with pytest.raises(ValueError, match="unknown study mode: bogus"):
        parse_study_mode("bogus")


def test_strong_mode_indivisible_is_an_error_row():
    rows = run_study(ExperimentConfig(mode="strong", k_list=[3], cells=8))
    assert len(rows) == 1 and not rows[0].converged
    assert rows[0].error == "strong mode: global cells 8 not divisible by k = 3"


def test_bundle_study_missing_file_is_an_error_row(tmp_path):
    rows = run_bundle_study(str(tmp_path / "missing" / "manifest.txt"), ExperimentConfig(k_list=[2]))
    assert len(rows) == 1 and rows[0].mode == "single" and "missing file" in rows[0].error


@pytest.mark.gpu
def test_compare_study_matches_reference_counts(gpu):
    # iteration counts of the reference (golden k2m4, k3m4: BDDC and plain CG)
    rows = run_study(ExperimentConfig(mode="compare", k_list=[2, 3], cells=4))
    assert [r.mode for r in rows] == ["compare"] * 4
    for i, name in enumerate(["k2m4", "k3m4"]):
        g = golden(name)
        bddc, plain = rows[2 * i], rows[2 * i + 1]
        assert bddc.converged and plain.converged and bddc.error == plain.error == ""
        assert bddc.iterations == int(g["pcg_report"][0])
        assert plain.iterations == int(g["plain_report"][0])
        assert bddc.coarse_dim == Problem.poisson(4 * (i + 2), i + 2).n_coarse and plain.coarse_dim == 0
        assert abs(bddc.final_relative_residual - g["pcg_history"][-1]) <= 1e-10
        assert bddc.condition_estimate is not None and bddc.condition_estimate > 1.0


@pytest.mark.gpu
def test_weak_and_bundle_study(gpu, tmp_path):
    rows = run_study(ExperimentConfig(mode="weak", k_list=[2, 4], cells=8))
    assert [(r.k, r.global_dofs) for r in rows] == [(2, 15 * 15), (4, 31 * 31)]
    assert all(r.converged and r.setup_seconds > 0 and r.solve_seconds > 0 for r in rows)
    g = golden("h4m8")
    cx, cy, kx, ky, dm, ks, seed = (int(v) for v in g["config"])
    p = Problem.poisson(cx, kx, cy, ky, kappa_decades=dm / 1000.0, kappa_seed=ks, rhs_seed=seed)
    rows = run_bundle_study(p.export_bundle(str(tmp_path)), ExperimentConfig(k_list=[2]))
    assert len(rows) == 1 and rows[0].converged, rows[0].error
    assert abs(rows[0].iterations - int(g["pcg_report"][0])) <= 1
    assert rows[0].n_subdomains == kx * ky == 16 and rows[0].k == 4  # square count: k = sqrt
