"""The C-ABI library loads and exports every symbol include/ftb.h declares;
error codes map onto the mktune exception classes."""

import ctypes

import pytest

from paper_2407_21418_b200 import _lib


def test_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing


def test_error_mapping_input_error():
    from paper_2407_21418_b200.mktune import errors
    from paper_2407_21418_b200.mktune._native import hw_struct, lib
    from paper_2407_21418_b200.mktune.hardware import b200_bf16

    h = hw_struct(b200_bf16())
    h.num_cores = 0
    L = lib()
    out = ctypes.c_void_p()
    tr = ctypes.c_int32()
    from paper_2407_21418_b200.runtime import dense_instance
    from paper_2407_21418_b200.mktune._native import inst_struct

    st = L.ftb_enumerate(ctypes.byref(h), ctypes.byref(inst_struct(dense_instance(5, 64, 64))), -1,
                         ctypes.byref(out), ctypes.byref(tr))
    assert st == _lib.FTB_INPUT_ERROR
    with pytest.raises(errors.InputError) as e:
        _lib.check(st)
    assert e.value.field == "num_cores"


def test_empty_pool_raises_empty_result():
    from paper_2407_21418_b200.mktune import combine, errors, ukernel, workload
    from cases import dense_doc

    inst = workload.WorkloadInstance(workload.parse_workload(dense_doc(64, 64, 4, 100)), {"i": 7})
    k = ukernel.UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 2, "j": 64, "k": 64},
                        padding_threshold=1.0, usage_eff=1.0, compute_eff=1.0)
    # tau = i (7 > ... no: j=64 > 7 -> tau = j; a 128-wide j tile cannot cover 64 exactly)
    k.smem_tile["j"] = 128
    with pytest.raises(errors.EmptyResultError) as e:
        combine.build_programs([k], inst)
    assert e.value.constraint == "main-axis coverage"
    with pytest.raises(errors.EmptyResultError):
        combine.build_programs([], inst)


def test_missing_metrics():
    from paper_2407_21418_b200.mktune import errors, scoring, ukernel, workload
    from cases import dense_doc

    inst = workload.WorkloadInstance(workload.parse_workload(dense_doc(64, 64, 4, 100)), {"i": 7})
    k = ukernel.UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 7, "j": 64, "k": 64})
    with pytest.raises(errors.MissingMetricsError):
        scoring.rank_topk([k], inst)


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with libftb.so absent, planning (and therefore every
    execute path) raises LibraryMissing instead of routing anywhere else."""
    import os
    import subprocess
    import sys

    code = (
        "from paper_2407_21418_b200 import _lib\n"
        "from paper_2407_21418_b200.runtime import Planner, dense_instance\n"
        "try:\n"
        "    Planner().plan([dense_instance(128, 768, 768)])\n"
        "except _lib.LibraryMissing as e:\n"
        "    print('RAISED', e)\n"
        "else:\n"
        "    print('NO-RAISE')\n"
    )
    env = dict(os.environ, FTB_LIB=str(tmp_path / "absent_libftb.so"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert "RAISED" in out.stdout, out.stdout + out.stderr


def test_status_codes_map_onto_error_classes():
    """Each FTB_* status of include/ftb.h becomes its mktune.errors class
    (errors.py:10-47), with the CLI exit code the reference assigns."""
    from paper_2407_21418_b200.mktune import errors as E

    cases = {
        _lib.FTB_INPUT_ERROR: (E.InputError, 2),
        _lib.FTB_EMPTY_RESULT: (E.EmptyResultError, 1),
        _lib.FTB_INTERNAL_ERROR: (E.InternalError, 3),
        _lib.FTB_CAPACITY_ERROR: (E.CapacityError, 2),
        _lib.FTB_MISSING_METRICS: (E.MissingMetricsError, 3),
        _lib.FTB_CUDA_ERROR: (E.DeviceError, 3),
    }
    for status, (cls, exit_code) in cases.items():
        e = E.TunerError.from_status(status, "msg", "fld")
        assert type(e) is cls and e.exit_code == exit_code and str(e) == "msg"
    assert E.TunerError.from_status(_lib.FTB_INPUT_ERROR, "m", "fld").field == "fld"
    assert E.TunerError.from_status(_lib.FTB_EMPTY_RESULT, "m", "c").constraint == "c"
    assert E.InputError("m", "f").field == "f" and E.EmptyResultError("m", "c", "h").hint == "h"
    with pytest.raises(TypeError):
        E.InputError("m", "f", "extra")
