"""The C-ABI library loads without a GPU and exports every symbol that
include/*.h declares; error paths map reference exceptions to pf_status
codes.  No kernel is launched here."""
import ctypes as C
import os
import re

import pytest

from paper_2211_14133_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in ("pf_sched.h", "pf_kfac.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(pf_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_library_loads_and_exports_all_declared_symbols():
    lib = L.lib()
    declared = declared_functions()
    assert len(declared) >= 35
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared) <= set(L.exported_symbols()) | set(declared)
    assert b"sm_100a" in lib.pf_version()


def test_kfac_entry_points_reject_bad_shapes_before_launching():
    lib = L.lib()
    before = lib.pf_kernel_launch_count()
    # d = 0 -> bad shape; nothing may be launched
    rc = lib.pf_curvature_syrk(None, 0, 16, 16, 1.0, 0, None, 0, 1, None)
    assert rc == L.PF_BAD_SHAPE
    assert b"shape mismatch" in lib.pf_last_error()
    size = C.c_size_t()
    assert lib.pf_damped_inverse_workspace(0, size) == L.PF_BAD_ARG
    assert lib.pf_damped_inverse_workspace(1024, size) == L.PF_OK
    assert size.value >= 5 * 1024 * 1024 * 4  # five fp32 planes + digit slots
    assert lib.pf_precondition_workspace(4096, 1024, size) == L.PF_OK
    assert lib.pf_kernel_launch_count() == before


def test_scheduler_status_codes():
    from paper_2211_14133_b200 import schedule as S
    with pytest.raises(ValueError, match="horizon_steps"):
        S.build_schedule(S.PipelineConfig(), S.CostTable(t_f=1, t_b=1), 0)
    cfg = S.PipelineConfig(stages=2, micro_batches=2)
    base = S.build_schedule(cfg, S.CostTable(t_f=1, t_b=1))
    q = S.KfacWorkQueue([S.KfacWork(kind=S.WorkKind.Curvature, stage=0, micro_batch=7,
                                    device=0, duration=0.1, base_anchor=S.WorkKind.Forward)])
    with pytest.raises(ValueError, match="no matching forward/backward"):
        S.assign_works(base, cfg, S.CostTable(t_f=1, t_b=1), q)
    with pytest.raises(ValueError, match="device count"):
        S.assign_works(base, S.PipelineConfig(stages=4, micro_batches=2), S.CostTable(t_f=1, t_b=1),
                       S.KfacWorkQueue())


def test_empty_batches_are_noops_through_the_c_interface():
    """count == 0 returns PF_OK without touching the device (the
    batched inverse used to index an empty group list); count < 0 is BAD_ARG."""
    lib = L.lib()
    before = lib.pf_kernel_launch_count()
    assert lib.pf_damped_inverse_batched(None, 0, None) == L.PF_OK
    assert lib.pf_curvature_syrk_grouped(None, 0, 1, None) == L.PF_OK
    assert lib.pf_precondition_update_sliced(None, 0, None) == L.PF_OK
    assert lib.pf_damped_inverse_batched(None, -1, None) == L.PF_BAD_ARG
    assert lib.pf_curvature_syrk_grouped(None, -1, 1, None) == L.PF_BAD_ARG
    assert lib.pf_precondition_update_sliced(None, -1, None) == L.PF_BAD_ARG
    assert lib.pf_kernel_launch_count() == before
