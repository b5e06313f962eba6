"""C-ABI boundary checks that need no GPU: the library loads, exports every function that
include/dem.h declares, and its host-only planner helpers agree with the oracle's pinned ones."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def demlib():
    from paper_2501_05300_b200 import build, dem
    build.build()
    return dem


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dem_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(demlib):
    L = demlib.lib()
    decl = declared_functions()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(demlib.EXPORTS) == decl


def test_struct_sizes_match_header(demlib, tmp_path):
    """The binding's ctypes layouts equal the C compiler's layout of include/dem.h."""
    import ctypes as C
    import subprocess
    structs = {"dem_bed_desc": demlib.BedDesc, "dem_dist_desc": demlib.DistDesc, "dem_step_report": demlib.StepReport,
               "dem_state_view": demlib.StateView, "dem_contact_view": demlib.ContactView,
               "dem_plate_desc": demlib.PlateDesc, "dem_plate_state": demlib.PlateState, "dem_timing": demlib.Timing,
               "dem_wall_state": demlib.WallState,
               "dem_solver": demlib.Solver, "dem_material": demlib.Material, "dem_box": demlib.Box,
               "dem_particles": demlib.Particles, "dem_generator": demlib.Generator}
    src = tmp_path / "sz.c"
    body = "".join(f'printf("%s %zu\\n", "{k}", sizeof({k}));' for k in structs)
    src.write_text('#include <stdio.h>\n#include "dem.h"\nint main(void){' + body + 'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().splitlines())
    for k, cls in structs.items():
        assert int(out[k]) == C.sizeof(cls), k


def test_create_without_gpu_fails_cleanly(demlib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import ctypes as C
    d = demlib.BedDesc()
    d.struct_size = 1   # wrong version -> DEM_ERR_INVALID before touching CUDA
    h = C.c_void_p()
    assert demlib.lib().dem_create_bed(C.byref(d), None, C.byref(h)) == demlib.DEM_ERR_INVALID
    assert b"struct_size" in demlib.lib().dem_last_error(None)


def test_planner_helpers_match_oracle(demlib, oracle_mod):
    for args in [(8.5e-3, 30e-3, 0.05, 0.0), (8.5e-3, 30e-3, 0.05, 0.1), (8.5e-3, 30e-3, 0.05, 0.5), (2e-3, 2e-3, 0.0, 0.3)]:
        assert demlib.profile_diameter(*args) == pytest.approx(oracle_mod.profile_diameter(*args), rel=1e-14)
    for args in [(8.5e-3, 8.5e-3, 1.0, 1.0, 0.6), (8.5e-3, 30e-3, 1.1, 1.0, 0.6), (4e-3, 32e-3, 1.2, 2.0, 0.5)]:
        assert demlib.contact_network_length(*args) == pytest.approx(oracle_mod.contact_network_length(*args), rel=1e-12)
    for nd in [70.6, 20.0, 45.0, 37.1, 18.3]:
        assert demlib.plan_iterations(nd, 0.02) == oracle_mod.solver_iterations(nd, 0.02)
    assert demlib.plan_timestep(8.5e-3, 0.02, 2200, 5e4) == pytest.approx(oracle_mod.planned_timestep(8.5e-3, 0.02, 2200, 5e4), rel=1e-14)


# ------------------------------------------------------------------ on-device generator: host side
BANDS4 = [(0.08, 2e-3), (0.25, 6e-3), (0.6, 16e-3)]          # config 4, top band first


def test_generator_count_matches_synth_recipe(demlib):
    """The generator's lattice (host plane table) has exactly the sites of synth's recipe for
    the same bands / profile (synth places spheres with numpy; the library on the device)."""
    import synth
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.3, 0.2, 0.6))
    for sp in (2.0, 2.25):
        n_lib = demlib.generator_count(dict(kind="bands", bands=BANDS4, spacing_factor=sp), box)
        b = synth.banded_bed((0.3, 0.2, 0.6), [(0.0, 0.08, 2e-3), (0.08, 0.25, 6e-3), (0.25, 0.6, 16e-3)], 1,
                             spacing=sp)
        assert n_lib == b.n, (sp, n_lib, b.n)
    boxg = dict(lo=(0.0, 0.0, 0.0), hi=(0.2, 0.1, 0.5))
    n_lib = demlib.generator_count(dict(kind="profile", d_min=4e-3, gamma=0.056, d_max=32e-3), boxg)
    g = synth.graded_bed((0.2, 0.1, 0.5), 2e-3, 16e-3, 0.5, 1)
    assert n_lib == g.n


def test_generator_slabs_partition_the_bed(demlib):
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.3, 0.2, 0.6))
    gen = dict(kind="bands", bands=BANDS4, spacing_factor=2.0)
    n = demlib.generator_count(gen, box)
    faces = [-np.inf, 0.07, 0.151, 0.2, np.inf]
    parts = [demlib.generator_count(gen, box, (faces[k], faces[k + 1])) for k in range(4)]
    assert sum(parts) == n and min(parts) > 0


def test_generator_layer_schedule_and_validation(demlib):
    box = dict(lo=(0.0, 0.0, 0.0), hi=(0.1, 0.1, 0.3))
    n = demlib.generator_count(dict(kind="layers", d_min=4e-3, d_max=16e-3, ratio_r=2.0, eta=3.0), box)
    assert n > 0
    with pytest.raises(demlib.DemError):
        demlib.generator_count(dict(kind="layers", d_min=4e-3, d_max=16e-3, ratio_r=1.0, eta=3.0), box)
    with pytest.raises(demlib.DemError):
        demlib.generator_count(dict(kind="bands", bands=[(0.2, 2e-3), (0.1, 4e-3)]), box)   # depths not increasing
