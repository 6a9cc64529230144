"""Shared test helpers (fixtures, config objects)."""
import glob
import os

import numpy as np

from paper_2602_08501_b200 import configs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def two_stage_fixtures():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "two_stage_*.npz")))


def scl_fixtures():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "scl_*.npz")))


def osd_list_fixtures():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "osd_*.npz")))


def osd_two_stage_fixtures():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "osdts_*.npz")))


def osd_code(fixture: str):
    """The code an OSD fixture was generated on (tests/golden/make_golden.py:gen_osd)."""
    from paper_2602_08501_b200 import codes
    if "_rm_" in fixture:
        return configs.CONFIGS["cfg2"].code()
    if "_ca64_" in fixture:
        return codes.build_ca_polar_code(64, 16)
    if "_cfg1_" in fixture:
        return configs.CONFIGS["cfg1"].code()
    raise KeyError(fixture)


def osd_sphere(g, code):
    from paper_2602_08501_b200.sphere import sphere_from_members
    mem = np.asarray(g["sphere_members"], dtype=np.uint64)
    return sphere_from_members(code.n, code.k, int(g["radius_index"]), mem[1:])


def cfg_of(fixture: str):
    return configs.CONFIGS[fixture.split("_")[2] if fixture.startswith("two_stage") else
                           fixture.split("_")[1].split(".")[0]]


_spheres = {}
_codes = {}


def code_and_sphere(cfg):
    if cfg.name not in _codes:
        _codes[cfg.name] = cfg.code()
        _spheres[cfg.name] = configs.build_sphere_for(cfg, _codes[cfg.name])
    return _codes[cfg.name], _spheres[cfg.name]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))
