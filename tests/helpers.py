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
