"""On-disk formats around the train step, over the C ABI:

* LAMMCKPT checkpoints, byte-compatible with lamm::model::save_checkpoint /
  load_checkpoint (S/model.cpp:429-497);
* LAMMRMS1: the RMS optimizer state in the same layout (an extension: the
  reference keeps it in memory only);
* LAMMDS1 catalogs (S/dataset.cpp:273-393): catalog.json (plain JSON, read here)
  plus one .bin per subset, read by liblamm_b200 straight into packed batches.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from ._lib import ModelConfigC, check, lib
from .api import ModelConfig, _c, _p

TASKS = ("energy_and_forces", "energy_only", "denoising")


def save_checkpoint(path: str, cfg: ModelConfig, params: np.ndarray) -> None:
    p = _c(params, np.float64)
    check(lib().lamm_checkpoint_save(os.fsencode(path), C.byref(cfg.c()), _p(p), C.c_size_t(len(p))))


def load_checkpoint(path: str) -> tuple[ModelConfig, np.ndarray]:
    c, n = ModelConfigC(), C.c_size_t()
    check(lib().lamm_checkpoint_load(os.fsencode(path), C.byref(c), None, C.c_size_t(0), C.byref(n)))
    out = np.empty(n.value, np.float64)
    check(lib().lamm_checkpoint_load(os.fsencode(path), C.byref(c), _p(out), C.c_size_t(n.value), C.byref(n)))
    return ModelConfig(c.hidden, c.layers, c.rbf, c.cutoff, c.heads), out


def save_rms_state(path: str, cfg: ModelConfig, v: np.ndarray) -> None:
    p = _c(v, np.float64)
    check(lib().lamm_rms_state_save(os.fsencode(path), C.byref(cfg.c()), _p(p), C.c_size_t(len(p))))


def load_rms_state(path: str) -> tuple[ModelConfig, np.ndarray]:
    c, n = ModelConfigC(), C.c_size_t()
    check(lib().lamm_rms_state_load(os.fsencode(path), C.byref(c), None, C.c_size_t(0), C.byref(n)))
    out = np.empty(n.value, np.float64)
    check(lib().lamm_rms_state_load(os.fsencode(path), C.byref(c), _p(out), C.c_size_t(n.value), C.byref(n)))
    return ModelConfig(c.hidden, c.layers, c.rbf, c.cutoff, c.heads), out


def read_subset(path: str, head_index: int = 0) -> dict:
    """One LAMMDS1 subset file as a packed batch dict (dataset_index = head_index)."""
    cnt, atoms = C.c_int64(), C.c_int64()
    check(lib().lamm_subset_info(os.fsencode(path), C.byref(cnt), C.byref(atoms)))
    B, N = cnt.value, atoms.value
    b = dict(atom_ptr=np.empty(B + 1, np.int64), pos=np.empty((N, 3)), Z=np.empty(N, np.int32),
             dataset_index=np.empty(B, np.int32), energy_mask=np.empty(B, np.uint8), force_mask=np.empty(B, np.uint8),
             energy=np.empty(B), forces=np.empty((N, 3)), denoise=np.zeros(B, np.uint8))
    check(lib().lamm_subset_read(os.fsencode(path), head_index, C.c_int64(B), C.c_int64(N), _p(b["atom_ptr"]), _p(b["pos"]), _p(b["Z"]),
                                 _p(b["dataset_index"]), _p(b["energy_mask"]), _p(b["force_mask"]), _p(b["energy"]),
                                 _p(b["forces"])))
    return b


def read_catalog(directory: str) -> dict:
    """lamm::dataset::read_catalog: {"seed", "subsets": [{"name", "task", "head_index",
    "has_energy", "has_forces", "batch"}]}; denoising subsets get denoise = 1."""
    with open(os.path.join(directory, "catalog.json")) as f:
        meta = json.load(f)
    if meta.get("format") != "lamm-catalog":
        raise ValueError("not a catalog directory")
    subsets = []
    for e in meta["subsets"]:
        if e["task"] not in TASKS:
            raise ValueError(f"unknown task {e['task']}")
        b = read_subset(os.path.join(directory, e["file"]), int(e["head_index"]))
        if len(b["atom_ptr"]) - 1 != int(e["size"]):
            raise ValueError(f"catalog.json size disagrees with {e['name']}.bin")
        if e["task"] == "denoising":
            b["denoise"][:] = 1
        subsets.append(dict(name=e["name"], task=e["task"], head_index=int(e["head_index"]),
                            has_energy=bool(e["has_energy"]), has_forces=bool(e["has_forces"]), batch=b))
    return dict(seed=int(meta["seed"]), subsets=subsets)
