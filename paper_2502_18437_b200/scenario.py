"""The scenario harness on the B200 engine: run_scenario of
scenario.hpp:188-279 -- metrics.csv, frame dumps and the per-frame cut metric -- with the
physics and both metrics (compute_components, mean_nearest_neighbor_spacing) on the device.

Output formats are byte-compatible with the reference writers:
  frame_%06d.bin  u64 particle count + float32 x, y, z per particle, little endian, ALL
                  particles (active or not), scenario.hpp:151-160
  frame_%06d.csv  "x,y,z" header, "%.9g" per coordinate, scenario.hpp:162-172
  metrics.csv     frame,sim_time,wall_ms,total_mass,momentum_x/y/z,kinetic_energy,pushed_out,
                  inverted_f,shape<i>_impulse_x/y/z...,component_count (scenario.hpp:211-219,
                  258-268); wall_ms is this run's own wall clock
"""
from __future__ import annotations

import math
import struct
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import api, capi, scenes

F32 = np.float32


def write_frame_bin(path, pos: np.ndarray) -> None:
    """scenario.hpp:151-160."""
    pos = np.ascontiguousarray(pos, dtype="<f4").reshape(-1, 3)
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", pos.shape[0]))
        f.write(pos.tobytes())


def write_frame_csv(path, pos: np.ndarray) -> None:
    """scenario.hpp:162-172 ("%.9g" of each float widened to double)."""
    pos = np.asarray(pos, dtype=F32).reshape(-1, 3)
    with open(path, "w", newline="\n") as f:
        f.write("x,y,z\n")
        f.writelines("%.9g,%.9g,%.9g\n" % (float(a), float(b), float(c)) for a, b, c in pos)


def frame_has_nan(r: dict) -> bool:
    """scenario.hpp:174-183."""
    vals = [r["total_mass"], r["kinetic_energy"], *r["momentum"]]
    return (not all(math.isfinite(v) for v in vals)) or not np.isfinite(r["positions"]).all()


def components(scene: api.Scene, radius: float) -> int:
    """compute_components (scenario.hpp:100-139) of the scene's resident particles."""
    c = np.zeros(1, np.int32)
    api.check(scene.lib.mpmb_components(scene.h, api._fp(np.array([radius], F32)), c.ctypes.data_as(capi.ip)),
              scene.lib, "components")
    return int(c[0])


def nn_spacing(scene: api.Scene, cell_hint: float) -> float:
    """mean_nearest_neighbor_spacing (scenario.hpp:68-96) of the resident particles."""
    out = np.zeros(1, F32)
    api.check(scene.lib.mpmb_nn_spacing(scene.h, api._fp(np.array([cell_hint], F32)), api._fp(out)), scene.lib,
              "nn_spacing")
    return float(out[0])


@dataclass
class ScenarioSummary:
    frames_done: int = 0
    nan_detected: bool = False
    final_component_count: int = 0
    mean_abs_shape_impulse: list = field(default_factory=list)


def run_scenario(spec: dict, frames: int, out_dir, write_outputs: bool = True, stride: int = 0) -> ScenarioSummary:
    """scenario.hpp:188-279 on the device; `spec` is a scene dict (scenes.py, the JSON
    schema of scene_spec.hpp)."""
    out = Path(out_dir)
    outputs = spec.get("outputs", {})
    stride = stride or int(outputs.get("stride", 1))
    formats = outputs.get("formats", ["bin"])
    cfg = api.scene_config(**scenes.config_kwargs(spec))
    scene = api.Scene(cfg)
    scenes.populate(scene, spec)
    n_shapes = len(spec.get("shapes", []))
    metrics = None
    if write_outputs:
        out.mkdir(parents=True, exist_ok=True)
        metrics = open(out / "metrics.csv", "w", newline="\n")
        head = ("frame,sim_time,wall_ms,total_mass,momentum_x,momentum_y,momentum_z,kinetic_energy,pushed_out,"
                "inverted_f")
        for i in range(n_shapes):
            head += f",shape{i}_impulse_x,shape{i}_impulse_y,shape{i}_impulse_z"
        metrics.write(head + ",component_count\n")
    spacing = nn_spacing(scene, float(F32(spec["grid"]["dx"])))
    link = float(F32(F32(1.5) * F32(spacing)))  # Real(1.5) * nn_spacing
    summary = ScenarioSummary(mean_abs_shape_impulse=[np.zeros(3) for _ in range(n_shapes)])
    try:
        for frame in range(frames):
            t0 = time.perf_counter()
            scene.advance(spec["dt_frame"])
            r = scene.fetch_results()
            wall_ms = 1e3 * (time.perf_counter() - t0)
            if frame_has_nan(r):
                summary.nan_detected = True
                break
            comps = components(scene, link)
            summary.final_component_count = comps
            for i, imp in enumerate(r["shape_impulses"]):
                summary.mean_abs_shape_impulse[i] += np.abs(imp.astype(np.float64))
            if write_outputs:
                row = "%d,%.9g,%.6g,%.9g,%.9g,%.9g,%.9g,%.9g,%d,%d" % (
                    frame, float(F32(r["time"])), wall_ms, r["total_mass"], r["momentum"][0], r["momentum"][1],
                    r["momentum"][2], r["kinetic_energy"], r["pushed_out"], r["inverted_f"])
                for imp in r["shape_impulses"]:
                    row += ",%.9g,%.9g,%.9g" % (float(imp[0]), float(imp[1]), float(imp[2]))
                metrics.write(row + ",%d\n" % comps)
                if frame % stride == 0:
                    if "bin" in formats:
                        write_frame_bin(out / ("frame_%06d.bin" % frame), r["positions"])
                    if "csv" in formats:
                        write_frame_csv(out / ("frame_%06d.csv" % frame), r["positions"])
            summary.frames_done = frame + 1
    finally:
        if metrics:
            metrics.close()
        scene.destroy()
    if summary.frames_done:
        summary.mean_abs_shape_impulse = [v / summary.frames_done for v in summary.mean_abs_shape_impulse]
    return summary
