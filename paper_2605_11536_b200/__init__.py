"""B200-native ToF ReSTIR renderer (time-gated and transient, path-length
preserving reservoir reuse).  The compute path is libtofr_b200.so (sm_100a
kernels behind the C ABI in include/tofr_gpu.h); this package is the Python
mirror of the reference render API over that ABI."""
from . import _ffi
from .api import (GateSpec, RenderConfig, RenderOutput, Renderer, Scene, Session, TofrError,
                  TransientHistogram, reference_render, render_doppler, render_gated, render_transient,
                  render_transient_plain)
from .scenes import (Camera, CameraPose, DeltaLight, Material, ObjectDef, PoseKey, SceneDef, boxes_doppler,
                     bundled, cornell, cornell_box, cornell_wide, flat_wall)

__all__ = [
    "GateSpec", "RenderConfig", "RenderOutput", "Renderer", "Scene", "Session", "TofrError",
    "TransientHistogram", "reference_render", "render_doppler", "render_gated", "render_transient",
    "render_transient_plain", "Camera", "CameraPose", "DeltaLight", "Material", "ObjectDef", "PoseKey",
    "SceneDef", "boxes_doppler", "bundled", "cornell", "cornell_box", "cornell_wide", "flat_wall", "_ffi",
]
