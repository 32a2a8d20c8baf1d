"""Scene definitions (the reference's SceneDef, scene.hpp:411-429) as plain
Python objects that lower to the C ABI's tofr_scene_desc.

Also holds the programmatic builders the reference tests use
(test_scenes.hpp:27-101: cornell_box, flat_wall) and the three bundled
scenes (proj/scenes/*.scn) expressed as builders, so the GPU box -- which has
no /root/reference -- renders exactly the scenes the reference ships.  A CPU
test checks each builder against the reference parser's SceneDef (identical
BVH and identical renders).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

from . import _ffi as F

KPI = 3.14159265358979323846


def deg2rad(d: float) -> float:
    return d * KPI / 180.0  # degrees_to_radians (math.hpp:186)


def normalize(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    return (v[0] / n, v[1] / n, v[2] / n)


@dataclass
class Material:
    kind: int = F.MAT_DIFFUSE
    albedo: tuple = (0.5, 0.5, 0.5)
    roughness: float = 0.5


@dataclass
class DeltaLight:
    position: tuple = (0.0, 0.0, 0.0)
    direction: tuple = (0.0, 0.0, -1.0)
    cone_half_angle: float = KPI / 2
    intensity: tuple = (1.0, 1.0, 1.0)
    regime: int = F.LIGHT_WIDE


@dataclass
class CameraPose:
    position: tuple = (0.0, 0.0, 0.0)
    forward: tuple = (0.0, 0.0, -1.0)
    up: tuple = (0.0, 1.0, 0.0)


@dataclass
class Camera:
    base: CameraPose = field(default_factory=CameraPose)
    fov_y: float = deg2rad(45)
    width: int = 128
    height: int = 128
    track: list = field(default_factory=list)  # [(frame, CameraPose)]


@dataclass
class PoseKey:
    frame: float = 0.0
    q: tuple = (1.0, 0.0, 0.0, 0.0)  # w, x, y, z
    t: tuple = (0.0, 0.0, 0.0)


@dataclass
class ObjectDef:
    name: str = ""
    tris: list = field(default_factory=list)  # [(v0, v1, v2, material)]
    track: list = field(default_factory=list)  # [PoseKey]

    def quad(self, a, b, c, d, mat):  # scene_io.hpp:278-281
        self.tris.append((a, b, c, mat))
        self.tris.append((a, c, d, mat))

    def tri(self, a, b, c, mat):
        self.tris.append((a, b, c, mat))


@dataclass
class SceneDef:
    camera: Camera = field(default_factory=Camera)
    materials: list = field(default_factory=list)
    light: DeltaLight = field(default_factory=DeltaLight)
    objects: list = field(default_factory=list)
    dt_frame: float = 1.0

    def add_material(self, m: Material) -> int:
        self.materials.append(m)
        return len(self.materials) - 1

    def to_desc(self):
        """Lower to tofr_scene_desc.  Returns (desc, keepalive)."""
        keep = []
        d = F.SceneDesc()
        cam = self.camera
        d.cam_position = F.D3(*cam.base.position)
        d.cam_forward = F.D3(*cam.base.forward)
        d.cam_up = F.D3(*cam.base.up)
        d.fov_y = cam.fov_y
        d.width = cam.width
        d.height = cam.height
        if cam.track:
            keys = (F.CameraKey * len(cam.track))()
            for i, (fr, p) in enumerate(cam.track):
                keys[i].frame = fr
                keys[i].position = F.D3(*p.position)
                keys[i].forward = F.D3(*p.forward)
                keys[i].up = F.D3(*p.up)
            keep.append(keys)
            d.n_cam_keys = len(cam.track)
            d.cam_keys = keys
        mats = (F.Material * max(1, len(self.materials)))()
        for i, m in enumerate(self.materials):
            mats[i].kind = m.kind
            mats[i].albedo = F.D3(*m.albedo)
            mats[i].roughness = m.roughness
        keep.append(mats)
        d.n_materials = len(self.materials)
        d.materials = mats
        L = self.light
        d.light.regime = L.regime
        d.light.position = F.D3(*L.position)
        d.light.direction = F.D3(*L.direction)
        d.light.cone_half_angle = L.cone_half_angle
        d.light.intensity = F.D3(*L.intensity)
        objs = (F.ObjectDesc * max(1, len(self.objects)))()
        for i, o in enumerate(self.objects):
            n = len(o.tris)
            verts = (C.c_double * (9 * max(1, n)))()
            mids = (C.c_int32 * max(1, n))()
            for t, (a, b, c, m) in enumerate(o.tris):
                verts[9 * t:9 * t + 9] = [*a, *b, *c]
                mids[t] = m
            name = o.name.encode()
            keep += [verts, mids, name]
            objs[i].name = name
            objs[i].n_tris = n
            objs[i].verts = verts
            objs[i].materials = mids
            if o.track:
                ks = (F.PoseKey * len(o.track))()
                for j, k in enumerate(o.track):
                    ks[j].frame = k.frame
                    ks[j].q = (C.c_double * 4)(*k.q)
                    ks[j].t = F.D3(*k.t)
                keep.append(ks)
                objs[i].n_keys = len(o.track)
                objs[i].keys = ks
        keep.append(objs)
        d.n_objects = len(self.objects)
        d.objects = objs
        d.dt_frame = self.dt_frame
        return d, keep


def to_scn(sd: SceneDef) -> str:
    """Scene description text (scene_io.hpp grammar) of a SceneDef, for the
    CLI.  Rotated pose keys are not expressible from a quaternion here and
    raise ValueError; translation tracks and static scenes round-trip."""
    g = lambda v: format(float(v), ".17g")  # noqa: E731
    v3 = lambda t: " ".join(g(x) for x in t)  # noqa: E731
    cam = sd.camera
    lines = ["camera {", f"  position {v3(cam.base.position)}", f"  forward {v3(cam.base.forward)}",
             f"  up {v3(cam.base.up)}", f"  fov_deg {g(cam.fov_y * 180.0 / KPI)}",
             f"  resolution {cam.width} {cam.height}"]
    if cam.track:
        lines.append("  track {")
        for fr, p in cam.track:
            lines.append(f"    frame {g(fr)} position {v3(p.position)} forward {v3(p.forward)} up {v3(p.up)}")
        lines.append("  }")
    lines += ["}", f"dt_frame {g(sd.dt_frame)}"]
    kinds = {F.MAT_DIFFUSE: "diffuse", F.MAT_GLOSSY: "glossy", F.MAT_MIRROR: "mirror"}
    for i, m in enumerate(sd.materials):
        lines.append(f"material m{i} {{ kind {kinds[m.kind]} albedo {v3(m.albedo)} roughness {g(m.roughness)} }}")
    L = sd.light
    lines += ["light {", f"  regime {'wide' if L.regime == F.LIGHT_WIDE else 'collimated'}",
              f"  position {v3(L.position)}", f"  direction {v3(L.direction)}",
              f"  cone_deg {g(L.cone_half_angle * 180.0 / KPI)}", f"  intensity {v3(L.intensity)}", "}"]
    for i, o in enumerate(sd.objects):
        lines.append(f"object {o.name or f'o{i}'} {{")
        cur = None
        for (a, b, c, m) in o.tris:
            if m != cur:
                lines.append(f"  material m{m}")
                cur = m
            lines.append(f"  tri {v3(a)}   {v3(b)}   {v3(c)}")
        if o.track:
            lines.append("  track {")
            for k in o.track:
                if tuple(k.q) != (1.0, 0.0, 0.0, 0.0):
                    raise ValueError("to_scn: rotated pose keys are not supported")
                lines.append(f"    frame {g(k.frame)} translate {v3(k.t)}")
            lines.append("  }")
        lines.append("}")
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# test-suite builders (test_scenes.hpp:17-101)

def cornell_box(collimated=True, resolution=32, tall_box_material=-1, tall_box_roughness=0.3,
                tall_box_kind=F.MAT_GLOSSY) -> SceneDef:
    d = SceneDef()
    white = d.add_material(Material(F.MAT_DIFFUSE, (0.73, 0.73, 0.73), 0.5))
    red = d.add_material(Material(F.MAT_DIFFUSE, (0.63, 0.065, 0.05), 0.5))
    green = d.add_material(Material(F.MAT_DIFFUSE, (0.14, 0.45, 0.091), 0.5))
    d.add_material(Material(tall_box_kind, (0.8, 0.8, 0.8), tall_box_roughness))
    box = ObjectDef("box")
    box.quad((-1, -1, -1), (1, -1, -1), (1, -1, 1), (-1, -1, 1), white)
    box.quad((-1, 1, -1), (-1, 1, 1), (1, 1, 1), (1, 1, -1), white)
    box.quad((-1, -1, -1), (-1, 1, -1), (1, 1, -1), (1, -1, -1), white)
    box.quad((-1, -1, -1), (-1, -1, 1), (-1, 1, 1), (-1, 1, -1), red)
    box.quad((1, -1, -1), (1, 1, -1), (1, 1, 1), (1, -1, 1), green)
    d.objects.append(box)
    if tall_box_material >= 0:
        inner = ObjectDef("tall_box")
        m = tall_box_material
        x0, x1, z0, z1, y0, y1 = -0.55, -0.05, -0.6, -0.1, -1.0, 0.2
        inner.quad((x0, y0, z0), (x0, y1, z0), (x1, y1, z0), (x1, y0, z0), m)
        inner.quad((x0, y0, z1), (x1, y0, z1), (x1, y1, z1), (x0, y1, z1), m)
        inner.quad((x0, y0, z0), (x0, y0, z1), (x0, y1, z1), (x0, y1, z0), m)
        inner.quad((x1, y0, z0), (x1, y1, z0), (x1, y1, z1), (x1, y0, z1), m)
        inner.quad((x0, y1, z0), (x0, y1, z1), (x1, y1, z1), (x1, y1, z0), m)
        d.objects.append(inner)
    d.camera.base = CameraPose((0, 0, 3), (0, 0, -1), (0, 1, 0))
    d.camera.fov_y = 2.0 * math.atan(1.0 / 3.0)
    d.camera.width = resolution
    d.camera.height = resolution
    if collimated:
        d.light = DeltaLight((0, 0.6, 3), (0, 0, -1), 0.0, (40, 40, 40), F.LIGHT_COLLIMATED)
    else:
        d.light = DeltaLight((0, 0.9, 0), (0, -1, 0), 2.8, (8, 8, 8), F.LIGHT_WIDE)
    return d


def flat_wall(resolution=8, wall_albedo=0.7) -> SceneDef:
    d = SceneDef()
    white = d.add_material(Material(F.MAT_DIFFUSE, (wall_albedo,) * 3, 0.5))
    wall = ObjectDef("wall")
    wall.quad((-8, -8, 0), (8, -8, 0), (8, 8, 0), (-8, 8, 0), white)
    d.objects.append(wall)
    d.camera.base = CameraPose((0, 0, 4), (0, 0, -1), (0, 1, 0))
    d.camera.fov_y = deg2rad(40)
    d.camera.width = resolution
    d.camera.height = resolution
    d.light = DeltaLight((1.5, 1.5, 3), (0, 0, -1), 2.9, (10, 10, 10), F.LIGHT_WIDE)
    return d


# ---------------------------------------------------------------------------
# bundled scenes (proj/scenes/*.scn), as the .scn parser would build them

def _cornell_shell(d: SceneDef, white, red, green) -> None:
    box = ObjectDef("box")
    box.quad((-1, -1, -1), (1, -1, -1), (1, -1, 1), (-1, -1, 1), white)
    box.quad((-1, 1, -1), (-1, 1, 1), (1, 1, 1), (1, 1, -1), white)
    box.quad((-1, -1, -1), (-1, 1, -1), (1, 1, -1), (1, -1, -1), white)
    left = ObjectDef("left")
    left.quad((-1, -1, -1), (-1, -1, 1), (-1, 1, 1), (-1, 1, -1), red)
    right = ObjectDef("right")
    right.quad((1, -1, -1), (1, 1, -1), (1, 1, 1), (1, -1, 1), green)
    d.objects += [box, left, right]


def _cornell_materials(d: SceneDef):
    white = d.add_material(Material(F.MAT_DIFFUSE, (0.73, 0.73, 0.73)))
    red = d.add_material(Material(F.MAT_DIFFUSE, (0.63, 0.065, 0.05)))
    green = d.add_material(Material(F.MAT_DIFFUSE, (0.14, 0.45, 0.091)))
    metal = d.add_material(Material(F.MAT_GLOSSY, (0.8, 0.8, 0.8), 0.3))
    return white, red, green, metal


def cornell() -> SceneDef:
    """scenes/cornell.scn: 2x2x2 open box, collimated laser on the back wall."""
    d = SceneDef()
    d.camera = Camera(CameraPose((0, 0, 3), normalize((0, 0, -1)), normalize((0, 1, 0))), deg2rad(36.87), 128, 128)
    white, red, green, _ = _cornell_materials(d)
    d.light = DeltaLight((0, 0.6, 3), normalize((0, 0, -1)), 1e-3, (40, 40, 40), F.LIGHT_COLLIMATED)
    _cornell_shell(d, white, red, green)
    return d


def cornell_wide() -> SceneDef:
    """scenes/cornell_wide.scn: wide spotlight below the ceiling, glossy tall box."""
    d = SceneDef()
    d.camera = Camera(CameraPose((0, 0, 3), normalize((0, 0, -1)), normalize((0, 1, 0))), deg2rad(36.87), 128, 128)
    white, red, green, metal = _cornell_materials(d)
    d.light = DeltaLight((0, 0.9, 0), normalize((0, -1, 0)), deg2rad(160), (8, 8, 8), F.LIGHT_WIDE)
    _cornell_shell(d, white, red, green)
    tall = ObjectDef("tall_box")
    tall.quad((-0.55, -1, -0.6), (-0.55, 0.2, -0.6), (-0.05, 0.2, -0.6), (-0.05, -1, -0.6), metal)
    tall.quad((-0.55, -1, -0.1), (-0.05, -1, -0.1), (-0.05, 0.2, -0.1), (-0.55, 0.2, -0.1), metal)
    tall.quad((-0.55, -1, -0.6), (-0.55, -1, -0.1), (-0.55, 0.2, -0.1), (-0.55, 0.2, -0.6), metal)
    tall.quad((-0.05, -1, -0.6), (-0.05, 0.2, -0.6), (-0.05, 0.2, -0.1), (-0.05, -1, -0.1), metal)
    tall.quad((-0.55, 0.2, -0.6), (-0.55, 0.2, -0.1), (-0.05, 0.2, -0.1), (-0.05, 0.2, -0.6), metal)
    d.objects.append(tall)
    return d


def boxes_doppler() -> SceneDef:
    """scenes/boxes_doppler.scn: backdrop + receding big box + approaching small box."""
    d = SceneDef()
    d.camera = Camera(CameraPose((0, 0, 4), normalize((0, 0, -1)), normalize((0, 1, 0))), deg2rad(40), 96, 96)
    d.dt_frame = 1.0
    white = d.add_material(Material(F.MAT_DIFFUSE, (0.7, 0.7, 0.7)))
    blue = d.add_material(Material(F.MAT_DIFFUSE, (0.2, 0.3, 0.7)))
    amber = d.add_material(Material(F.MAT_DIFFUSE, (0.8, 0.55, 0.2)))
    d.light = DeltaLight((0, 1.6, 3.5), normalize((0, -0.4, -1)), deg2rad(150), (12, 12, 12), F.LIGHT_WIDE)
    back = ObjectDef("backdrop")
    back.quad((-3, -1.5, -2), (3, -1.5, -2), (3, 2.5, -2), (-3, 2.5, -2), white)
    back.quad((-3, -1.5, -2), (-3, -1.5, 2), (3, -1.5, 2), (3, -1.5, -2), white)
    big = ObjectDef("big_box")
    big.quad((-1.4, -1.5, -0.6), (-0.4, -1.5, -0.6), (-0.4, 0.0, -0.6), (-1.4, 0.0, -0.6), blue)
    big.quad((-1.4, -1.5, -1.4), (-1.4, 0.0, -1.4), (-0.4, 0.0, -1.4), (-0.4, -1.5, -1.4), blue)
    big.quad((-1.4, -1.5, -1.4), (-1.4, -1.5, -0.6), (-1.4, 0.0, -0.6), (-1.4, 0.0, -1.4), blue)
    big.quad((-0.4, -1.5, -1.4), (-0.4, 0.0, -1.4), (-0.4, 0.0, -0.6), (-0.4, -1.5, -0.6), blue)
    big.quad((-1.4, 0.0, -1.4), (-1.4, 0.0, -0.6), (-0.4, 0.0, -0.6), (-0.4, 0.0, -1.4), blue)
    big.track = [PoseKey(0, t=(0, 0, 0)), PoseKey(40, t=(0, 0, -2.0))]
    small = ObjectDef("small_box")
    small.quad((0.5, -1.5, 0.0), (1.1, -1.5, 0.0), (1.1, -0.7, 0.0), (0.5, -0.7, 0.0), amber)
    small.quad((0.5, -1.5, -0.6), (0.5, -0.7, -0.6), (1.1, -0.7, -0.6), (1.1, -1.5, -0.6), amber)
    small.quad((0.5, -1.5, -0.6), (0.5, -1.5, 0.0), (0.5, -0.7, 0.0), (0.5, -0.7, -0.6), amber)
    small.quad((1.1, -1.5, -0.6), (1.1, -0.7, -0.6), (1.1, -0.7, 0.0), (1.1, -1.5, 0.0), amber)
    small.quad((0.5, -0.7, -0.6), (0.5, -0.7, 0.0), (1.1, -0.7, 0.0), (1.1, -0.7, -0.6), amber)
    small.track = [PoseKey(0, t=(0, 0, 0)), PoseKey(40, t=(0, 0, 1.2))]
    d.objects += [back, big, small]
    return d


BUNDLED = {"cornell": cornell, "cornell_wide": cornell_wide, "boxes_doppler": boxes_doppler}


def bundled(name: str, width: int | None = None, height: int | None = None) -> SceneDef:
    if name in ("mesh", "mesh_anim"):  # the BVH stress scene (not a bundled .scn)
        return mesh_scene(width or 256, height, animated=name == "mesh_anim")
    d = BUNDLED[name]()
    if width:
        d.camera.width = width
        d.camera.height = height or width
    return d


# ---------------------------------------------------------------------------
# BVH stress scene: the cornell_wide box with a finely
# tessellated, displaced torus loaded through the OBJ path (scene_io.hpp:102-132)


def torus_mesh(nu: int = 320, nv: int = 160, R: float = 0.45, r: float = 0.18, bumps: float = 0.04,
               center=(0.0, -0.35, 0.0)):
    """Displaced torus: (vertices, faces) with 2 * nu * nv triangles and no
    degenerate ones.  Vertices are rounded through 17 significant digits, so
    the OBJ text (write_torus_obj) and the inline triangles (mesh_scene) hold
    the same doubles."""
    verts = []
    cx, cy, cz = center
    for i in range(nu):
        u = 2 * math.pi * i / nu
        for j in range(nv):
            v = 2 * math.pi * j / nv
            rr = r * (1.0 + bumps / r * math.sin(7 * u) * math.sin(5 * v))
            x = (R + rr * math.cos(v)) * math.cos(u)
            z = (R + rr * math.cos(v)) * math.sin(u)
            y = rr * math.sin(v)
            verts.append(tuple(float(f"{c:.17g}") for c in (x + cx, y * 0.8 + cy, z + cz)))
    faces = []
    for i in range(nu):
        for j in range(nv):
            a = i * nv + j
            b = ((i + 1) % nu) * nv + j
            c = ((i + 1) % nu) * nv + (j + 1) % nv
            d = i * nv + (j + 1) % nv
            faces += [(a, b, c), (a, c, d)]
    return verts, faces


def write_torus_obj(path, nu: int = 320, nv: int = 160) -> int:
    """The torus as an OBJ triangle list ("v" / "f" records, scene_io.hpp:102-132)."""
    verts, faces = torus_mesh(nu, nv)
    lines = [f"v {x:.17g} {y:.17g} {z:.17g}" for x, y, z in verts]
    lines += [f"f {a + 1} {b + 1} {c + 1}" for a, b, c in faces]
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    return len(faces)


def mesh_scene(width: int = 256, height: int | None = None, nu: int = 320, nv: int = 160,
               animated: bool = False) -> SceneDef:
    """cornell_wide's box, light and camera plus the torus (glossy) with its
    triangles inline: the same scene as mesh_scene_file's .scn + OBJ.
    animated: the torus turns about y (30 degrees over 20 frames) and drifts
    along x, so every frame needs a new BVH (the device build's case)."""
    d = cornell_wide()
    d.objects = d.objects[:3]  # box, left, right (no tall box)
    metal = 3
    verts, faces = torus_mesh(nu, nv)
    t = ObjectDef("torus")
    for a, b, c in faces:
        t.tri(verts[a], verts[b], verts[c], metal)
    if animated:
        half = math.radians(30.0) / 2
        t.track = [PoseKey(0.0, (1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0)),
                   PoseKey(20.0, (math.cos(half), 0.0, math.sin(half), 0.0), (0.1, 0.0, 0.0))]
    d.objects.append(t)
    d.camera.width = width
    d.camera.height = height or width
    return d


def mesh_scene_file(directory, width: int = 256, height: int = 256, nu: int = 320, nv: int = 160) -> str:
    """Writes torus.obj + mesh_box.scn into `directory` (cornell_wide's box,
    wide light and camera; 2 * nu * nv torus triangles: 102,400 by default)
    and returns the .scn path (load with Scene.create / the oracle's RefScene)."""
    from pathlib import Path
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    write_torus_obj(d / "torus.obj", nu, nv)
    scn = f"""camera {{
  position 0 0 3
  forward 0 0 -1
  up 0 1 0
  fov_deg 36.87
  resolution {width} {height}
}}
material white {{ kind diffuse albedo 0.73 0.73 0.73 }}
material red   {{ kind diffuse albedo 0.63 0.065 0.05 }}
material green {{ kind diffuse albedo 0.14 0.45 0.091 }}
material metal {{ kind glossy albedo 0.8 0.8 0.8 roughness 0.3 }}
light {{
  regime wide
  position 0 0.9 0
  direction 0 -1 0
  cone_deg 160
  intensity 8 8 8
}}
object box {{
  material white
  quad -1 -1 -1   1 -1 -1   1 -1 1   -1 -1 1
  quad -1 1 -1   -1 1 1   1 1 1   1 1 -1
  quad -1 -1 -1   -1 1 -1   1 1 -1   1 -1 -1
}}
object left {{
  material red
  quad -1 -1 -1   -1 -1 1   -1 1 1   -1 1 -1
}}
object right {{
  material green
  quad 1 -1 -1   1 1 -1   1 1 1   1 -1 1
}}
object torus {{
  material metal
  obj torus.obj
}}
"""
    p = d / "mesh_box.scn"
    p.write_text(scn)
    return str(p)
