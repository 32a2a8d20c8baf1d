// host_scene.h -- host runtime for the ToF renderer: scene definition, the
// per-frame snapshot (rigid motion, camera, collimated beam) and the binned
// SAH BVH whose output is re-laid out for the device.
//
// The BVH build is the reference algorithm (geometry.hpp:234-317) so that the
// device tree -- and with it traversal order and the ellipsoid-descent
// probabilities -- is identical to the CPU oracle's.  Frame construction
// follows build_frame (scene.hpp:479-548); the .scn grammar follows
// parse_scene (scene_io.hpp:136-302).
#pragma once

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tofr_geom.h"

namespace tofr_b200 {

struct HMaterial {
    int kind = MAT_DIFFUSE;
    V3 albedo{0.5, 0.5, 0.5};
    double roughness = 0.5;
    bool reconnectable() const {
        return kind == MAT_DIFFUSE || (kind == MAT_GLOSSY && roughness >= 0.2);
    }
};

struct HTri {
    V3 v0, v1, v2, n;
    int material = 0, object = 0;
    double area = 0;
};
HTri make_tri(const V3& a, const V3& b, const V3& c, int material, int object = 0);

struct HQuat {
    double w = 1, x = 0, y = 0, z = 0;
};
struct HPose {
    HQuat q;
    V3 t{0, 0, 0};
};
struct HPoseKey {
    double frame = 0;
    HPose pose;
};
struct HTrack {
    std::vector<HPoseKey> keys;
    bool animated() const { return keys.size() > 1; }
    HPose pose_at(double frame) const;
    bool moving_at(double frame) const;  // velocity_field(...).moving
};

struct HObject {
    std::string name;
    std::vector<HTri> local;
    HTrack track;
};

struct HCamPose {
    V3 position{0, 0, 0};
    V3 forward{0, 0, -1};
    V3 up{0, 1, 0};
};

struct HCamera {
    HCamPose base;
    double fov_y = 45 * kPi / 180.0;
    int width = 128, height = 128;
    std::vector<std::pair<double, HCamPose>> track;
    HCamPose pose_at(double frame) const;
};

struct HLight {
    V3 position{0, 0, 0};
    V3 direction{0, 0, -1};
    double cone_half_angle = kPi / 2;
    V3 intensity{1, 1, 1};
    int regime = LIGHT_WIDE;
};

struct HScene {
    HCamera camera;
    std::vector<HMaterial> materials;
    HLight light;
    std::vector<HObject> objects;
    double dt_frame = 1.0;
};

struct ParseError : std::runtime_error {
    int line, col;
    ParseError(int l, int c, const std::string& m) : std::runtime_error(m), line(l), col(c) {}
};

HScene parse_scene_text(const std::string& text, const std::string& base_dir);
HScene load_scene_file(const std::string& path);

// Host BVH node (reference layout, geometry.hpp:126-134).
struct HNode {
    V3 lo{kInf, kInf, kInf}, hi{-kInf, -kInf, -kInf};
    double tri_area = 0;
    int left = -1, right = -1, first = 0, count = 0, parent = -1;
};

// Packed device image of one frame: every array the kernels read, laid out
// back to back in one allocation so a frame upload is a single copy.
struct PackedFrame {
    std::vector<unsigned char> blob;
    size_t off_nodes = 0, off_aux = 0, off_isect = 0, off_tri_id = 0, off_tri = 0, off_mats = 0, off_vel = 0,
           off_tframe = 0;
    FrameView view;  // pointers are offsets until rebased
};

struct HFrame {
    double frame = 0;
    std::vector<HTri> tris;
    std::vector<HNode> nodes;
    std::vector<int> tri_order, leaf_of;
    double diag = 0, eps_ray = 0;
    GCam cam;
    GLight light;
    GLightSub lsub;
    int geo_motion = 0;
    int max_depth = 0;  // deepest root-to-leaf path (for sanity checks)
    std::vector<GVel> obj_vel;  // velocity_field per object (scene.hpp:318-335)
    V3 cam_vel{0, 0, 0};
};

// Builds the snapshot for `frame` (scene.hpp:479-548).  Throws
// std::runtime_error("bvh: empty mesh" / "bvh: degenerate triangle").
HFrame build_frame(const HScene& s, double frame, bool build_bvh = true);
// pack_frame's layout for an nn-node tree built elsewhere (the device): the
// blob holds the materials and velocity fields only; the rest is written in place
PackedFrame pack_frame_shell(const HScene& s, const HFrame& f, int nn, int frame_id);

// Device layout of a frame; `view` pointers are relative to blob start.
PackedFrame pack_frame(const HScene& s, const HFrame& f, int frame_id);
// Returns a FrameView whose pointers address `base` (host or device copy).
FrameView rebase_view(const PackedFrame& p, const unsigned char* base);

std::vector<GMat> device_materials(const HScene& s);

}  // namespace tofr_b200
