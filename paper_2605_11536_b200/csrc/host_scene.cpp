// host_scene.cpp -- scene parsing, per-frame snapshot and SAH BVH build.
// See host_scene.h for the reference sections each part follows.
#include "host_scene.h"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

namespace tofr_b200 {

HTri make_tri(const V3& a, const V3& b, const V3& c, int material, int object) {
    // geometry.hpp:25-38
    HTri t;
    t.v0 = a;
    t.v1 = b;
    t.v2 = c;
    V3 cr = cross(b - a, c - a);
    double l = norm(cr);
    t.area = 0.5 * l;
    t.n = l > 0 ? cr / l : V3{0, 0, 1};
    t.material = material;
    t.object = object;
    return t;
}

// ---------------------------------------------------------------------------
// rigid motion (scene.hpp:213-335)

static HQuat quat_normalized(const HQuat& q) {
    double n = std::sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    return {q.w / n, q.x / n, q.y / n, q.z / n};
}

static HQuat quat_axis_angle(const V3& axis, double angle) {
    double s = std::sin(angle / 2);
    V3 a = normalize(axis);
    return {std::cos(angle / 2), a.x * s, a.y * s, a.z * s};
}

static M3 quat_matrix(const HQuat& q) {
    double w = q.w, x = q.x, y = q.y, z = q.z;
    M3 r;
    r.m[0][0] = 1 - 2 * (y * y + z * z);
    r.m[0][1] = 2 * (x * y - z * w);
    r.m[0][2] = 2 * (x * z + y * w);
    r.m[1][0] = 2 * (x * y + z * w);
    r.m[1][1] = 1 - 2 * (x * x + z * z);
    r.m[1][2] = 2 * (y * z - x * w);
    r.m[2][0] = 2 * (x * z - y * w);
    r.m[2][1] = 2 * (y * z + x * w);
    r.m[2][2] = 1 - 2 * (x * x + y * y);
    return r;
}

static HQuat slerp(const HQuat& a, HQuat b, double t) {
    double d = a.w * b.w + a.x * b.x + a.y * b.y + a.z * b.z;
    if (d < 0) {
        b = {-b.w, -b.x, -b.y, -b.z};
        d = -d;
    }
    if (d > 0.9995) {
        HQuat r{a.w + (b.w - a.w) * t, a.x + (b.x - a.x) * t, a.y + (b.y - a.y) * t,
                a.z + (b.z - a.z) * t};
        return quat_normalized(r);
    }
    double th = std::acos(d);
    double sa = std::sin((1 - t) * th) / std::sin(th);
    double sb = std::sin(t * th) / std::sin(th);
    return quat_normalized(
        {a.w * sa + b.w * sb, a.x * sa + b.x * sb, a.y * sa + b.y * sb, a.z * sa + b.z * sb});
}

HPose HTrack::pose_at(double frame) const {
    if (keys.empty()) return {};
    if (frame <= keys.front().frame) return keys.front().pose;
    if (frame >= keys.back().frame) return keys.back().pose;
    size_t i = 1;
    while (keys[i].frame < frame) ++i;
    const HPoseKey& a = keys[i - 1];
    const HPoseKey& b = keys[i];
    double u = (frame - a.frame) / (b.frame - a.frame);
    HPose p;
    p.t = a.pose.t * (1 - u) + b.pose.t * u;
    p.q = slerp(a.pose.q, b.pose.q, u);
    return p;
}

bool HTrack::moving_at(double f) const {
    // velocity_field (scene.hpp:318-335): moving iff animated and the clamped
    // central-difference window is non-empty.
    if (!animated()) return false;
    double fmin = keys.front().frame, fmax = keys.back().frame;
    double lo = std::max(fmin, f - 1.0);
    double hi = std::min(fmax, f + 1.0);
    if (hi <= lo) {
        lo = f;
        hi = f;
    }
    return hi > lo;
}

HCamPose HCamera::pose_at(double frame) const {
    if (track.empty()) return base;
    if (frame <= track.front().first) return track.front().second;
    if (frame >= track.back().first) return track.back().second;
    size_t i = 1;
    while (track[i].first < frame) ++i;
    const auto& a = track[i - 1];
    const auto& b = track[i];
    double u = (frame - a.first) / (b.first - a.first);
    HCamPose p;
    p.position = a.second.position * (1 - u) + b.second.position * u;
    p.forward = normalize(a.second.forward * (1 - u) + b.second.forward * u);
    p.up = normalize(a.second.up * (1 - u) + b.second.up * u);
    return p;
}

// ---------------------------------------------------------------------------
// .scn parser (scene_io.hpp:18-302)

namespace {

struct Lexer {
    std::string src;
    size_t pos = 0;
    int line = 1, col = 1;

    void advance() {
        if (src[pos] == '\n') {
            line++;
            col = 1;
        } else {
            col++;
        }
        pos++;
    }
    void skip_ws() {
        while (pos < src.size()) {
            char c = src[pos];
            if (c == '#') {
                while (pos < src.size() && src[pos] != '\n') advance();
            } else if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
                advance();
            } else {
                break;
            }
        }
    }
    bool eof() {
        skip_ws();
        return pos >= src.size();
    }
    std::string next() {
        skip_ws();
        if (pos >= src.size()) throw ParseError(line, col, "unexpected end of file");
        if (src[pos] == '{' || src[pos] == '}') {
            std::string t(1, src[pos]);
            advance();
            return t;
        }
        std::string t;
        while (pos < src.size() && !std::isspace((unsigned char)src[pos]) && src[pos] != '{' &&
               src[pos] != '}' && src[pos] != '#') {
            t += src[pos];
            advance();
        }
        return t;
    }
    std::string peek() {
        size_t p = pos;
        int l = line, c = col;
        std::string t = eof() ? "" : next();
        pos = p;
        line = l;
        col = c;
        return t;
    }
    double number() {
        skip_ws();
        int l = line, c = col;
        std::string t = next();
        char* end = nullptr;
        double v = std::strtod(t.c_str(), &end);
        if (end == t.c_str() || *end != '\0')
            throw ParseError(l, c, "expected a number, got '" + t + "'");
        return v;
    }
    V3 vec3() {
        double x = number(), y = number(), z = number();
        return {x, y, z};
    }
    void expect(const std::string& tok) {
        skip_ws();
        int l = line, c = col;
        std::string t = next();
        if (t != tok) throw ParseError(l, c, "expected '" + tok + "', got '" + t + "'");
    }
    [[noreturn]] void fail(const std::string& msg) { throw ParseError(line, col, msg); }
};

double deg2rad(double d) { return d * kPi / 180.0; }

std::vector<HTri> load_obj(const std::string& path, int material) {
    // minimal OBJ: "v x y z", "f i j k ..." fan-triangulated (scene_io.hpp:102-132)
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cannot open mesh file " + path);
    std::vector<V3> verts;
    std::vector<HTri> tris;
    std::string word, lbuf;
    while (std::getline(f, lbuf)) {
        std::istringstream ls(lbuf);
        if (!(ls >> word)) continue;
        if (word == "v") {
            V3 v{0, 0, 0};
            ls >> v.x >> v.y >> v.z;
            verts.push_back(v);
        } else if (word == "f") {
            std::vector<int> idx;
            std::string tok;
            while (ls >> tok) {
                size_t slash = tok.find('/');
                int i = std::stoi(slash == std::string::npos ? tok : tok.substr(0, slash));
                if (i < 0) i = int(verts.size()) + 1 + i;
                idx.push_back(i - 1);
            }
            for (size_t k = 2; k < idx.size(); ++k)
                tris.push_back(make_tri(verts.at(idx[0]), verts.at(idx[k - 1]),
                                        verts.at(idx[k]), material));
        }
    }
    return tris;
}

}  // namespace

HScene parse_scene_text(const std::string& text, const std::string& base_dir) {
    Lexer lx;
    lx.src = text;
    HScene def;
    std::map<std::string, int> mat_ids;
    bool have_light = false;

    auto parse_track = [&](HTrack& track) {
        lx.expect("{");
        while (lx.peek() != "}") {
            lx.expect("frame");
            HPoseKey key;
            key.frame = lx.number();
            for (std::string w = lx.peek(); w == "translate" || w == "rotate"; w = lx.peek()) {
                lx.next();
                if (w == "translate") {
                    key.pose.t = lx.vec3();
                } else {
                    lx.expect("axis");
                    V3 axis = lx.vec3();
                    lx.expect("deg");
                    double deg = lx.number();
                    key.pose.q = quat_axis_angle(axis, deg2rad(deg));
                }
            }
            track.keys.push_back(key);
        }
        lx.expect("}");
    };

    while (!lx.eof()) {
        int l = lx.line, c = lx.col;
        std::string section = lx.next();
        if (section == "camera") {
            lx.expect("{");
            while (lx.peek() != "}") {
                std::string key = lx.next();
                if (key == "position")
                    def.camera.base.position = lx.vec3();
                else if (key == "forward")
                    def.camera.base.forward = normalize(lx.vec3());
                else if (key == "up")
                    def.camera.base.up = normalize(lx.vec3());
                else if (key == "fov_deg")
                    def.camera.fov_y = deg2rad(lx.number());
                else if (key == "resolution") {
                    def.camera.width = int(lx.number());
                    def.camera.height = int(lx.number());
                } else if (key == "track") {
                    lx.expect("{");
                    while (lx.peek() != "}") {
                        lx.expect("frame");
                        double fi = lx.number();
                        HCamPose p = def.camera.base;
                        for (std::string w = lx.peek();
                             w == "position" || w == "forward" || w == "up"; w = lx.peek()) {
                            lx.next();
                            if (w == "position")
                                p.position = lx.vec3();
                            else if (w == "forward")
                                p.forward = normalize(lx.vec3());
                            else
                                p.up = normalize(lx.vec3());
                        }
                        def.camera.track.emplace_back(fi, p);
                    }
                    lx.expect("}");
                } else {
                    lx.fail("unknown camera key '" + key + "'");
                }
            }
            lx.expect("}");
        } else if (section == "material") {
            std::string name = lx.next();
            HMaterial m;
            lx.expect("{");
            while (lx.peek() != "}") {
                std::string key = lx.next();
                if (key == "kind") {
                    std::string kind = lx.next();
                    if (kind == "diffuse")
                        m.kind = MAT_DIFFUSE;
                    else if (kind == "glossy")
                        m.kind = MAT_GLOSSY;
                    else if (kind == "mirror")
                        m.kind = MAT_MIRROR;
                    else
                        lx.fail("unknown material kind '" + kind + "'");
                } else if (key == "albedo") {
                    m.albedo = lx.vec3();
                } else if (key == "roughness") {
                    m.roughness = lx.number();
                } else {
                    lx.fail("unknown material key '" + key + "'");
                }
            }
            lx.expect("}");
            def.materials.push_back(m);
            mat_ids[name] = int(def.materials.size()) - 1;
        } else if (section == "light") {
            lx.expect("{");
            while (lx.peek() != "}") {
                std::string key = lx.next();
                if (key == "regime") {
                    std::string r = lx.next();
                    if (r == "wide")
                        def.light.regime = LIGHT_WIDE;
                    else if (r == "collimated")
                        def.light.regime = LIGHT_COLLIMATED;
                    else
                        lx.fail("unknown light regime '" + r + "'");
                } else if (key == "position") {
                    def.light.position = lx.vec3();
                } else if (key == "direction") {
                    def.light.direction = normalize(lx.vec3());
                } else if (key == "cone_deg") {
                    def.light.cone_half_angle = deg2rad(lx.number());
                } else if (key == "intensity") {
                    def.light.intensity = lx.vec3();
                } else {
                    lx.fail("unknown light key '" + key + "'");
                }
            }
            lx.expect("}");
            if (def.light.regime == LIGHT_COLLIMATED && def.light.cone_half_angle > 1e-3)
                def.light.cone_half_angle = 1e-3;
            have_light = true;
        } else if (section == "dt_frame") {
            def.dt_frame = lx.number();
        } else if (section == "object") {
            HObject obj;
            obj.name = lx.next();
            int mat = 0;
            lx.expect("{");
            while (lx.peek() != "}") {
                std::string key = lx.next();
                if (key == "material") {
                    std::string name = lx.next();
                    auto it = mat_ids.find(name);
                    if (it == mat_ids.end()) lx.fail("unknown material '" + name + "'");
                    mat = it->second;
                } else if (key == "tri") {
                    V3 a = lx.vec3(), b = lx.vec3(), cc = lx.vec3();
                    obj.local.push_back(make_tri(a, b, cc, mat));
                } else if (key == "quad") {
                    V3 a = lx.vec3(), b = lx.vec3(), cc = lx.vec3(), d = lx.vec3();
                    obj.local.push_back(make_tri(a, b, cc, mat));
                    obj.local.push_back(make_tri(a, cc, d, mat));
                } else if (key == "obj") {
                    std::string rel = lx.next();
                    for (const HTri& t : load_obj(base_dir + "/" + rel, mat)) obj.local.push_back(t);
                } else if (key == "track") {
                    parse_track(obj.track);
                } else {
                    lx.fail("unknown object key '" + key + "'");
                }
            }
            lx.expect("}");
            def.objects.push_back(std::move(obj));
        } else {
            throw ParseError(l, c, "unknown section '" + section + "'");
        }
    }
    if (def.materials.empty()) def.materials.push_back(HMaterial{});
    if (!have_light) throw ParseError(lx.line, lx.col, "scene has no light");
    if (def.objects.empty()) throw ParseError(lx.line, lx.col, "scene has no objects");
    return def;
}

HScene load_scene_file(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cannot open scene file " + path);
    std::ostringstream ss;
    ss << f.rdbuf();
    std::string dir = ".";
    size_t slash = path.find_last_of('/');
    if (slash != std::string::npos) dir = path.substr(0, slash);
    return parse_scene_text(ss.str(), dir);
}

// ---------------------------------------------------------------------------
// binned-SAH BVH (geometry.hpp:124-325)

namespace {

struct Box {
    V3 lo{kInf, kInf, kInf}, hi{-kInf, -kInf, -kInf};
    void grow(const V3& p) {
        lo = vmin(lo, p);
        hi = vmax(hi, p);
    }
    void grow(const Box& b) {
        lo = vmin(lo, b.lo);
        hi = vmax(hi, b.hi);
    }
    V3 extent() const { return hi - lo; }
    double area() const {
        V3 e = extent();
        if (e.x < 0) return 0;
        return 2.0 * (e.x * e.y + e.y * e.z + e.z * e.x);
    }
};

struct SahBuilder {
    const std::vector<HTri>& tris;
    std::vector<int>& order;
    std::vector<HNode>& nodes;

    int build(int first, int count, int parent) {
        int idx = int(nodes.size());
        nodes.push_back(HNode{});
        HNode node;
        node.parent = parent;
        Box box, cbox;
        double area = 0;
        for (int i = first; i < first + count; ++i) {
            const HTri& t = tris[order[i]];
            box.grow(t.v0);
            box.grow(t.v1);
            box.grow(t.v2);
            cbox.grow((t.v0 + t.v1 + t.v2) / 3.0);
            area += t.area;
        }
        node.lo = box.lo;
        node.hi = box.hi;
        node.tri_area = area;
        if (count <= 4) {
            node.first = first;
            node.count = count;
            nodes[idx] = node;
            return idx;
        }
        V3 ext = cbox.extent();
        int axis = ext.x > ext.y ? (ext.x > ext.z ? 0 : 2) : (ext.y > ext.z ? 1 : 2);
        constexpr int kBins = 8;
        double lo = comp(cbox.lo, axis), width = comp(ext, axis);
        int mid;
        if (width < 1e-12) {
            mid = first + count / 2;
        } else {
            Box bbox[kBins];
            int bcount[kBins] = {0, 0, 0, 0, 0, 0, 0, 0};
            auto bin_of = [&](const HTri& t) {
                double c = ((comp(t.v0, axis) + comp(t.v1, axis) + comp(t.v2, axis)) / 3.0 - lo) /
                           width;
                return std::min(kBins - 1, int(c * kBins));
            };
            for (int i = first; i < first + count; ++i) {
                const HTri& t = tris[order[i]];
                int b = bin_of(t);
                bcount[b]++;
                bbox[b].grow(t.v0);
                bbox[b].grow(t.v1);
                bbox[b].grow(t.v2);
            }
            double best_cost = kInf;
            int best_split = -1;
            for (int s = 1; s < kBins; ++s) {
                Box lb, rb;
                int lc = 0, rc = 0;
                for (int i = 0; i < s; ++i) {
                    if (bcount[i]) lb.grow(bbox[i]);
                    lc += bcount[i];
                }
                for (int i = s; i < kBins; ++i) {
                    if (bcount[i]) rb.grow(bbox[i]);
                    rc += bcount[i];
                }
                if (lc == 0 || rc == 0) continue;
                double cost = lb.area() * lc + rb.area() * rc;
                if (cost < best_cost) {
                    best_cost = cost;
                    best_split = s;
                }
            }
            if (best_split < 0) {
                mid = first + count / 2;
            } else {
                auto it = std::stable_partition(order.begin() + first, order.begin() + first + count,
                                                [&](int id) { return bin_of(tris[id]) < best_split; });
                mid = int(it - order.begin());
                if (mid == first || mid == first + count) mid = first + count / 2;
            }
        }
        node.left = build(first, mid - first, idx);
        node.right = build(mid, first + count - mid, idx);
        nodes[idx] = node;
        return idx;
    }
};

int tree_depth(const std::vector<HNode>& nodes, int i) {
    if (nodes[i].count > 0) return 1;
    return 1 + std::max(tree_depth(nodes, nodes[i].left), tree_depth(nodes, nodes[i].right));
}

}  // namespace

std::vector<GMat> device_materials(const HScene& s) {
    std::vector<GMat> out;
    for (const HMaterial& m : s.materials) {
        GMat g;
        std::memset(&g, 0, sizeof(g));
        g.kind = m.kind;
        g.reconnectable = m.reconnectable() ? 1 : 0;
        g.albedo = m.albedo;
        g.roughness = m.roughness;
        g.alpha = std::max(1e-3, m.roughness * m.roughness);
        out.push_back(g);
    }
    return out;
}

HFrame build_frame(const HScene& def, double frame, bool build_bvh) {
    HFrame f;
    f.frame = frame;
    for (size_t i = 0; i < def.objects.size(); ++i) {
        const HObject& obj = def.objects[i];
        HPose pose = obj.track.pose_at(frame);
        M3 rot = quat_matrix(pose.q);
        bool moved = obj.track.animated();
        for (const HTri& t : obj.local) {
            HTri w = t;
            if (moved || norm(pose.t) > 0) {
                w.v0 = rot * t.v0 + pose.t;
                w.v1 = rot * t.v1 + pose.t;
                w.v2 = rot * t.v2 + pose.t;
                w.n = normalize(rot * t.n);
            }
            w.object = int(i);
            f.tris.push_back(w);
        }
        if (obj.track.moving_at(frame)) f.geo_motion = 1;
        // velocity_field (scene.hpp:318-335)
        GVel gv;
        std::memset(&gv, 0, sizeof(gv));
        if (obj.track.animated()) {
            double fmin = obj.track.keys.front().frame, fmax = obj.track.keys.back().frame;
            double lo = std::max(fmin, frame - 1.0), hi = std::min(fmax, frame + 1.0);
            if (hi <= lo) lo = hi = frame;
            if (hi > lo) {
                HPose pf = obj.track.pose_at(frame), pp = obj.track.pose_at(hi), pm = obj.track.pose_at(lo);
                double inv = 1.0 / ((hi - lo) * def.dt_frame);
                M3 rf_t = transpose(quat_matrix(pf.q));
                M3 dr = (quat_matrix(pp.q) - quat_matrix(pm.q)) * inv;
                gv.A = dr * rf_t;
                gv.c = (pp.t - pm.t) * inv - gv.A * pf.t;
                gv.moving = 1;
            }
        }
        f.obj_vel.push_back(gv);
    }
    if (f.tris.empty()) throw std::runtime_error("bvh: empty mesh");
    for (const HTri& t : f.tris)
        if (t.area <= 1e-12) throw std::runtime_error("bvh: degenerate triangle");
    if (build_bvh) {
        f.tri_order.resize(f.tris.size());
        for (size_t i = 0; i < f.tris.size(); ++i) f.tri_order[i] = int(i);
        f.nodes.reserve(f.tris.size() * 2);
        SahBuilder b{f.tris, f.tri_order, f.nodes};
        b.build(0, int(f.tris.size()), -1);
        f.diag = norm(f.nodes[0].hi - f.nodes[0].lo);
        f.leaf_of.assign(f.tris.size(), -1);
        for (size_t n = 0; n < f.nodes.size(); ++n)
            if (f.nodes[n].count > 0)
                for (int i = 0; i < f.nodes[n].count; ++i) f.leaf_of[f.tri_order[f.nodes[n].first + i]] = int(n);
        f.max_depth = tree_depth(f.nodes, 0);
    } else {
        // the tree is built on the device (bvh_build.cu); its root box is the
        // box of every vertex (min / max: the same bounds in any order)
        Box box;
        for (const HTri& t : f.tris) {
            box.grow(t.v0);
            box.grow(t.v1);
            box.grow(t.v2);
        }
        f.diag = norm(box.hi - box.lo);
    }
    f.eps_ray = 1e-4 * f.diag;

    // camera frame (scene.hpp:375-384)
    HCamPose pose = def.camera.pose_at(frame);
    std::memset(&f.cam, 0, sizeof(f.cam));
    f.cam.pos = pose.position;
    f.cam.fwd = pose.forward;
    f.cam.right = normalize(cross(pose.forward, pose.up));
    f.cam.up = cross(f.cam.right, pose.forward);
    f.cam.tan_half = std::tan(def.camera.fov_y / 2);
    f.cam.w = def.camera.width;
    f.cam.h = def.camera.height;
    if (def.camera.track.size() > 1) {  // central difference on the camera position track
        double lo = std::max(def.camera.track.front().first, frame - 1.0);
        double hi = std::min(def.camera.track.back().first, frame + 1.0);
        if (hi > lo) {
            V3 pp = def.camera.pose_at(hi).position, pm = def.camera.pose_at(lo).position;
            f.cam_vel = (pp - pm) / ((hi - lo) * def.dt_frame);
        }
    }

    std::memset(&f.light, 0, sizeof(f.light));
    f.light.pos = def.light.position;
    f.light.dir = def.light.direction;
    f.light.intensity = def.light.intensity;
    f.light.cone_half_angle = def.light.cone_half_angle;
    f.light.cos_cone = std::cos(def.light.cone_half_angle);
    f.light.regime = def.light.regime;

    std::memset(&f.lsub, 0, sizeof(f.lsub));
    f.lsub.tri = f.lsub.obj = f.lsub.mat = -1;
    if (def.light.regime == LIGHT_COLLIMATED) {
        if (!build_bvh) throw std::runtime_error("device BVH build: the collimated beam trace needs the host tree");
        // trace the beam through mirrors to its first non-delta hit
        PackedFrame pk = pack_frame(def, f, 0);
        FrameView v = rebase_view(pk, pk.blob.data());
        V3 o = def.light.position, d = def.light.direction;
        V3 power = def.light.intensity;
        double len = 0;
        for (int bounce = 0; bounce < 16; ++bounce) {
            Hit h;
            if (!intersect(v, o, d, h)) break;
            len += h.t;
            const HTri& tri = f.tris[h.tri];
            const HMaterial& m = def.materials[tri.material];
            if (m.kind == MAT_MIRROR) {
                V3 n = oriented_normal(tri.n, -d);
                power = power * m.albedo;
                V3 nd = reflect(-d, n);
                o = h.pos;
                d = nd;
                continue;
            }
            f.lsub.valid = 1;
            f.lsub.pos = h.pos;
            f.lsub.n = tri.n;
            f.lsub.tri = h.tri;
            f.lsub.obj = tri.object;
            f.lsub.mat = tri.material;
            f.lsub.wo_light = -d;
            f.lsub.power = power;
            f.lsub.chain_len = len;
            break;
        }
    }
    return f;
}

PackedFrame pack_frame(const HScene& s, const HFrame& f, int frame_id) {
    PackedFrame p;
    int nn = int(f.nodes.size()), nt = int(f.tris.size());
    std::vector<GNode> nodes(nn);
    std::vector<GNodeAux> aux(nn);
    // escape links reproduce the stack order: right child first, then left
    std::vector<int> esc(nn, -1);
    for (int i = 0; i < nn; ++i) {  // parents precede children in build order
        const HNode& h = f.nodes[i];
        if (h.count == 0) {
            esc[h.right] = h.left;
            esc[h.left] = esc[i];
        }
    }
    for (int i = 0; i < nn; ++i) {
        const HNode& h = f.nodes[i];
        GNode& g = nodes[i];
        g.lo[0] = h.lo.x;
        g.lo[1] = h.lo.y;
        g.lo[2] = h.lo.z;
        g.hi[0] = h.hi.x;
        g.hi[1] = h.hi.y;
        g.hi[2] = h.hi.z;
        g.first = h.first;
        g.count = h.count;
        g.miss_next = esc[i];
        g.hit_next = h.count > 0 ? esc[i] : h.right;
        GNodeAux& a = aux[i];
        std::memset(&a, 0, sizeof(a));
        a.tri_area = h.tri_area;
        a.left = h.left;
        a.right = h.right;
        a.parent = h.parent;
        a.first = h.first;
        a.count = h.count;
    }
    std::vector<GTriIsect> isect(nt);
    std::vector<int> tri_id(nt);
    for (int j = 0; j < nt; ++j) {
        const HTri& t = f.tris[f.tri_order[j]];
        isect[j].v0 = t.v0;
        isect[j].e1 = t.v1 - t.v0;
        isect[j].e2 = t.v2 - t.v0;
        tri_id[j] = f.tri_order[j];
    }
    std::vector<GTriInfo> info(nt);
    for (int i = 0; i < nt; ++i) {
        std::memset(&info[i], 0, sizeof(GTriInfo));
        info[i].n = f.tris[i].n;
        info[i].mat = f.tris[i].material;
        info[i].obj = f.tris[i].object;
        info[i].area = f.tris[i].area;
        info[i].leaf = f.leaf_of[i];
    }
    for (int j = 0; j < nt; ++j) info[f.tri_order[j]].leaf_slot = j;
    std::vector<Frame2> tframe(nt);
    for (int i = 0; i < nt; ++i) {
        const HTri& t = f.tris[i];
        tframe[i] = tangent_frame_of(t.n, t.v1 - t.v0, t.v2 - t.v0);
    }
    std::vector<GMat> mats = device_materials(s);

    auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t off = 0;
    p.off_nodes = off;
    off = align(off + nn * sizeof(GNode));
    p.off_aux = off;
    off = align(off + nn * sizeof(GNodeAux));
    p.off_isect = off;
    off = align(off + nt * sizeof(GTriIsect));
    p.off_tri_id = off;
    off = align(off + nt * sizeof(int));
    p.off_tri = off;
    off = align(off + nt * sizeof(GTriInfo));
    p.off_mats = off;
    off = align(off + mats.size() * sizeof(GMat));
    p.off_vel = off;
    off = align(off + f.obj_vel.size() * sizeof(GVel));
    p.off_tframe = off;
    off = align(off + nt * sizeof(Frame2));
    p.blob.assign(off, 0);
    std::memcpy(p.blob.data() + p.off_tframe, tframe.data(), nt * sizeof(Frame2));
    std::memcpy(p.blob.data() + p.off_nodes, nodes.data(), nn * sizeof(GNode));
    std::memcpy(p.blob.data() + p.off_aux, aux.data(), nn * sizeof(GNodeAux));
    std::memcpy(p.blob.data() + p.off_isect, isect.data(), nt * sizeof(GTriIsect));
    std::memcpy(p.blob.data() + p.off_tri_id, tri_id.data(), nt * sizeof(int));
    std::memcpy(p.blob.data() + p.off_tri, info.data(), nt * sizeof(GTriInfo));
    std::memcpy(p.blob.data() + p.off_mats, mats.data(), mats.size() * sizeof(GMat));
    if (!f.obj_vel.empty()) std::memcpy(p.blob.data() + p.off_vel, f.obj_vel.data(), f.obj_vel.size() * sizeof(GVel));

    FrameView& v = p.view;
    std::memset(&v, 0, sizeof(v));
    v.n_nodes = nn;
    v.n_tris = nt;
    v.n_mats = int(mats.size());
    v.geo_motion = f.geo_motion;
    v.cam = f.cam;
    v.light = f.light;
    v.lsub = f.lsub;
    v.eps_ray = f.eps_ray;
    v.diag = f.diag;
    v.frame_id = frame_id;
    v.n_obj = int(f.obj_vel.size());
    v.cam_vel = f.cam_vel;
    return p;
}

PackedFrame pack_frame_shell(const HScene& s, const HFrame& f, int nn, int frame_id) {
    // the layout of pack_frame for nn nodes; only the materials and velocity
    // fields are filled (the device writes the tree and triangle arrays)
    PackedFrame p;
    const int nt = int(f.tris.size());
    std::vector<GMat> mats = device_materials(s);
    auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t off = 0;
    p.off_nodes = off;
    off = align(off + nn * sizeof(GNode));
    p.off_aux = off;
    off = align(off + nn * sizeof(GNodeAux));
    p.off_isect = off;
    off = align(off + nt * sizeof(GTriIsect));
    p.off_tri_id = off;
    off = align(off + nt * sizeof(int));
    p.off_tri = off;
    off = align(off + nt * sizeof(GTriInfo));
    p.off_mats = off;
    off = align(off + mats.size() * sizeof(GMat));
    p.off_vel = off;
    off = align(off + f.obj_vel.size() * sizeof(GVel));
    p.off_tframe = off;
    off = align(off + nt * sizeof(Frame2));
    p.blob.assign(off, 0);
    std::memcpy(p.blob.data() + p.off_mats, mats.data(), mats.size() * sizeof(GMat));
    if (!f.obj_vel.empty()) std::memcpy(p.blob.data() + p.off_vel, f.obj_vel.data(), f.obj_vel.size() * sizeof(GVel));
    FrameView& v = p.view;
    std::memset(&v, 0, sizeof(v));
    v.n_nodes = nn;
    v.n_tris = nt;
    v.n_mats = int(mats.size());
    v.geo_motion = f.geo_motion;
    v.cam = f.cam;
    v.light = f.light;
    v.lsub = f.lsub;
    v.eps_ray = f.eps_ray;
    v.diag = f.diag;
    v.frame_id = frame_id;
    v.n_obj = int(f.obj_vel.size());
    v.cam_vel = f.cam_vel;
    return p;
}

FrameView rebase_view(const PackedFrame& p, const unsigned char* base) {
    FrameView v = p.view;
    v.nodes = reinterpret_cast<const GNode*>(base + p.off_nodes);
    v.aux = reinterpret_cast<const GNodeAux*>(base + p.off_aux);
    v.tri_isect = reinterpret_cast<const GTriIsect*>(base + p.off_isect);
    v.tri_id = reinterpret_cast<const int*>(base + p.off_tri_id);
    v.tri = reinterpret_cast<const GTriInfo*>(base + p.off_tri);
    v.mats = reinterpret_cast<const GMat*>(base + p.off_mats);
    v.vel = reinterpret_cast<const GVel*>(base + p.off_vel);
    v.tframe = reinterpret_cast<const Frame2*>(base + p.off_tframe);
    return v;
}

}  // namespace tofr_b200
