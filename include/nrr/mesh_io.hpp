// Mesh / point-cloud files for the pipeline and the CLI (reference
// mesh_io.hpp:105-351): OBJ (`v` / `f` records, polygons fanned into
// triangles, `i/j/k` slashes ignored) and PLY (ascii or binary little-endian;
// any vertex element with x/y/z, a face element with a `vertex_indices` or
// `vertex_index` list). Vertex order is preserved; meshes take their edges
// from the faces, point clouds symmetric kNN connectivity (make_surface).
// Writers emit full double precision (%.17g); an optional per-vertex scalar
// becomes the PLY `quality` property or OBJ vertex colours on a blue-to-red
// ramp normalised by the scalar maximum. Errors are IoError with
// "path:line: what" where a line is known, as the reference reports them.
#pragma once

#include <algorithm>
#include <array>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "nrr/common.hpp"
#include "nrr/surface.hpp"

namespace nrr {

namespace io_detail {

inline std::string extension_of(const std::string& path) {
    const size_t dot = path.rfind('.');
    std::string ext = dot == std::string::npos ? std::string() : path.substr(dot + 1);
    std::transform(ext.begin(), ext.end(), ext.begin(), [](unsigned char ch) { return static_cast<char>(std::tolower(ch)); });
    return ext;
}

[[noreturn]] inline void fail(const std::string& path, size_t line, const std::string& what) {
    throw IoError(path + ":" + std::to_string(line) + ": " + what);
}

inline bool blank_or_comment(const std::string& line) {
    const size_t k = line.find_first_not_of(" \t\r");
    return k == std::string::npos || line[k] == '#';
}

inline std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

/// blue (0) -> cyan -> green -> yellow -> red (1): each channel is a clamped
/// tent 1.5 - |4t - c| centred at c = 3 (red), 2 (green), 1 (blue)
inline Vec3 error_ramp(double t) {
    t = std::min(1.0, std::max(0.0, t));
    auto tent = [t](double c) { return std::min(1.0, std::max(0.0, 1.5 - std::abs(4.0 * t - c))); };
    return {tent(3.0), tent(2.0), tent(1.0)};
}

// PLY scalar types by name -> (bytes, decoder)
enum class PlyType { i8, u8, i16, u16, i32, u32, f32, f64, bad };
inline PlyType ply_type(const std::string& t) {
    if (t == "char" || t == "int8") return PlyType::i8;
    if (t == "uchar" || t == "uint8") return PlyType::u8;
    if (t == "short" || t == "int16") return PlyType::i16;
    if (t == "ushort" || t == "uint16") return PlyType::u16;
    if (t == "int" || t == "int32") return PlyType::i32;
    if (t == "uint" || t == "uint32") return PlyType::u32;
    if (t == "float" || t == "float32") return PlyType::f32;
    if (t == "double" || t == "float64") return PlyType::f64;
    return PlyType::bad;
}
inline int ply_bytes(PlyType t) {
    switch (t) {
        case PlyType::i8:
        case PlyType::u8:
            return 1;
        case PlyType::i16:
        case PlyType::u16:
            return 2;
        case PlyType::i32:
        case PlyType::u32:
        case PlyType::f32:
            return 4;
        case PlyType::f64:
            return 8;
        default:
            return 0;
    }
}
template <typename T>
inline double decode_as(const unsigned char* b) {
    T v;
    std::memcpy(&v, b, sizeof(T));
    return static_cast<double>(v);
}
inline double decode(PlyType t, const unsigned char* b) {
    switch (t) {
        case PlyType::i8:
            return decode_as<int8_t>(b);
        case PlyType::u8:
            return decode_as<uint8_t>(b);
        case PlyType::i16:
            return decode_as<int16_t>(b);
        case PlyType::u16:
            return decode_as<uint16_t>(b);
        case PlyType::i32:
            return decode_as<int32_t>(b);
        case PlyType::u32:
            return decode_as<uint32_t>(b);
        case PlyType::f32:
            return decode_as<float>(b);
        default:
            return decode_as<double>(b);
    }
}

struct PlyProp {
    std::string name, type_name, count_type_name;
    bool list = false;
};
struct PlyElem {
    std::string name;
    size_t count = 0;
    std::vector<PlyProp> props;
};

// one value source for a PLY body: whitespace tokens of the current line
// (ascii) or little-endian bytes (binary)
class PlyBody {
public:
    PlyBody(std::istream& in, bool binary, const std::string& path, size_t lineno)
        : in_(in), binary_(binary), path_(path), lineno_(lineno) {}
    void next_record() {
        if (binary_) return;
        std::string line;
        ++lineno_;
        if (!std::getline(in_, line)) fail(path_, lineno_, "unexpected end of file");
        tokens_.clear();
        tokens_.str(line);
    }
    double value(const std::string& type_name, const char* what) {
        const PlyType t = ply_type(type_name);
        if (binary_) {
            const int nb = ply_bytes(t);
            if (nb == 0) throw IoError(path_ + ": unsupported property type '" + type_name + "'");
            unsigned char buf[8];
            if (!in_.read(reinterpret_cast<char*>(buf), nb))
                throw IoError(path_ + ": unexpected end of binary payload at offset " +
                              std::to_string(static_cast<long long>(in_.tellg())));
            return decode(t, buf);
        }
        double v;
        if (!(tokens_ >> v)) fail(path_, lineno_, what);
        return v;
    }

private:
    std::istream& in_;
    bool binary_;
    const std::string& path_;
    size_t lineno_;
    std::istringstream tokens_;
};

inline void fan(const std::vector<int>& poly, std::vector<std::array<int, 3>>& faces) {
    for (size_t t = 1; t + 1 < poly.size(); ++t) faces.push_back({poly[0], poly[t], poly[t + 1]});
}

inline void read_obj(const std::string& path, std::vector<Vec3>& points, std::vector<std::array<int, 3>>& faces) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open '" + path + "'");
    std::string line;
    for (size_t lineno = 1; std::getline(in, line); ++lineno) {
        std::istringstream ls(line);
        std::string tag;
        if (!(ls >> tag) || tag[0] == '#') continue;
        if (tag == "v") {
            double x, y, z;
            if (!(ls >> x >> y >> z)) fail(path, lineno, "malformed vertex record");
            points.emplace_back(x, y, z);
        } else if (tag == "f") {
            std::vector<int> poly;
            for (std::string tok; ls >> tok;) {
                int v = 0;
                try {
                    v = std::stoi(tok.substr(0, tok.find('/')));
                } catch (const std::exception&) {
                    fail(path, lineno, "malformed face index '" + tok + "'");
                }
                if (v < 1 || v > static_cast<int>(points.size())) fail(path, lineno, "face index out of range");
                poly.push_back(v - 1);
            }
            if (poly.size() < 3) fail(path, lineno, "face needs at least 3 vertices");
            fan(poly, faces);
        }
    }
}

inline void read_ply(const std::string& path, std::vector<Vec3>& points, std::vector<std::array<int, 3>>& faces) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "'");
    std::string line;
    size_t lineno = 1;
    if (!std::getline(in, line) || line.compare(0, 3, "ply") != 0) fail(path, 1, "not a PLY file");
    bool binary = false;
    std::vector<PlyElem> elems;
    for (bool done = false; !done;) {
        if (!std::getline(in, line)) break;
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::istringstream ls(line);
        std::string tag;
        ls >> tag;
        if (tag.empty() || tag == "comment" || tag == "obj_info") continue;
        if (tag == "end_header") {
            done = true;
        } else if (tag == "format") {
            std::string f;
            ls >> f;
            if (f == "ascii") binary = false;
            else if (f == "binary_little_endian") binary = true;
            else fail(path, lineno, "unsupported PLY format '" + f + "'");
        } else if (tag == "element") {
            PlyElem e;
            if (!(ls >> e.name >> e.count)) fail(path, lineno, "malformed element record");
            elems.push_back(std::move(e));
        } else if (tag == "property") {
            if (elems.empty()) fail(path, lineno, "property before any element");
            PlyProp p;
            std::string t;
            ls >> t;
            if (t == "list") {
                p.list = true;
                if (!(ls >> p.count_type_name >> p.type_name >> p.name)) fail(path, lineno, "malformed list property");
            } else {
                p.type_name = t;
                if (!(ls >> p.name)) fail(path, lineno, "malformed property record");
            }
            elems.back().props.push_back(std::move(p));
        } else {
            fail(path, lineno, "unexpected header record '" + tag + "'");
        }
    }
    PlyBody body(in, binary, path, lineno);
    for (const PlyElem& e : elems) {
        int slot[3] = {-1, -1, -1}, index_list = -1;
        for (size_t p = 0; p < e.props.size(); ++p) {
            const auto& pr = e.props[p];
            for (int c = 0; c < 3; ++c)
                if (pr.name == std::string(1, static_cast<char>('x' + c))) slot[c] = static_cast<int>(p);
            if (pr.list && (pr.name == "vertex_indices" || pr.name == "vertex_index")) index_list = static_cast<int>(p);
        }
        const bool vertex = e.name == "vertex", face = e.name == "face";
        if (vertex && (slot[0] < 0 || slot[1] < 0 || slot[2] < 0))
            throw IoError(path + ": vertex element lacks x/y/z properties");
        if (face && index_list < 0) throw IoError(path + ": face element lacks a vertex index list");
        std::vector<double> val(e.props.size());
        std::vector<int> poly;
        for (size_t r = 0; r < e.count; ++r) {
            body.next_record();
            poly.clear();
            for (size_t p = 0; p < e.props.size(); ++p) {
                const auto& pr = e.props[p];
                if (!pr.list) {
                    val[p] = body.value(pr.type_name, "malformed property value");
                    continue;
                }
                const int cnt = static_cast<int>(body.value(pr.count_type_name, "malformed list count"));
                for (int k = 0; k < cnt; ++k) {
                    const double v = body.value(pr.type_name, "malformed list entry");
                    if (static_cast<int>(p) == index_list) poly.push_back(static_cast<int>(v));
                }
            }
            if (vertex) points.emplace_back(val[slot[0]], val[slot[1]], val[slot[2]]);
            if (face) {
                if (poly.size() < 3) throw IoError(path + ": face with fewer than 3 vertices");
                for (int v : poly)
                    if (v < 0 || v >= static_cast<int>(points.size())) throw IoError(path + ": face index out of range");
                fan(poly, faces);
            }
        }
    }
}

}  // namespace io_detail

/// mesh_io.hpp:105-264
inline Surface load_surface(const std::string& path, int knn_k = 6) {
    const std::string ext = io_detail::extension_of(path);
    std::vector<Vec3> points;
    std::vector<std::array<int, 3>> faces;
    if (ext == "obj") io_detail::read_obj(path, points, faces);
    else if (ext == "ply") io_detail::read_ply(path, points, faces);
    else throw IoError("unsupported mesh format '." + ext + "' (expected .obj or .ply)");
    if (points.empty()) throw IoError(path + ": no vertices found");
    return make_surface(std::move(points), std::move(faces), knn_k);
}

struct SaveOptions {
    bool binary_ply = false;
};

/// mesh_io.hpp:270-349
inline void save_surface(const Surface& surface, const std::string& path,
                         const std::vector<double>& per_vertex_scalar = {}, const SaveOptions& opts = {}) {
    const bool channel = !per_vertex_scalar.empty();
    if (channel && per_vertex_scalar.size() != surface.points.size())
        throw ConfigError("save_surface: scalar channel length mismatch");
    const std::string ext = io_detail::extension_of(path);
    if (ext != "obj" && ext != "ply")
        throw IoError("unsupported mesh format '." + ext + "' (expected .obj or .ply)");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    using io_detail::g17;
    if (ext == "obj") {
        double top = 0.0;
        for (double v : per_vertex_scalar) top = std::max(top, v);
        for (size_t i = 0; i < surface.points.size(); ++i) {
            const Vec3& p = surface.points[i];
            out << "v " << g17(p.x()) << ' ' << g17(p.y()) << ' ' << g17(p.z());
            if (channel) {
                const Vec3 rgb = io_detail::error_ramp(top > 0.0 ? per_vertex_scalar[i] / top : 0.0);
                out << ' ' << g17(rgb.x()) << ' ' << g17(rgb.y()) << ' ' << g17(rgb.z());
            }
            out << '\n';
        }
        for (const auto& f : surface.faces) out << "f " << f[0] + 1 << ' ' << f[1] + 1 << ' ' << f[2] + 1 << '\n';
    } else {
        out << "ply\nformat " << (opts.binary_ply ? "binary_little_endian" : "ascii") << " 1.0\n"
            << "element vertex " << surface.points.size() << "\n"
            << "property double x\nproperty double y\nproperty double z\n";
        if (channel) out << "property double quality\n";
        out << "element face " << surface.faces.size() << "\n"
            << "property list uchar int vertex_indices\nend_header\n";
        if (opts.binary_ply) {
            std::vector<double> rec;
            for (size_t i = 0; i < surface.points.size(); ++i) {
                rec.assign({surface.points[i].x(), surface.points[i].y(), surface.points[i].z()});
                if (channel) rec.push_back(per_vertex_scalar[i]);
                out.write(reinterpret_cast<const char*>(rec.data()), static_cast<std::streamsize>(8 * rec.size()));
            }
            for (const auto& f : surface.faces) {
                unsigned char frec[13];
                frec[0] = 3;
                for (int c = 0; c < 3; ++c) {
                    const int32_t v = f[c];
                    std::memcpy(frec + 1 + 4 * c, &v, 4);
                }
                out.write(reinterpret_cast<const char*>(frec), 13);
            }
        } else {
            for (size_t i = 0; i < surface.points.size(); ++i) {
                const Vec3& p = surface.points[i];
                out << g17(p.x()) << ' ' << g17(p.y()) << ' ' << g17(p.z());
                if (channel) out << ' ' << g17(per_vertex_scalar[i]);
                out << '\n';
            }
            for (const auto& f : surface.faces) out << "3 " << f[0] << ' ' << f[1] << ' ' << f[2] << '\n';
        }
    }
    if (!out) throw IoError("write to '" + path + "' failed");
}

}  // namespace nrr
