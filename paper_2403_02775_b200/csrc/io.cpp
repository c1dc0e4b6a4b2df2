// ezquant/io.hpp for the B200 engine (reference io.cpp:108-390): manifests
// (nlohmann ordered_json, the reference's formatting), raw f32 tensor files,
// and the .ezqt container over the C-ABI codec (codec.cpp).
//
// Derived from the reference's io.cpp: save_manifest, read_tensor_f32,
// write_tensor_f32, write_quantized / read_quantized and tensor_file_stem
// follow it closely on purpose -- their JSON key order, formatting and
// exception texts are the byte-identical-output contract that
// tests/test_model_driver.py enforces against the compiled reference. Off the
// hot path; the codec itself (codec.cpp) is an independent C implementation.
#include <bit>
#include <cstring>
#include <fstream>
#include <set>
#include <string>

#include <json.hpp>

#include "../../include/ezquant/io.hpp"
#include "../../include/ezquant_c.h"

namespace ezquant {

namespace {

using ordered_json = nlohmann::ordered_json;

// C-ABI status -> the reference's exception (io errors keep their offset).
[[noreturn]] void raise_status(int code) {
    char msg[1024];
    int64_t idx = -1;
    ezq_last_error(msg, sizeof msg, &idx);
    const uint64_t off = idx >= 0 ? static_cast<uint64_t>(idx) : 0;
    switch (code) {
        case EZQ_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case EZQ_ERR_IO_FAILURE: throw io_error(IoErrorKind::IoFailure, off, msg);
        case EZQ_ERR_IO_FORMAT: throw io_error(IoErrorKind::FormatViolation, off, msg);
        case EZQ_ERR_IO_VERSION: throw io_error(IoErrorKind::VersionMismatch, off, msg);
        default: throw std::runtime_error(msg);
    }
}

[[noreturn]] void bad_manifest(const std::string& msg) {
    throw io_error(IoErrorKind::FormatViolation, 0, "manifest: " + msg);
}

// Typed accessors over one manifest entry; every failure is a
// FormatViolation naming the entry (`ctx`) and the key.
struct Entry {
    const ordered_json& j;
    std::string ctx;
    bool has(const char* key) const { return j.contains(key); }
    std::string text(const char* key) const {
        if (!has(key) || !j[key].is_string()) bad_manifest(ctx + " needs string field '" + key + "'");
        return j[key].get<std::string>();
    }
    int64_t count(const char* key) const {
        if (!has(key) || !j[key].is_number_integer()) bad_manifest(ctx + " needs integer field '" + key + "'");
        const int64_t v = j[key].get<int64_t>();
        if (v <= 0) bad_manifest(ctx + " field '" + key + "' must be positive");
        return v;
    }
};

ordered_json parse_json_file(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw io_error(IoErrorKind::IoFailure, 0, "cannot open " + path.string());
    try {
        return ordered_json::parse(in);
    } catch (const nlohmann::json::exception& e) {
        bad_manifest(std::string("invalid JSON: ") + e.what());
    }
}

void write_text(const std::filesystem::path& path, const std::string& text) {
    std::ofstream out(path);
    if (!out) throw io_error(IoErrorKind::IoFailure, 0, "cannot open " + path.string());
    out << text;
    out.flush();
    if (!out) throw io_error(IoErrorKind::IoFailure, 0, "short write to " + path.string());
}

ManifestTensor parse_tensor(const ordered_json& t) {
    if (!t.is_object()) bad_manifest("tensor entries must be objects");
    ManifestTensor mt;
    mt.name = Entry{t, "tensor"}.text("name");
    const Entry e{t, "tensor '" + mt.name + "'"};
    mt.rows = e.count("rows");
    mt.cols = e.count("cols");
    mt.dtype = e.text("dtype");
    if (mt.dtype != "f32") bad_manifest(e.ctx + " has dtype '" + mt.dtype + "', only f32 in v1");
    mt.file = e.text("file");
    if (e.has("role")) {
        if (!t["role"].is_string()) bad_manifest(e.ctx + " field 'role' must be a string");
        mt.role = t["role"].get<std::string>();
    }
    if (e.has("layer")) {
        if (!t["layer"].is_number_integer()) bad_manifest(e.ctx + " field 'layer' must be an integer");
        mt.layer = t["layer"].get<int64_t>();
    }
    return mt;
}

}  // namespace

// ---- model manifest (io.cpp:108-178) ------------------------------------
ModelManifest load_manifest(const std::filesystem::path& path) {
    const ordered_json j = parse_json_file(path);
    if (!j.is_object()) bad_manifest("top level must be an object");
    const auto ver = j.find("version");
    if (ver == j.end() || !ver->is_number_integer()) bad_manifest("missing integer 'version'");
    ModelManifest m;
    m.version = ver->get<int>();
    if (m.version != 1)
        throw io_error(IoErrorKind::VersionMismatch, 0,
                       "manifest version " + std::to_string(m.version) + ", expected 1");
    const auto list = j.find("tensors");
    if (list == j.end() || !list->is_array()) bad_manifest("missing 'tensors' array");
    m.base_dir = path.parent_path();
    std::set<std::string> seen;
    for (const auto& t : *list) {
        ManifestTensor mt = parse_tensor(t);
        if (!seen.insert(mt.name).second) bad_manifest("duplicate tensor name '" + mt.name + "'");
        m.tensors.push_back(std::move(mt));
    }
    return m;
}

void save_manifest(const ModelManifest& m, const std::filesystem::path& path) {
    ordered_json j;
    j["version"] = m.version;
    j["tensors"] = ordered_json::array();
    for (const auto& t : m.tensors) {
        ordered_json e;
        e["name"] = t.name;
        e["rows"] = t.rows;
        e["cols"] = t.cols;
        e["dtype"] = t.dtype;
        e["file"] = t.file;
        if (!t.role.empty()) e["role"] = t.role;
        if (t.layer) e["layer"] = *t.layer;
        j["tensors"].push_back(std::move(e));
    }
    write_text(path, j.dump(2) + "\n");
}

// ---- raw tensors (io.cpp:182-217); little-endian hosts only -------------
static_assert(std::endian::native == std::endian::little, "B200 hosts are little-endian");

DenseMatrix read_tensor_f32(const std::filesystem::path& path, int64_t rows, int64_t cols) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error(IoErrorKind::IoFailure, 0, "cannot open " + path.string());
    const size_t count = static_cast<size_t>(rows) * static_cast<size_t>(cols);
    DenseMatrix m(rows, cols);
    in.read(reinterpret_cast<char*>(m.data.data()), static_cast<std::streamsize>(count * sizeof(float)));
    if (static_cast<size_t>(in.gcount()) != count * sizeof(float))
        throw io_error(IoErrorKind::FormatViolation, static_cast<uint64_t>(in.gcount()),
                       path.string() + ": raw tensor shorter than rows*cols*4");
    in.peek();
    if (!in.eof())
        throw io_error(IoErrorKind::FormatViolation, count * sizeof(float),
                       path.string() + ": trailing bytes after rows*cols*4");
    return m;
}

void write_tensor_f32(const DenseMatrix& m, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw io_error(IoErrorKind::IoFailure, 0, "cannot open " + path.string());
    out.write(reinterpret_cast<const char*>(m.data.data()),
              static_cast<std::streamsize>(m.data.size() * sizeof(float)));
    out.flush();
    if (!out) throw io_error(IoErrorKind::IoFailure, 0, "short write to " + path.string());
}

// ---- .ezqt container ------------------------------------------------------
std::vector<uint8_t> encode_quantized(const QuantizedWeight& q) {
    std::vector<ezq_outlier> e(q.outliers.entries.size());
    for (size_t i = 0; i < e.size(); ++i)
        e[i] = {q.outliers.entries[i].row, q.outliers.entries[i].col, q.outliers.entries[i].value};
    ezq_qweight* w = nullptr;
    if (int s = ezq_qweight_wrap(q.rows, q.cols, q.bits, q.packed_levels.data(),
                                 static_cast<int64_t>(q.packed_levels.size()), q.scales.scales.data(),
                                 q.scales.size(), e.data(), static_cast<int64_t>(e.size()), q.outliers.mean,
                                 q.outliers.stddev, q.outliers.sigma_n, EZQ_MEM_HOST, &w))
        raise_status(s);
    uint8_t* buf = nullptr;
    int64_t len = 0;
    const int s = ezq_encode_quantized(w, &buf, &len);
    ezq_qweight_free(w);
    if (s != EZQ_OK) raise_status(s);
    std::vector<uint8_t> out(buf, buf + len);
    ezq_free(buf);
    return out;
}

QuantizedWeight decode_quantized(std::span<const uint8_t> bytes) {
    ezq_qweight* q = nullptr;
    if (int s = ezq_decode_quantized(bytes.data(), static_cast<int64_t>(bytes.size()), &q)) raise_status(s);
    QuantizedWeight w;
    w.rows = q->rows;
    w.cols = q->cols;
    w.bits = q->bits;
    w.packed_levels.assign(q->packed, q->packed + q->packed_bytes);
    w.scales.scales.assign(q->scales, q->scales + q->cols);
    w.outliers.entries.resize(static_cast<size_t>(q->n_outliers));
    for (int64_t i = 0; i < q->n_outliers; ++i)
        w.outliers.entries[i] = {q->outliers[i].row, q->outliers[i].col, q->outliers[i].value};
    w.outliers.mean = q->mean;
    w.outliers.stddev = q->stddev;
    w.outliers.sigma_n = q->sigma_n;
    ezq_qweight_free(q);
    return w;
}

void write_quantized(const QuantizedWeight& q, const std::filesystem::path& path) {
    const std::vector<uint8_t> bytes = encode_quantized(q);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw io_error(IoErrorKind::IoFailure, 0, "cannot open " + path.string());
    out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    out.flush();
    if (!out) throw io_error(IoErrorKind::IoFailure, 0, "short write to " + path.string());
}

QuantizedWeight read_quantized(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary | std::ios::ate);
    if (!in) throw io_error(IoErrorKind::IoFailure, 0, "cannot open " + path.string());
    const std::streamsize size = in.tellg();
    in.seekg(0);
    std::vector<uint8_t> bytes(static_cast<size_t>(size));
    in.read(reinterpret_cast<char*>(bytes.data()), size);
    if (in.gcount() != size)
        throw io_error(IoErrorKind::IoFailure, static_cast<uint64_t>(in.gcount()),
                       "read failed on " + path.string());
    try {
        return decode_quantized(bytes);
    } catch (const io_error& e) {
        throw io_error(e.kind(), e.offset(), path.string() + ": " + e.what());
    }
}

std::string tensor_file_stem(const std::string& name) {
    std::string out = name;
    for (char& ch : out) {
        const bool keep = (ch >= 'a' && ch <= 'z') || (ch >= 'A' && ch <= 'Z') || (ch >= '0' && ch <= '9') ||
                          ch == '.' || ch == '_' || ch == '-';
        if (!keep) ch = '_';
    }
    return out.empty() ? std::string("_") : out;
}

}  // namespace ezquant
