// Parameter persistence (SPEC.md:466-469 Snapshot, :489-496 save/load, :529 file format):
// `<dir>/<name>.ddt` = "DDSL" | u32 version = 1 | u32 rank | u32 dims[rank] | f32 payload, little
// endian, reference (NCHW / (out, in)) layout.  Velocities ride along as `<name>.velocity.ddt` so
// a resumed momentum-SGD run continues bit-exactly.  Built on the public runtime ABI only.
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "status.hpp"
#include "tc_runtime.h"

namespace {

constexpr char kMagic[4] = {'D', 'D', 'S', 'L'};
constexpr uint32_t kVersion = 1;

std::string join(const char* dir, const std::string& name) {
    std::string d(dir);
    if (!d.empty() && d.back() != '/') d += '/';
    return d + name;
}

int64_t count_of(const tc_param_desc& pd) {
    int64_t n = 1;
    for (int j = 0; j < pd.rank; ++j) n *= pd.dims[j];
    return n;
}

tc_status write_ddt(const std::string& path, const tc_param_desc& pd, const std::vector<float>& data) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) return tcb::fail(TC_IO_ERROR, "snapshot: cannot write " + path + ": " + std::strerror(errno));
    bool ok = std::fwrite(kMagic, 1, 4, f) == 4;
    const uint32_t hdr[2] = {kVersion, static_cast<uint32_t>(pd.rank)};
    ok = ok && std::fwrite(hdr, 4, 2, f) == 2;
    for (int j = 0; j < pd.rank; ++j) {
        const uint32_t d = static_cast<uint32_t>(pd.dims[j]);
        ok = ok && std::fwrite(&d, 4, 1, f) == 1;
    }
    ok = ok && std::fwrite(data.data(), 4, data.size(), f) == data.size();
    ok = (std::fclose(f) == 0) && ok;
    return ok ? TC_OK : tcb::fail(TC_IO_ERROR, "snapshot: write failed: " + path);
}

// 1 = loaded, 0 = file absent, else an error status (negated)
int read_ddt(const std::string& path, const tc_param_desc& pd, std::vector<float>& data, tc_status* err) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) {
        if (errno == ENOENT) return 0;
        *err = tcb::fail(TC_IO_ERROR, "snapshot: cannot read " + path + ": " + std::strerror(errno));
        return -1;
    }
    char magic[4];
    uint32_t hdr[2] = {0, 0};
    bool ok = std::fread(magic, 1, 4, f) == 4 && std::memcmp(magic, kMagic, 4) == 0;
    if (!ok) {
        std::fclose(f);
        *err = tcb::fail(TC_FORMAT_ERROR, "snapshot: bad magic in " + path + " (expected DDSL)");
        return -1;
    }
    ok = std::fread(hdr, 4, 2, f) == 2 && hdr[0] == kVersion && hdr[1] == static_cast<uint32_t>(pd.rank);
    for (int j = 0; ok && j < pd.rank; ++j) {
        uint32_t d = 0;
        ok = std::fread(&d, 4, 1, f) == 1 && d == static_cast<uint32_t>(pd.dims[j]);
    }
    if (!ok) {
        std::fclose(f);
        *err = tcb::fail(TC_FORMAT_ERROR, "snapshot: version / rank / dims of " + path + " do not match parameter " + pd.name);
        return -1;
    }
    data.resize(static_cast<size_t>(count_of(pd)));
    ok = std::fread(data.data(), 4, data.size(), f) == data.size();
    char extra;
    ok = ok && std::fread(&extra, 1, 1, f) == 0;
    std::fclose(f);
    if (!ok) {
        *err = tcb::fail(TC_FORMAT_ERROR, "snapshot: payload size of " + path + " does not match its dims");
        return -1;
    }
    return 1;
}

}  // namespace

extern "C" {

tc_status tc_snapshot_save(tc_ctx* ctx, const char* dir) {
    const tc_plan* p = tc_ctx_plan(ctx);
    if (!p || !dir) return tcb::fail(TC_INVALID_ARG, "tc_snapshot_save: null argument");
    if (::mkdir(dir, 0755) != 0 && errno != EEXIST) return tcb::fail(TC_IO_ERROR, std::string("snapshot: cannot create ") + dir);
    for (int i = 0; i < p->nparams; ++i) {
        const tc_param_desc& pd = p->params[i];
        std::vector<float> buf(static_cast<size_t>(count_of(pd)));
        tc_status r = tc_param_download(ctx, i, buf.data());
        if (r == TC_OK) r = write_ddt(join(dir, std::string(pd.name) + ".ddt"), pd, buf);
        if (r == TC_OK) r = tc_velocity_download(ctx, i, buf.data());
        if (r == TC_OK) r = write_ddt(join(dir, std::string(pd.name) + ".velocity.ddt"), pd, buf);
        if (r != TC_OK) return r;
    }
    return TC_OK;
}

tc_status tc_snapshot_load(tc_ctx* ctx, const char* dir, int* loaded, int* missing) {
    const tc_plan* p = tc_ctx_plan(ctx);
    if (!p || !dir) return tcb::fail(TC_INVALID_ARG, "tc_snapshot_load: null argument");
    int nl = 0, nm = 0;
    for (int i = 0; i < p->nparams; ++i) {
        const tc_param_desc& pd = p->params[i];
        std::vector<float> buf;
        tc_status err = TC_OK;
        const std::string path = join(dir, std::string(pd.name) + ".ddt");
        const int got = read_ddt(path, pd, buf, &err);
        if (got < 0) return err;
        if (got == 0) {  // fine-tune semantics: keep the initialised value
            std::fprintf(stderr, "tc_snapshot_load: warning: %s missing, %s keeps its current value\n", path.c_str(), pd.name);
            ++nm;
            continue;
        }
        tc_status r = tc_param_upload(ctx, i, buf.data());
        if (r != TC_OK) return r;
        const int gv = read_ddt(join(dir, std::string(pd.name) + ".velocity.ddt"), pd, buf, &err);
        if (gv < 0) return err;
        if (gv > 0 && (r = tc_velocity_upload(ctx, i, buf.data())) != TC_OK) return r;
        ++nl;
    }
    if (loaded) *loaded = nl;
    if (missing) *missing = nm;
    return TC_OK;
}

}  // extern "C"
