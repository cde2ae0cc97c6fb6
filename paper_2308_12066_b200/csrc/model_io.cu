// model_io.cu — PGMOE1 weight files (model_io.py:1-105) into / out of a model.
//
// Layout (little-endian): magic "PGMOE1", then d_model, d_ff, num_blocks,
// num_experts, top_k, activation_level as int32, then fp32 row-major
// matrices in block order: conventional gate (if wired), lookahead gate (if
// wired), w1 then w2 of every expert, the dense layer (model_io.py:24-36).
// Loading streams each matrix into the model (resident HBM, or the pinned
// host pool for offloaded experts); bf16 models round fp32 -> bf16 (RNE),
// the same rounding the rest of the package uses.  Errors carry the
// reference's messages (model_io.py:63-105) as PGMOE_E_WEIGHT_FILE.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace pgmoe {

static const char kMagic[6] = {'P', 'G', 'M', 'O', 'E', '1'};

static bool has_conv(const pgmoe_config &c, int b) { return c.activation_level == 0 || b < c.activation_level; }
static bool has_pre(const pgmoe_config &c, int b) {
    return c.activation_level != 0 && b < c.num_blocks - c.activation_level;
}

struct MatDesc {
    const char *name;
    int expert, rows, cols;
};

// model_io.py:24-36
static std::vector<MatDesc> block_layout(const pgmoe_config &c, int b) {
    std::vector<MatDesc> out;
    if (has_conv(c, b)) out.push_back({"gate", -1, c.d_model, c.num_experts});
    if (has_pre(c, b)) out.push_back({"pre_gate", -1, c.d_model, c.num_experts});
    for (int e = 0; e < c.num_experts; ++e) {
        out.push_back({"w1", e, c.d_ff, c.d_model});
        out.push_back({"w2", e, c.d_model, c.d_ff});
    }
    out.push_back({"non_moe", -1, c.d_model, c.d_model});
    return out;
}

static uint16_t f32_to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

static int read_header(FILE *fh, pgmoe_config *cfg) {
    char magic[6];
    const size_t got = fread(magic, 1, 6, fh);
    PG_REQUIRE(got == 6 && memcmp(magic, kMagic, 6) == 0, PGMOE_E_WEIGHT_FILE, "bad magic, expected b'PGMOE1'");
    int32_t dims[6];
    PG_REQUIRE(fread(dims, 4, 6, fh) == 6, PGMOE_E_WEIGHT_FILE, "truncated header");
    cfg->d_model = dims[0];
    cfg->d_ff = dims[1];
    cfg->num_blocks = dims[2];
    cfg->num_experts = dims[3];
    cfg->top_k = dims[4];
    cfg->activation_level = dims[5];
    const int32_t *v = dims;
    for (int i = 0; i < 5; ++i)
        PG_REQUIRE(v[i] >= 1, PGMOE_E_WEIGHT_FILE, "invalid header dimensions: dims must be positive");
    PG_REQUIRE(cfg->top_k <= cfg->num_experts && cfg->activation_level >= 0 &&
                   cfg->activation_level < cfg->num_blocks,
               PGMOE_E_WEIGHT_FILE, "invalid header dimensions: top_k / activation_level out of range");
    return PGMOE_OK;
}

}  // namespace pgmoe

using namespace pgmoe;

extern "C" int pgmoe_weight_file_config(const char *path, pgmoe_config *out) {
    FILE *fh = fopen(path, "rb");
    PG_REQUIRE(fh != nullptr, PGMOE_E_WEIGHT_FILE, "cannot open %s", path);
    pgmoe_config c{};
    const int st = read_header(fh, &c);
    fclose(fh);
    if (st == PGMOE_OK) *out = c;
    return st;
}

extern "C" int pgmoe_model_load_pgmoe1(pgmoe_model *m, const char *path) {
    pgmoe_config mc{};
    PG_TRY(pgmoe_model_config(m, &mc, nullptr));
    FILE *fh = fopen(path, "rb");
    PG_REQUIRE(fh != nullptr, PGMOE_E_WEIGHT_FILE, "cannot open %s", path);
    pgmoe_config c{};
    int st = read_header(fh, &c);
    if (st == PGMOE_OK && (c.d_model != mc.d_model || c.d_ff != mc.d_ff || c.num_blocks != mc.num_blocks ||
                           c.num_experts != mc.num_experts || c.top_k != mc.top_k ||
                           c.activation_level != mc.activation_level)) {
        set_error("weight file dimensions do not match the model");
        st = PGMOE_E_WEIGHT_FILE;
    }
    int32_t wdtype = 0;
    pgmoe_model_config(m, &mc, &wdtype);
    std::vector<float> buf;
    std::vector<uint16_t> bbuf;
    for (int b = 0; b < c.num_blocks && st == PGMOE_OK; ++b) {
        for (const MatDesc &md : block_layout(c, b)) {
            const size_t n = (size_t)md.rows * md.cols;
            buf.resize(n);
            if (fread(buf.data(), 4, n, fh) != n) {
                set_error("file ends inside block %d matrix '%s'", b, md.name);
                st = PGMOE_E_WEIGHT_FILE;
                break;
            }
            for (size_t i = 0; i < n; ++i)
                if (!std::isfinite(buf[i])) {
                    set_error("non-finite value in block %d matrix '%s'", b, md.name);
                    st = PGMOE_E_WEIGHT_FILE;
                    break;
                }
            if (st != PGMOE_OK) break;
            // expert-parallel shards keep only their experts (set_matrix refuses the rest)
            if (md.expert >= 0 && pgmoe_model_matrix_ptr(m, md.name, b, md.expert) == nullptr) continue;
            if (wdtype == PGMOE_BF16) {
                bbuf.resize(n);
                for (size_t i = 0; i < n; ++i) bbuf[i] = f32_to_bf16(buf[i]);
                st = pgmoe_model_set_matrix(m, md.name, b, md.expert, bbuf.data(), n * 2);
            } else {
                st = pgmoe_model_set_matrix(m, md.name, b, md.expert, buf.data(), n * 4);
            }
            if (st != PGMOE_OK) break;
        }
    }
    if (st == PGMOE_OK) {
        const long pos = ftell(fh);
        fseek(fh, 0, SEEK_END);
        const long end = ftell(fh);
        if (end != pos) {
            set_error("%ld trailing bytes after weights", end - pos);
            st = PGMOE_E_WEIGHT_FILE;
        }
    }
    fclose(fh);
    return st;
}

extern "C" int pgmoe_model_save_pgmoe1(pgmoe_model *m, const char *path) {
    pgmoe_config c{};
    int32_t wdtype = 0;
    PG_TRY(pgmoe_model_config(m, &c, &wdtype));
    FILE *fh = fopen(path, "wb");
    PG_REQUIRE(fh != nullptr, PGMOE_E_WEIGHT_FILE, "cannot open %s for writing", path);
    const int32_t dims[6] = {c.d_model, c.d_ff, c.num_blocks, c.num_experts, c.top_k, c.activation_level};
    fwrite(kMagic, 1, 6, fh);
    fwrite(dims, 4, 6, fh);
    std::vector<float> buf;
    std::vector<uint16_t> bbuf;
    int st = PGMOE_OK;
    for (int b = 0; b < c.num_blocks && st == PGMOE_OK; ++b) {
        for (const MatDesc &md : block_layout(c, b)) {
            const size_t n = (size_t)md.rows * md.cols;
            buf.resize(n);
            if (wdtype == PGMOE_BF16) {
                bbuf.resize(n);
                st = pgmoe_model_get_matrix(m, md.name, b, md.expert, bbuf.data(), n * 2);
                for (size_t i = 0; i < n; ++i) {
                    const uint32_t u = (uint32_t)bbuf[i] << 16;
                    memcpy(&buf[i], &u, 4);
                }
            } else {
                st = pgmoe_model_get_matrix(m, md.name, b, md.expert, buf.data(), n * 4);
            }
            if (st != PGMOE_OK) {
                set_error("cannot save a partial (expert-parallel) model: block %d %s %d", b, md.name, md.expert);
                break;
            }
            fwrite(buf.data(), 4, n, fh);
        }
    }
    fclose(fh);
    return st;
}
