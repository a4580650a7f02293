// C-ABI layout introspection (lf_abi_sizeof / lf_abi_offsetof, include/leafi_b200.h).
#include <cstddef>
#include <cstring>

#include "../../include/leafi_b200.h"

// Layout table generated from include/leafi_b200.h (every field of the public structs).
namespace {
struct AbiField { const char* type; const char* field; int64_t offset; };
#define LF_F(T, F) {#T, #F, (int64_t)offsetof(T, F)}
const AbiField kFields[] = {
    LF_F(lf_index, n_series),
    LF_F(lf_index, m),
    LF_F(lf_index, n_seg),
    LF_F(lf_index, n_nodes),
    LF_F(lf_index, n_leaves),
    LF_F(lf_index, max_leaf_rows),
    LF_F(lf_index, seg_start),
    LF_F(lf_index, seg_width),
    LF_F(lf_index, d_X),
    LF_F(lf_index, d_row_id),
    LF_F(lf_index, d_leaf_ptr),
    LF_F(lf_index, d_node_leaf),
    LF_F(lf_index, d_env_min),
    LF_F(lf_index, d_env_max),
    LF_F(lf_index, d_leaf_filter),
    LF_F(lf_index, d_X8),
    LF_F(lf_index, d_qmeta),
    LF_F(lf_index, pca_k),
    LF_F(lf_index, d_P),
    LF_F(lf_index, d_mu),
    LF_F(lf_index, d_Xp),
    LF_F(lf_index, d_pmeta),
    LF_F(lf_search_opts, k),
    LF_F(lf_search_opts, bsf_factor),
    LF_F(lf_search_opts, d_pred),
    LF_F(lf_search_opts, d_pred_f64),
    LF_F(lf_search_opts, d_offset),
    LF_F(lf_search_opts, n_filters),
    LF_F(lf_search_opts, sequential),
    LF_F(lf_search_opts, max_round_leaves),
    LF_F(lf_search_opts, want_trace),
    LF_F(lf_search_opts, early_abandon),
    LF_F(lf_search_opts, h_profile),
    LF_F(lf_search_opts, d_W1T),
    LF_F(lf_search_opts, d_b1),
    LF_F(lf_search_opts, d_W2),
    LF_F(lf_search_opts, d_b2),
    LF_F(lf_trace, d_len),
    LF_F(lf_trace, d_leaf),
    LF_F(lf_trace, d_lb),
    LF_F(lf_trace, d_searched),
    LF_F(lf_trace, d_leaf_nn),
    LF_F(lf_trace, d_bsf_before),
};
#undef LF_F
struct AbiType { const char* type; int64_t size; };
const AbiType kTypes[] = {{"lf_index", (int64_t)sizeof(lf_index)}, {"lf_search_opts", (int64_t)sizeof(lf_search_opts)}, {"lf_trace", (int64_t)sizeof(lf_trace)}};
}  // namespace

extern "C" int64_t lf_abi_sizeof(const char* type_name) {
    if (type_name == nullptr) return -1;
    for (const auto& t : kTypes)
        if (std::strcmp(t.type, type_name) == 0) return t.size;
    return -1;
}

extern "C" int64_t lf_abi_offsetof(const char* type_name, const char* field_name) {
    if (type_name == nullptr || field_name == nullptr) return -1;
    for (const auto& f : kFields)
        if (std::strcmp(f.type, type_name) == 0 && std::strcmp(f.field, field_name) == 0) return f.offset;
    return -1;
}
