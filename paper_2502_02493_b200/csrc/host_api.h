// Host-side analysis API: RunReport aggregation,
// the ESPEC1 model file, the similarity probe. See host_api.cpp.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "engine.h"

namespace espec {

// RunReport's derived metrics (proj/include/espec/report.hpp:40-57); times in
// seconds (the engine's device stage times).
struct ReportAgg {
    int iterations = 0;
    bool has_alpha = false;
    double alpha = 0.0;
    long tokens_emitted = 0;
    double mean_accept_len = 0.0;
    double tokens_per_s = 0.0;
    double draft_per100 = 0.0, verify_per100 = 0.0, calibrate_per100 = 0.0, draft_total_per100 = 0.0;
    double total = 0.0;  // measured device seconds of the three stages
    // the cost model's units (IterationTrace::*_sim, report.cpp:83-90)
    double draft_per100_sim = 0.0, verify_per100_sim = 0.0, calibrate_per100_sim = 0.0, draft_total_per100_sim = 0.0;
    double total_sim = 0.0;
    double speedup_vs_vanilla = 1.0;  // vanilla_baseline_sim / total_sim
};
ReportAgg aggregate_traces(const std::vector<IterationTrace>& traces, double vanilla_baseline_sim);
std::string report_csv(const ReportAgg& r, const std::string& algorithm, int n, int lp_size);
std::string report_json(const ReportAgg& r, const std::vector<IterationTrace>& traces, const std::string& algorithm,
                        int n, const std::vector<int>& widths, int lp_size);

struct ModelFileTensor {
    std::string file_name;   // manifest name, e.g. "layers.3.w_up"
    std::string short_name;  // engine tensor name, e.g. "w_up"
    int layer = -1;
    int rows = 0, cols = 0;
    int want_rows = 0, want_cols = 0;
    uint64_t offset = 0;  // byte offset of the tensor's data in the file
};
struct ModelFileInfo {
    ModelCfg cfg;
    std::vector<ModelFileTensor> tensors;
    uint64_t data_offset = 0;
};
// Parse and validate an ESPEC1 file (load_model's checks, proj/src/model_io.cpp:106-190);
// check_data also reads every tensor (truncation, non-finite values).
ModelFileInfo read_model_file(const std::string& path, bool check_data);
void load_model_file(Engine& eng, int which, const ModelCfg& engine_cfg, const std::string& path);
void save_model_file(Engine& eng, int which, const ModelCfg& cfg, const std::string& path);

struct SimilarityRow {
    int lp_size = 1;
    double h = 1.0, q = 1.0, k = 1.0, v = 1.0, attn_out = 1.0;
};
std::vector<SimilarityRow> probe_similarity(Engine& eng, int n_layers, const std::vector<int>& lp_sizes,
                                            const std::vector<std::vector<int>>& corpus);
std::string similarity_csv(const std::vector<SimilarityRow>& rows);

}  // namespace espec
