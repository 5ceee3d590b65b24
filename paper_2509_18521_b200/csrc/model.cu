// Placeholder until the transformer lands.
#include "engine.cuh"
namespace ab {
struct Model {};
Model* model_create(Engine&) { throw Error(AB_ERR_CONFIG, "transformer model not built"); }
void model_destroy(Model*) {}
int model_weight_count(Model*) { return 0; }
void model_weight_info(Model*, int, std::string*, int64_t*, int64_t*, void**) {}
void model_open_group(Engine&, int, const int32_t*, int) {}
void model_release_group(Engine&, int) {}
void model_submit(Engine&, const ab_sample_desc*, int) {}
void model_release(Engine&, const int32_t*, int) {}
void model_iteration(Engine&, int64_t, bool) {}
int64_t model_pages_total(Model*) { return 0; }
}
