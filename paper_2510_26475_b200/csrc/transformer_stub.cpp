// Placeholder until the transformer forwards land (model.cu).
#include <stdexcept>
#include "engine.h"
namespace rs {
std::unique_ptr<ModelPair> make_transformer_pair(rs_ctx *, const rs_model *, const rs_model *, int, int,
                                                 const std::vector<int> &, const std::vector<std::vector<int>> &, int) {
    throw std::invalid_argument("transformer models not built yet");
}
}  // namespace rs
extern "C" {
int rs_transformer_create(rs_ctx *, const rs_transformer_shape *, uint64_t, rs_model **) { return RS_EINVAL; }
int rs_drafter_create(rs_ctx *, const rs_model *, uint64_t, int32_t, rs_model **) { return RS_EINVAL; }
}
