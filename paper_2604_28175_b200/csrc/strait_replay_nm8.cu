// strait_replay_nm8.cu — the replay engine instantiated for 8 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(8)
}  // namespace rp
}  // namespace strait
