// strait_replay_nm3.cu — the replay engine instantiated for 3 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(3)
}  // namespace rp
}  // namespace strait
