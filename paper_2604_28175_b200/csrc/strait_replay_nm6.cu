// strait_replay_nm6.cu — the replay engine instantiated for 6 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(6)
}  // namespace rp
}  // namespace strait
