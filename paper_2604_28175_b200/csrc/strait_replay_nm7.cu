// strait_replay_nm7.cu — the replay engine instantiated for 7 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(7)
}  // namespace rp
}  // namespace strait
