// strait_replay_nm2.cu — the replay engine instantiated for 2 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(2)
}  // namespace rp
}  // namespace strait
