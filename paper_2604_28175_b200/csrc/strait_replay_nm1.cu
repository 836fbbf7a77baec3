// strait_replay_nm1.cu — the replay engine instantiated for 1 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(1)
}  // namespace rp
}  // namespace strait
