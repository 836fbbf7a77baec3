// strait_replay_nm4.cu — the replay engine instantiated for 4 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(4)
}  // namespace rp
}  // namespace strait
