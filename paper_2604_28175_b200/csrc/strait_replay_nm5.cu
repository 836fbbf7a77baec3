// strait_replay_nm5.cu — the replay engine instantiated for 5 metric(s).
#include "strait_replay_impl.cuh"

namespace strait {
namespace rp {
STRAIT_INSTANTIATE_REPLAY(5)
}  // namespace rp
}  // namespace strait
