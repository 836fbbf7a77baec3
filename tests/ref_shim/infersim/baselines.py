from paper_2604_28175_b200.baselines import *  # noqa: F401,F403
from paper_2604_28175_b200.baselines import (ABLATION_VARIANTS, POLICY_NAMES, ReactiveSpatialPolicy,  # noqa: F401
                                             ReactiveState, StaticSpatialPolicy, TemporalPolicy, make_policy)
from paper_2604_28175_b200.scheduler import *  # noqa: F401,F403
