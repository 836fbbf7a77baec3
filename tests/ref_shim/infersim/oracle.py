from paper_2604_28175_b200.config import GroundTruthParams, default_ground_truth  # noqa: F401
from paper_2604_28175_b200.ground_truth import ground_truth_slowdown  # noqa: F401
