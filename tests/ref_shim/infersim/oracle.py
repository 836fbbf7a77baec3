from paper_2604_28175_b200.config import GroundTruthParams, default_ground_truth  # noqa: F401
