from paper_2604_28175_b200.metrics import *  # noqa: F401,F403
from paper_2604_28175_b200.metrics import nearest_rank  # noqa: F401
