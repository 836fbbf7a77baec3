from paper_2604_28175_b200.report import *  # noqa: F401,F403
