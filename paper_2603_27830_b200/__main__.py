"""``python -m paper_2603_27830_b200 <command> ...``: the sgp4kit CLI contract."""

import sys

from .cli import main

sys.exit(main())
