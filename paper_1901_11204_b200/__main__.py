"""``python -m paper_1901_11204_b200 ...`` = the GPU harness CLI (the reference's
``paircount`` console script, pyproject.toml [project.scripts])."""

import sys

from .bench_cli import main

sys.exit(main())
