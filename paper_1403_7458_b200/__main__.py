"""``python -m paper_1403_7458_b200 ...``: the CLI drop-in (cli.py)."""
import sys

from .cli import main

sys.exit(main())
