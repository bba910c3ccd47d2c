"""`python -m paper_1404_0774_b200 encode|decode|metrics|bench ...` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
