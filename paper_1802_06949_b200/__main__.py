"""python -m paper_1802_06949_b200 run|compare ... (the collsim CLI drop-in, cli.py)."""
import sys

from .cli import main

sys.exit(main())
