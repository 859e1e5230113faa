"""python -m paper_2510_12357_b200 (cli.py)."""
import sys

from .cli import main

sys.exit(main())
