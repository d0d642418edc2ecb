"""python -m paper_2208_14228_b200 <train|reprocheck|bitdiff> ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
