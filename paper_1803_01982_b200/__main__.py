"""python -m paper_1803_01982_b200 {svd,tensor,rpca,complete} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
