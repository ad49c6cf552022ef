"""python -m paper_2404_02433_b200 generate|solve ... (see cli.py)."""

from .cli import main

raise SystemExit(main())
