"""``python -m paper_2307_05266_b200`` runs the CLI (reference __main__.py)."""
import sys

from .cli import main

sys.exit(main())
