"""`python -m paper_2512_18995_b200 run FILE ...` (circuit_file.main)."""
import sys

from .circuit_file import main

sys.exit(main())
