"""python -m paper_2508_17655_b200 ... -- the sbopt CLI on the GPU (cli.py)."""
import sys

from .cli import main

sys.exit(main())
