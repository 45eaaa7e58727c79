"""python -m paper_2401_14762_b200 {synth,recover,report,bench} (pipeline.py)."""
import sys

from .pipeline import main

sys.exit(main())
