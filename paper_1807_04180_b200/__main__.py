"""`python -m paper_1807_04180_b200 solve run.cfg` -- the helmddm command line
(proj/tools/helmddm_main.cpp) on the B200 engine; see cli.py."""
import sys

from .cli import main

sys.exit(main())
