S=rmatx:scale=28,ef=16,seed=1
python tools/probe.py $S --reps 3 --forest
python tools/probe.py $S --reps 3 --forest --ipc 1
python tools/probe.py $S --reps 3 --forest --ipc 2
python tools/probe.py $S --reps 3 --forest --ballast 20
python -c "
import sys; sys.path.insert(0,'.')
from paper_1612_01178_b200 import capi
c=capi.Context(0); g=c.generate('rmatx:scale=24,ef=16,seed=1'); c.cc(g); g.close()
import subprocess
" 
