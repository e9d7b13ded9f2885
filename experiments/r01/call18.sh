#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/ab.log 2>&1
for R in 1 2; do
for C in c2 c3 c3n8; do
  PYTHONPATH=$PWD/ab_old timeout 300 python -c "
import sys; sys.path.insert(0,'$PWD/ab_old'); sys.argv=['x','--cfg','$C','--splits','0']
import paper_2405_01814_b200 as P; print('old lib', P.__file__, file=sys.stderr)
exec(open('scripts/exp_decode.py').read().replace('sys.path.insert(0, str(Path(__file__).resolve().parent.parent))',''))
" | sed "s/^/OLD /"
  timeout 300 python scripts/exp_decode.py --cfg $C --splits 0 | sed "s/^/NEW /"
done
done
