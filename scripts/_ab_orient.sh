python scripts/explore.py --cfg C5 --tol 1e-7 --modes patchy > gpurun_out/warm.log 2>&1
for c in C5 C4 C3; do
for v in 0 1; do echo "$c no_orient=$v"; if [ $v = 1 ]; then export PDD_NO_ORIENT=1; else unset PDD_NO_ORIENT; fi
python scripts/explore.py --cfg $c --tol 1e-7 --modes patchy 2>&1 | tail -1; done; done
