python scripts/explore.py --cfg C5 --tol 1e-7 --modes patchy > gpurun_out/warm.log 2>&1
for c in C5 C4 C2; do for coh in 0.99 0.95 0.9 0.8; do echo "$c coh=$coh"; PDD_COH=$coh python scripts/explore.py --cfg $c --tol 1e-7 --modes patchy --k 1,2,4 2>&1 | tail -3 | cut -c1-190; done; done
