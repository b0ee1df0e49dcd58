python scripts/explore.py --cfg C5 --tol 1e-7 --modes patchy > gpurun_out/warm.log 2>&1
for c in C5 C4; do for x in 0x90 0x60 0xA0; do echo "$c oxor=$x"; PDD_OXOR=$x python scripts/explore.py --cfg $c --tol 1e-7 --modes patchy 2>&1 | tail -1 | cut -c1-200; done;
echo "$c k"; python scripts/explore.py --cfg $c --tol 1e-7 --modes patchy --k 2,3,5,6,8 2>&1 | tail -5 | cut -c1-200; done
