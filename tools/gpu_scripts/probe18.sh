timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "wide or star0 or adaptive" 2>&1 | tail -2
S=rmatx:scale=28,ef=16,seed=1
echo "wide  $(python tools/probe.py $S --reps 3 | cut -c60-170)"
echo "narrow $(HCC_COMP_WIDE=0 python tools/probe.py $S --reps 3 | cut -c60-170)"
echo "wide adaptive $(python tools/probe.py $S --reps 3 --algo adaptive | cut -c60-170)"
echo "narrow adaptive $(HCC_COMP_WIDE=0 python tools/probe.py $S --reps 3 --algo adaptive | cut -c60-170)"
for W in 1 0; do echo "rmat24 wide=$W $(HCC_COMP_WIDE=$W python tools/probe.py rmatx:scale=24,ef=16,seed=1 --reps 10 | cut -c60-170)"; done
for W in 1 0; do echo "er24 wide=$W $(HCC_COMP_WIDE=$W python tools/probe.py erx:n=16777216,m=268435456,seed=1 --reps 10 | cut -c60-170)"; done
for W in 1 0; do echo "grid wide=$W $(HCC_COMP_WIDE=$W python tools/probe.py grid:4096x4096 --reps 10 | cut -c60-170)"; done
