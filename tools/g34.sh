timeout -s KILL 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "eigengame or huge or oja or C2 or C4 or c4m or upload or minibatch or sampled or refine" 2>&1 | tail -3
timeout -s KILL 1200 python tools/huge_d.py --steps 60 --out gpurun_out/r2_huge_d.txt > gpurun_out/g34_huge.log 2>&1; grep -E "ms|gbs" gpurun_out/r2_huge_d.txt
timeout -s KILL 300 python tools/prof_minibatch.py C4 50 split
