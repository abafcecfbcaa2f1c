for c in c4 c5 c3; do for pr in 0 16; do
 timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --probe $pr > gpurun_out/s_${c}_$pr.json 2>/dev/null
done; done
