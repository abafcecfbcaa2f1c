for t in ft1 ft4 ft8; do
 echo "== $t" >> gpurun_out/fe_all.log
 CG_LIB=_ab/$t/libcachegram_b200.so timeout 600 python tools/_flush_exp.py >> gpurun_out/fe_all.log 2>&1
 CG_LIB=_ab/$t/libcachegram_b200.so timeout 600 python tools/quality_gates.py --configs c1 c2 --out gpurun_out/fe_q_$t.json > /dev/null 2>&1
done
