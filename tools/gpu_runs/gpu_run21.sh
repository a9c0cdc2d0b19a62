# MRG store-policy A/B; refreshed C3 bench lines with the new fast Box-Muller.
mkdir -p gpurun_out
python tools/ab_lib.py mrg_f64 28 3 main st1 > gpurun_out/r21_ab_mrg_st.txt 2>&1
python tools/ab_lib.py mrg_bits 28 2 main st1 >> gpurun_out/r21_ab_mrg_st.txt 2>&1
for w in c3_gauss c3_logn; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r21_$w.json 2>gpurun_out/r21_$w.err; done
cat gpurun_out/r21_*.txt gpurun_out/r21_*.json
