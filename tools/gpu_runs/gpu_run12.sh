# Refresh after the fast Box-Muller / exact method / bits64 changes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r12_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r12_smoke.txt 2>&1
for w in c3_gauss c3_logn; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r12_$w.json 2>gpurun_out/r12_$w.err; done
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r12_c2.json 2>gpurun_out/r12_c2.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"philox" -c 1 -s 1 -o gpurun_out/r12_gauss_f32 python tools/ncu_target.py gauss_f32 28 3 > /dev/null 2>&1
python tools/probe.py > gpurun_out/r12_probe.txt 2>&1
cat gpurun_out/r12_pytest.txt gpurun_out/r12_smoke.txt; cat gpurun_out/r12_probe.txt
