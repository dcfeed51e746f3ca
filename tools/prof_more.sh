# ncu --set full captures of the remaining hot kernels, in the bench (one GPU).
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu"
ncu --set full --clock-control none -k regex:panel_kernel -s 60 -c 1 -o gpurun_out/prof_panel_bench $B > gpurun_out/ncu_p.log 2>&1
ncu --set full --clock-control none -k "regex:dgemm_kernel<GemmCfg<128, 64, 16" -s 100 -c 1 -o gpurun_out/prof_schur_bench $B > gpurun_out/ncu_s.log 2>&1
ncu --set full --clock-control none -k regex:rng_attempt -s 60 -c 1 -o gpurun_out/prof_rng_bench $B > gpurun_out/ncu_r.log 2>&1
for r in prof_panel_bench prof_schur_bench prof_rng_bench; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
tail -n 2 gpurun_out/ncu_p.log gpurun_out/ncu_s.log gpurun_out/ncu_r.log
