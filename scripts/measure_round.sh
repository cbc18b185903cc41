# Round measurements on the GPU box: bench lines of every config, the reference arm, the ncu
# launch list (durations + DRAM bytes) of a host-driven C5 solve and a full capture of the
# Arnoldi passes; everything lands in gpurun_out/ (copy what is to be judged into profiles/).
set -x
for c in C5 C1 C2 C3 C4; do timeout 400 python bench.py --config $c > gpurun_out/m_bench_$c.log 2>&1; done
timeout 300 python bench.py --impl reference > gpurun_out/m_ref_C5.log 2>&1
export HD_GRAPH=0
python scripts/profile_c5.py 100 C5 > gpurun_out/m_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/m_launches_C5.csv python scripts/profile_c5.py 100 C5 > gpurun_out/m_ncu1.log 2>&1
python scripts/profile_c5.py 40 C5 > gpurun_out/m_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_lsa_dots|k_lsa_update" -s 50 -c 4 -o gpurun_out/m_full python scripts/profile_c5.py 40 C5 > gpurun_out/m_ncu2.log 2>&1
unset HD_GRAPH
timeout 900 python scripts/cpu_full_solve.py C5 > gpurun_out/m_cpu_full_C5.log 2>&1
