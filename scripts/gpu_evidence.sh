#!/bin/bash
# Round evidence on one GPU (run under gpurun; outputs in gpurun_out/, copied to profiles/ by hand):
#   1. bench.py (default workload M3) -> ev_bench.json
#   2. its ncu launch list (gpu__time_duration per launch, cold-cache, serialised) -> ev_launches_summary.txt
#   3. ncu --set full of the M3 set-up kernel -> ncu_details/raw/source CSVs + summary (fp64 pipe, DFMA count, DRAM)
#   4. ncu DRAM bytes of the SpMV kernels (G r, G^T t, A p) inside an M3 PCG -> ev_spmv_dram.csv
#   5. the DMMA microbenchmark -> ev_dmma.txt
# TAG names the outputs (e.g. r02).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/ncu
TAG=${TAG:-r02}
WL=${WL:-M3}
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | grep -i "model name" >> gpurun_out/${TAG}_nproc.txt
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py --workload $WL > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench $?"
  tail -1 gpurun_out/${TAG}_bench.json | cut -c1-400
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu-list $?"
  python scripts/summarize_launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt 2>&1
  gzip -f gpurun_out/${TAG}_launches.csv
fi
if [ -z "$SKIP_SETUP_NCU" ]; then
  KIND=${KIND:-hetero}; N=${N:-200}
  # every set-up launch of ONE afsai_setup (table-probe passes, the main pass, retries);
  # the summary picks the longest (the main pass)
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:afsai_setup_rows -c 8 \
     -o /tmp/ncu/setup_$TAG -f python scripts/prof_setup.py $KIND $N 1 > gpurun_out/${TAG}_ncu_setup.log 2>&1
  echo "ncu-setup $?"
  ncu -i /tmp/ncu/setup_$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_setup_raw.csv 2>&1
  ncu -i /tmp/ncu/setup_$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_setup_details.csv 2>&1
  ncu -i /tmp/ncu/setup_$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_setup_source.csv 2>&1
  python scripts/ncu_summary.py gpurun_out/${TAG}_setup_details.csv gpurun_out/${TAG}_setup_raw.csv \
     > gpurun_out/${TAG}_setup_summary.txt 2>&1
  python scripts/ncu_source_lines.py /tmp/ncu/setup_$TAG.ncu-rep afsai_setup_rows 60 > gpurun_out/${TAG}_setup_lines.txt 2>&1
  python scripts/ncu_traffic.py gpurun_out/${TAG}_setup_raw.csv $WL > gpurun_out/${TAG}_setup_traffic_$WL.json 2>&1
  gzip -f gpurun_out/${TAG}_setup_source.csv gpurun_out/${TAG}_setup_raw.csv
fi
if [ -z "$SKIP_SPMV_NCU" ]; then
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
     -k regex:"spmv|pcg_" -s 40 -c 30 --log-file gpurun_out/${TAG}_spmv_dram.csv \
     python scripts/prof_pcg.py $WL > gpurun_out/${TAG}_ncu_spmv.log 2>&1; echo "ncu-spmv $?"
fi
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma scripts/micro/dmma.cu && /tmp/dmma > gpurun_out/${TAG}_dmma.txt 2>&1
cat gpurun_out/${TAG}_dmma.txt
