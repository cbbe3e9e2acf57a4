# One gpurun command that regenerates every input of tools/write_profiles.py:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/refresh_profiles.sh'
#   python tools/write_profiles.py r02
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err || exit 2
python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1 || exit 3
python tools/overflow_stress.py --out gpurun_out/overflow.json > gpurun_out/overflow.log 2>&1 || exit 4
PASA_BENCH_NO_SWEEP=1 PASA_BENCH_NO_CPU=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_l.log 2>&1 || exit 5
ncu --set full --clock-control none --import-source on -k regex:pasa_fwd -s 2 -c 1 -f -o gpurun_out/ncu_fwd128 python tools/ncu_once.py --shape qwen16k > gpurun_out/ncu128.log 2>&1 || exit 6
ncu --set full --clock-control none --import-source on -k regex:pasa_fwd -s 2 -c 1 -f -o gpurun_out/ncu_fwd64 python tools/ncu_once.py --shape svd > gpurun_out/ncu64.log 2>&1 || exit 7
ncu --set full --clock-control none --import-source on -k regex:packed -s 2 -c 1 -f -o gpurun_out/ncu_packed python tools/ncu_once.py --shape temporal > gpurun_out/ncupk.log 2>&1 || exit 8
tail -1 gpurun_out/bench.json
