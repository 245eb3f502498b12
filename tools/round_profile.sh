#!/usr/bin/env bash
# One GPU call that regenerates the round's evidence into gpurun_out/ (run on
# the B200 box from the repo root, after build()):
#   gpu tests + smoke, the default bench line, the reference arm, the config-1
#   pipeline workload, the ncu launch list of the bench command, one
#   `ncu --set full` capture of the Gram kernel, the config sweeps and the C++
#   drop-in harness. Each step runs under its own timeout; ncu steps only after
#   the plain command exited 0.
set -u
out=gpurun_out
mkdir -p "$out"
log() { echo "[$(date +%T)] $*" | tee -a "$out/round_profile.log"; }

log "gpu tests"
timeout 1500 python -m pytest tests -m gpu -q > "$out/rp_gpu_tests.txt" 2>&1; log "gpu tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -s > "$out/rp_config_parity.txt" 2>&1; log "config parity rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/rp_smoke.txt" 2>&1; log "smoke rc=$?"
[ -x tests/cpp/_build/parity ] && { timeout 900 tests/cpp/_build/parity > "$out/rp_parity_harness.txt" 2>&1; log "harness rc=$?"; }

log "bench (default)"
timeout 900 python bench.py > "$out/rp_bench.json" 2> "$out/rp_bench.err"; rc=$?; log "bench rc=$rc"
timeout 900 python bench.py --impl reference > "$out/rp_bench_reference.json" 2> "$out/rp_bench_reference.err"; log "reference arm rc=$?"
timeout 900 python bench.py --workload c1-pipeline > "$out/rp_bench_c1.json" 2> "$out/rp_bench_c1.err"; log "c1 pipeline rc=$?"

if [ "$rc" = 0 ]; then
  log "ncu launch list"
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file "$out/rp_launches.csv" python bench.py --steps 2 --warmup 1 > "$out/rp_ncu_bench.log" 2>&1
  log "launch list rc=$?"
  log "ncu full (gram)"
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gram_dmma -s 1 -c 1 \
      -o "$out/rp_gram" -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > "$out/rp_ncu_gram.log" 2>&1
  log "ncu gram rc=$?"
fi

log "config sweeps"
timeout 1200 python tools/config_sweep.py --configs c1,c3,c5,c5f > "$out/rp_sweep.log" 2>&1; log "sweep rc=$?"
cp "$out/config_sweep.jsonl" "$out/rp_sweep_c1_c3_c5.jsonl" 2>/dev/null
timeout 900 python tools/config_sweep.py --configs c4 > "$out/rp_sweep_c4.log" 2>&1; log "sweep c4 rc=$?"
cp "$out/config_sweep.jsonl" "$out/rp_sweep_c4.jsonl" 2>/dev/null
log "done"
