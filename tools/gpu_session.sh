#!/bin/bash
# One gpurun session: GPU tests, smoke, per-level diagnostics, bench line, ncu launch list and one
# --set full capture of the dominant kernel.  Usage (from this container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_session.sh [tests] [explore] [bench] [ncu]'
set -u
mkdir -p gpurun_out
OUT=gpurun_out
STEPS="${*:-tests explore bench ncu}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo "build failed" >> $OUT/build.log
for s in $STEPS; do
  case $s in
    tests)
      timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
      ;;
    explore)
      timeout 600 python tools/explore.py C1,C3,C4 set,edge -1 2 > $OUT/explore.log 2>&1
      timeout 600 python tools/explore.py C2 set 3 >> $OUT/explore.log 2>&1
      ;;
    c5)
      timeout 900 python tools/explore.py C5a,C5b,C5c set 2 > $OUT/explore_c5.log 2>&1
      timeout 900 python tools/explore.py C5d set 1 >> $OUT/explore_c5.log 2>&1
      timeout 900 python tools/explore.py C5e set 1 >> $OUT/explore_c5.log 2>&1
      ;;
    l1dense)
      for v in 0 1; do
        PCS_L1_DENSE=$v timeout 900 python tools/explore.py C5b,C5d set 1 2 >> $OUT/l1dense_$v.log 2>&1
      done
      PCS_L1_DENSE=1 timeout 900 python tools/explore.py C5e set 1 >> $OUT/l1dense_1.log 2>&1
      ;;
    merge)
      PCS_MERGE_PASSES=0 timeout 600 python tools/explore.py C2 set 3 2 > $OUT/merge_ab.log 2>&1
      timeout 600 python tools/explore.py C2 set 3 2 >> $OUT/merge_ab.log 2>&1
      ;;
    c2)
      timeout 600 python tools/explore.py C2 set 3 > $OUT/explore_c2.log 2>&1
      ;;
    ncutraffic)
      timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:level_set_kernel --csv --log-file $OUT/traffic.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-secondary > $OUT/ncu_traffic.log 2>&1
      ;;
    trace)
      PCS_TRACE=1 timeout 600 python bench.py --workload C3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e \
        --no-secondary > $OUT/trace_c3.json 2> $OUT/trace_c3.err
      ;;
    ncul1)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level1_kernel -c 1 -f -o $OUT/l1 \
        python tools/explore.py C5b set 1 > $OUT/ncu_l1.log 2>&1
      ;;
    ncufull)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_set --launch-skip 1 -c 1 -f -o $OUT/top \
        python tools/profile_target.py 3 16 set > $OUT/ncu_full.log 2>&1
      ;;
    balance)
      timeout 1200 python tools/shard_balance.py 8 C5 1 set > $OUT/balance.json 2> $OUT/balance.err
      timeout 1200 python tools/shard_balance.py 8 C2 3 set >> $OUT/balance.json 2>> $OUT/balance.err
      timeout 900 python tools/shard_balance.py 8 C3 -1 set >> $OUT/balance.json 2>> $OUT/balance.err
      timeout 900 python tools/shard_balance.py 8 C4 -1 set >> $OUT/balance.json 2>> $OUT/balance.err
      ;;
    candtrace)
      PCS_TRACE=1 timeout 900 python tools/variants.py run ${CANDV:-cand} --workload C2 --max-level 3 --repeats 1 > $OUT/cand.json 2> $OUT/cand.err
      ;;
    variantsl2)
      timeout 1500 python tools/variants.py run --workload C5 --max-level 2 --repeats 1 > $OUT/variants_c5l2.json 2> $OUT/variants_c5l2.err
      timeout 900 python tools/variants.py run --workload C2 --max-level 2 --repeats 3 > $OUT/variants_c2l2.json 2> $OUT/variants_c2l2.err
      ;;
    variantsl1)
      timeout 900 python tools/variants.py run --workload C5 --max-level 1 --repeats 2 > $OUT/variants_c5.json 2> $OUT/variants_c5.err
      timeout 900 python tools/variants.py run --workload C3 --max-level -1 --repeats 3 > $OUT/variants_c3.json 2> $OUT/variants_c3.err
      ;;
    variants)
      timeout 900 python tools/variants.py run --workload C2 --max-level 3 --repeats 2 > $OUT/variants.json 2> $OUT/variants.err
      ;;
    balance5)
      timeout 1500 python tools/shard_balance.py 8 C5 2 set > $OUT/balance_c5.json 2> $OUT/balance_c5.err
      ;;
    bench2)
      PCS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 1 --warmup 1 --no-cpu-baseline \
        --no-secondary > $OUT/bench2.json 2> $OUT/bench2.err
      ;;
    golden)
      timeout 1500 python -m pytest tests/test_gpu_golden.py -x -q -s > $OUT/pytest_golden.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_golden.log
      ;;
    l1tile)
      for v in 0 1; do
        PCS_L1_TILE=$v timeout 900 python tools/explore.py C3,C5b set 1 2 >> $OUT/l1tile_$v.log 2>&1
      done
      PCS_L1_TILE=1 timeout 900 python tools/explore.py C5d,C5e set 1 >> $OUT/l1tile_1.log 2>&1
      PCS_L1_TILE=0 timeout 900 python tools/explore.py C5d set 1 >> $OUT/l1tile_0.log 2>&1
      ;;
    ncul1t)
      PCS_L1_TILE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:level1_tile -c 1 -f -o $OUT/l1t \
        python tools/explore.py C5b set 1 > $OUT/ncu_l1t.log 2>&1
      ;;
    gram)
      for v in 1 2; do PCS_GRAM=$v timeout 900 python tools/time_corr.py C2,C3,C5b,C5e 5 >> $OUT/gram_ab.log 2>&1; done
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_dmma2 -c 1 -f -o $OUT/gram2 \
        python tools/time_corr.py C2 1 > $OUT/ncu_gram2.log 2>&1
      ;;
    sanitize)
      for tool in memcheck racecheck synccheck initcheck; do
        timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/explore.py C1 set,edge -1 \
          > $OUT/sanitizer_${tool}_C1.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_${tool}_C1.log
        timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 python tools/explore.py C3 set,edge -1 \
          > $OUT/sanitizer_${tool}_C3.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_${tool}_C3.log
      done
      PCS_L1_TILE=1 timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/explore.py C3 set 1 \
        > $OUT/sanitizer_racecheck_C3_l1tile.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_racecheck_C3_l1tile.log
      PCS_L1_TILE=1 timeout 1800 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/explore.py C3 set 1 \
        > $OUT/sanitizer_synccheck_C3_l1tile.log 2>&1; echo "rc=$?" >> $OUT/sanitizer_synccheck_C3_l1tile.log
      ;;
    shardtests)
      timeout 1200 python -m pytest tests/test_gpu_shards.py tests/test_gpu_multiproc.py tests/test_gpu_bench_multirank.py \
        tests/test_gpu_nccl.py -x -q > $OUT/pytest_shards.log 2>&1; echo "rc=$?" >> $OUT/pytest_shards.log
      ls /usr/include/eigen3 /usr/local/include/eigen3 > $OUT/eigen_check.txt 2>&1; find / -name "Dense" -path "*Eigen*" 2>/dev/null | head -3 >> $OUT/eigen_check.txt
      ;;
    ncur2)
      PCS_L1_TILE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:level1_tile -c 1 -f -o $OUT/l1t \
        python tools/explore.py C5b set 1 > $OUT/ncu_l1t.log 2>&1
      timeout 900 ncu --set full --clock-control none -k regex:gram_dmma2 -c 1 -f -o $OUT/gram2_c5e \
        python tools/time_corr.py C5e 1 > $OUT/ncu_gram2_c5e.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_set_rt -c 1 -f -o $OUT/rt \
        python tools/explore.py C3 set -1 > $OUT/ncu_rt.log 2>&1
      ;;
    balance5l2)
      PCS_BALANCE_REPEATS=1 timeout 2400 python tools/shard_balance.py 8 C5 2 set > $OUT/balance_c5l2.json 2> $OUT/balance_c5l2.err
      ;;
    pinvtab)
      for v in 0 2; do
        PCS_PINV_TABLE=$v timeout 900 python tools/explore.py C2 set 3 2 >> $OUT/pinvtab_$v.log 2>&1
        PCS_PINV_TABLE=$v timeout 900 python tools/explore.py C5a,C5c set 2 2 >> $OUT/pinvtab_$v.log 2>&1
      done
      ;;
    edgetab)
      for v in 0 2; do PCS_PINV_TABLE=$v timeout 900 python tools/explore.py C2 edge 2 2 >> $OUT/edgetab_$v.log 2>&1; done
      timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_random_sweep.py tests/test_gpu_parity.py -x -q \
        > $OUT/pytest_edgetab.log 2>&1; echo "rc=$?" >> $OUT/pytest_edgetab.log
      ;;
    ncul2)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_set_kernel -c 1 -f -o $OUT/l2 \
        python tools/explore.py C5a set 2 > $OUT/ncu_l2.log 2>&1
      ;;
    l2wide)
      timeout 1500 python tools/explore.py C5b set 2 > $OUT/l2wide.log 2>&1
      timeout 1200 python -m pytest tests/test_gpu_random_sweep.py tests/test_gpu_golden.py -x -q > $OUT/pytest_l2wide.log 2>&1; echo "rc=$?" >> $OUT/pytest_l2wide.log
      ;;
    c2l4)
      timeout 2400 python tools/explore.py C2 set 4 > $OUT/c2_level4.log 2>&1
      ;;
    ntvar)
      timeout 1200 python tools/variants.py run $VARIANTS --workload C2 --max-level 3 --repeats 2 > $OUT/ntvar_c2.json 2> $OUT/ntvar.err
      ;;
    ntvar5)
      timeout 1500 python tools/variants.py run $VARIANTS --workload C5 --max-level 2 --repeats 1 > $OUT/ntvar_c5.json 2> $OUT/ntvar5.err
      timeout 900 python tools/variants.py run $VARIANTS --workload C3 --max-level -1 --repeats 3 > $OUT/ntvar_c3.json 2>> $OUT/ntvar5.err
      ;;
    edgeab)
      timeout 900 python tools/variants.py run --strategy edge --workload C2 --max-level 2 --repeats 2 > $OUT/edgeab_c2.json 2> $OUT/edgeab.err
      timeout 900 python tools/variants.py run --strategy edge --workload C3 --max-level -1 --repeats 3 > $OUT/edgeab_c3.json 2>> $OUT/edgeab.err
      timeout 900 python tools/variants.py run --strategy edge --workload C4 --max-level -1 --repeats 3 > $OUT/edgeab_c4.json 2>> $OUT/edgeab.err
      timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_random_sweep.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q \
        > $OUT/pytest_edge.log 2>&1; echo "rc=$?" >> $OUT/pytest_edge.log
      ;;
    edgeab2)
      timeout 900 python tools/variants.py run spl1 spl4 spl2m3 --strategy edge --workload C2 --max-level 2 --repeats 2 > $OUT/edgeab2_c2.json 2> $OUT/edgeab2.err
      timeout 900 python tools/variants.py run spl1 spl4 spl2m3 --strategy edge --workload C3 --max-level -1 --repeats 3 > $OUT/edgeab2_c3.json 2>> $OUT/edgeab2.err
      timeout 900 python tools/variants.py run stagerep2 p1rep2 dbuf --workload C2 --max-level 3 --repeats 2 > $OUT/probes_c2.json 2>> $OUT/edgeab2.err
      timeout 900 python tools/explore.py C2 edge 3 > $OUT/explore_c2_edge.log 2>&1
      ;;
    edgel3)
      PCS_PINV_TABLE=0 timeout 900 python tools/explore.py C2 edge 3 > $OUT/explore_c2_edge_notable.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_edge_staged -c 1 -f -o $OUT/edge2 \
        python tools/profile_target.py 2 4 edge > $OUT/ncu_edge2.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_edge_staged -c 1 -f -o $OUT/edge3 \
        python tools/profile_target.py 3 256 edge > $OUT/ncu_edge3.log 2>&1
      ;;
    edgeab3)
      timeout 900 python tools/variants.py run spl2 spl2m4 unstaged --strategy edge --workload C2 --max-level 2 --repeats 2 > $OUT/edgeab3_c2.json 2> $OUT/edgeab3.err
      timeout 900 python tools/variants.py run spl2 spl2m4 unstaged --strategy edge --workload C3 --max-level -1 --repeats 3 > $OUT/edgeab3_c3.json 2>> $OUT/edgeab3.err
      timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_random_sweep.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q \
        > $OUT/pytest_edge.log 2>&1; echo "rc=$?" >> $OUT/pytest_edge.log
      timeout 900 python tools/explore.py C2 edge 3 > $OUT/explore_c2_edge.log 2>&1
      ;;
    l2links)
      timeout 900 python tools/variants.py run old dbuf ntl24 --workload C5a --max-level 2 --repeats 2 > $OUT/l2links_c5a.json 2> $OUT/l2links.err
      timeout 900 python tools/variants.py run old dbuf ntl24 --workload C5c --max-level 2 --repeats 1 > $OUT/l2links_c5c.json 2>> $OUT/l2links.err
      timeout 900 python tools/variants.py run old --workload C2 --max-level 3 --repeats 2 > $OUT/l2links_c2.json 2>> $OUT/l2links.err
      timeout 1800 python tools/variants.py run old --workload C5 --max-level 2 --repeats 1 > $OUT/l2links_c5.json 2>> $OUT/l2links.err
      timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_random_sweep.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q \
        > $OUT/pytest_l2links.log 2>&1; echo "rc=$?" >> $OUT/pytest_l2links.log
      ;;
    dbuf2)
      timeout 900 python tools/variants.py run dbuf2 --workload C5a --max-level 2 --repeats 3 > $OUT/dbuf2_c5a.json 2> $OUT/dbuf2.err
      timeout 900 python tools/variants.py run dbuf2 --workload C5c --max-level 2 --repeats 2 > $OUT/dbuf2_c5c.json 2>> $OUT/dbuf2.err
      timeout 900 python tools/variants.py run dbuf2 --workload C2 --max-level 3 --repeats 2 > $OUT/dbuf2_c2.json 2>> $OUT/dbuf2.err
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_edge_staged -c 1 -f -o $OUT/edge2 \
        python tools/profile_target.py 2 4 edge > $OUT/ncu_edge2.log 2>&1
      ;;
    edgepf)
      timeout 900 python tools/variants.py run prev --strategy edge --workload C2 --max-level 2 --repeats 2 > $OUT/edgepf_c2.json 2> $OUT/edgepf.err
      timeout 900 python tools/variants.py run prev --strategy edge --workload C3 --max-level -1 --repeats 3 > $OUT/edgepf_c3.json 2>> $OUT/edgepf.err
      timeout 900 python tools/variants.py run l2m5 l2m6 --workload C5a --max-level 2 --repeats 3 > $OUT/l2m_c5a.json 2>> $OUT/edgepf.err
      timeout 900 python tools/variants.py run l2m5 l2m6 --workload C5c --max-level 2 --repeats 2 > $OUT/l2m_c5c.json 2>> $OUT/edgepf.err
      timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_random_sweep.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q \
        > $OUT/pytest_edgepf.log 2>&1; echo "rc=$?" >> $OUT/pytest_edgepf.log
      timeout 900 python tools/explore.py C2 edge 3 > $OUT/explore_c2_edge.log 2>&1
      ;;
    occ)
      timeout 900 python tools/variants.py run nt3m5 nt2m6 --workload C2 --max-level 3 --repeats 2 > $OUT/occ_c2.json 2> $OUT/occ.err
      timeout 1800 python tools/variants.py run l2m4 --workload C5 --max-level 2 --repeats 1 > $OUT/occ_c5.json 2>> $OUT/occ.err
      ;;
    final)
      timeout 900 python tools/variants.py run l2m7 --workload C5a --max-level 2 --repeats 3 > $OUT/l2m7_c5a.json 2> $OUT/final.err
      timeout 900 python tools/variants.py run l2m7 --workload C5c --max-level 2 --repeats 2 > $OUT/l2m7_c5c.json 2>> $OUT/final.err
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_set_kernel -c 1 -f -o $OUT/l2 \
        python tools/explore.py C5a set 2 > $OUT/ncu_l2.log 2>&1
      ;;
    tracec2)
      PCS_TRACE=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-secondary > $OUT/trace_c2.json 2> $OUT/trace_c2.err
      ;;
    h00s)
      timeout 900 python tools/variants.py run prev --workload C2 --max-level 3 --repeats 2 > $OUT/h00s_c2.json 2> $OUT/h00s.err
      timeout 900 python tools/variants.py run prev --workload C5a --max-level 2 --repeats 3 > $OUT/h00s_c5a.json 2>> $OUT/h00s.err
      timeout 900 python tools/variants.py run prev --workload C5c --max-level 2 --repeats 2 > $OUT/h00s_c5c.json 2>> $OUT/h00s.err
      timeout 900 python tools/variants.py run prev --workload C3 --max-level -1 --repeats 3 > $OUT/h00s_c3.json 2>> $OUT/h00s.err
      timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_h00s.log 2>&1; echo "rc=$?" >> $OUT/pytest_h00s.log
      ;;
    tracee2e)
      PCS_TRACE=1 timeout 600 python bench.py --workload C4 --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > $OUT/trace_c4.json 2> $OUT/trace_c4.err
      PCS_TRACE=1 timeout 600 python bench.py --workload C3 --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > $OUT/trace_c3.json 2> $OUT/trace_c3.err
      ;;
    eocc)
      timeout 900 python tools/variants.py run eminb5 eminb6 --strategy edge --workload C2 --max-level 2 --repeats 2 > $OUT/eocc_c2.json 2> $OUT/eocc.err
      timeout 900 python tools/variants.py run eminb5 eminb6 --strategy edge --workload C5a --max-level 2 --repeats 2 > $OUT/eocc_c5a.json 2>> $OUT/eocc.err
      ;;
    c3launch)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/c3_launches.csv \
        python tools/explore.py C3 set -1 > $OUT/c3_launch.log 2>&1
      ;;
    rtmerge)
      timeout 900 python tools/variants.py run prev --workload C3 --max-level -1 --repeats 3 > $OUT/rtm_c3.json 2> $OUT/rtm.err
      timeout 900 python tools/variants.py run prev --strategy edge --workload C3 --max-level -1 --repeats 3 > $OUT/rtm_c3e.json 2>> $OUT/rtm.err
      timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_random_sweep.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_shards.py tests/test_gpu_multiproc.py -x -q \
        > $OUT/pytest_rtm.log 2>&1; echo "rc=$?" >> $OUT/pytest_rtm.log
      ;;
    ncudeep)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_set_kernel --launch-skip 6 -c 1 -f -o $OUT/deep8 \
        python tools/explore.py C3 set -1 > $OUT/ncu_deep8.log 2>&1
      timeout 900 python tools/explore.py C3 set -1 > $OUT/explore_c3.log 2>&1
      ;;
    deep)
      timeout 900 python tools/variants.py run deep2 --workload C3 --max-level -1 --repeats 3 > $OUT/deep_c3.json 2> $OUT/deep.err
      timeout 900 python tools/variants.py run deep2 --strategy edge --workload C3 --max-level -1 --repeats 3 > $OUT/deep_c3e.json 2>> $OUT/deep.err
      ;;
    fp64ilp)
      ./tools/micro/fp64_ilp > $OUT/fp64_ilp.log 2>&1
      ;;
    l1compact)
      timeout 900 python tools/variants.py run nocompact --workload C3 --max-level 1 --repeats 3 > $OUT/l1c_c3.json 2> $OUT/l1c.err
      timeout 900 python tools/variants.py run nocompact --workload C4 --max-level 1 --repeats 3 > $OUT/l1c_c4.json 2>> $OUT/l1c.err
      timeout 900 python tools/variants.py run nocompact --workload C2 --max-level 1 --repeats 3 > $OUT/l1c_c2.json 2>> $OUT/l1c.err
      timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_l1c.log 2>&1; echo "rc=$?" >> $OUT/pytest_l1c.log
      ;;
    links6)
      timeout 900 python tools/variants.py run links --workload C5a --max-level 2 --repeats 3 > $OUT/links6_c5a.json 2> $OUT/links6.err
      timeout 900 python tools/variants.py run links --workload C5c --max-level 2 --repeats 2 > $OUT/links6_c5c.json 2>> $OUT/links6.err
      timeout 900 python tools/variants.py run links --workload C2 --max-level 2 --repeats 3 > $OUT/links6_c2.json 2>> $OUT/links6.err
      ;;
    bench)
      timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
      ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-secondary > $OUT/ncu_bench.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_set --launch-skip 1 -c 1 -f -o $OUT/top \
        python tools/profile_target.py 3 16 set > $OUT/ncu_full.log 2>&1
      ;;
  esac
done
echo done > $OUT/session_done.txt
