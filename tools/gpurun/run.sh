#!/bin/bash
# Named steps for one GPU call:  gpurun -- 'bash tools/gpurun/run.sh STEP [STEP...]'
# Every step writes gpurun_out/<tag>_<step>.log (TAG env, default "g").
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
TAG=${TAG:-g}
O=gpurun_out/${TAG}
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm,power.draw --format=csv > ${O}_smi.txt 2>&1
for step in "$@"; do
  case "$step" in
    build)  python -m paper_2206_00057_b200.build > ${O}_build.log 2>&1 ;;
    roof)   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/gather_roof tools/gather_roof.cu \
              && timeout 900 tools/gather_roof > ${O}_roof.jsonl 2> ${O}_roof.err ;;
    spmm)   timeout 900 python tools/spmm_bench.py --widths 256,100,48 > ${O}_spmm.log 2>&1 ;;
    spmm8)  timeout 900 python tools/spmm_bench.py --parts 8 --widths 256,100,48 > ${O}_spmm8.log 2>&1 ;;
    async)  timeout 900 python -m pytest tests/test_gpu_async.py -q -x -p no:cacheprovider > ${O}_async.log 2>&1 ;;
    tests)  timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > ${O}_tests.log 2>&1; echo "rc=$?" >> ${O}_tests.log ;;
    fast)   timeout 2400 python -m pytest tests -q -m "gpu and not slow" -p no:cacheprovider > ${O}_fast.log 2>&1; echo "rc=$?" >> ${O}_fast.log ;;
    smoke)  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "rc=$?" >> ${O}_smoke.log ;;
    bench)  timeout 900 python bench.py > ${O}_bench.log 2>&1 ;;
    launches) timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
              --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-ncu --no-parts-variant > ${O}_launches.log 2>&1 ;;
    nsweep) for kv in ${NSWEEP:-"DIGEST_SPMM_N=1" "DIGEST_SPMM_N=5" "DIGEST_SPMM_N=6" "DIGEST_SPMM_N=7" "DIGEST_SPMM_N=8"}; do
              kvs=$(echo $kv | tr ',' ' ')
              echo "== $kvs" >> ${O}_nsweep.log
              env DIGEST_KNOBS=1 $kvs timeout 300 python tools/spmm_bench.py --widths ${NW:-256,100,48} --iters 5 >> ${O}_nsweep.log 2>&1
              env DIGEST_KNOBS=1 $kvs timeout 300 python tools/spmm_bench.py --parts 8 --widths ${NW:-256,100,48} --iters 5 >> ${O}_nsweep.log 2>&1
            done ;;
    variants) timeout 1500 python -m pytest tests/test_gpu_spmm_variants.py -q -x -p no:cacheprovider ${VK:+-k "$VK"} > ${O}_variants.log 2>&1 ;;
    parity) timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > ${O}_parity.log 2>&1; echo "rc=$?" >> ${O}_parity.log ;;
    oraclefull) timeout 1500 python tools/oracle_full_epoch.py --frac 1.0 > ${O}_oraclefull.log 2>&1
                timeout 600 python tools/oracle_full_epoch.py --frac 0.1 >> ${O}_oraclefull.log 2>&1 ;;
    ncun)   for spec in "w48:48:1::" "w256s64:256:4:DIGEST_SPMM_SMAX=64:" "w48old:48:1:DIGEST_SPMM_N=0:" ${NCUN_EXTRA}; do
              IFS=: read name wd skip kn _ <<< "$spec"
              env DIGEST_KNOBS=1 $(echo $kn | tr ',' ' ') timeout 600 $NCU --set full --import-source on \
                --clock-control none -k regex:k_spmm -s $skip -c 1 -o ${O}_ncu_$name \
                python tools/spmm_bench.py --widths $wd --iters 1 >> ${O}_ncun.log 2>&1
              $NCU -i ${O}_ncu_$name.ncu-rep --page raw --csv > ${O}_ncu_${name}_raw.csv 2>> ${O}_ncun.log
              $NCU -i ${O}_ncu_$name.ncu-rep --page details --csv > ${O}_ncu_${name}_details.csv 2>> ${O}_ncun.log
              $NCU -i ${O}_ncu_$name.ncu-rep --page source --csv > ${O}_ncu_${name}_source.csv 2>> ${O}_ncun.log
              gzip -f ${O}_ncu_${name}_source.csv
              rm -f ${O}_ncu_$name.ncu-rep
            done ;;
    full)   timeout 2400 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_halo_grad.py tests/test_gpu_async.py -q -x -s -p no:cacheprovider > ${O}_full.log 2>&1; echo "rc=$?" >> ${O}_full.log ;;
    async_roof) nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/gather_async tools/gather_async.cu \
              && timeout 900 tools/gather_async > ${O}_async_roof.jsonl 2> ${O}_async_roof.err ;;
    sanitize) CS=/usr/local/cuda/bin/compute-sanitizer
            for tool in memcheck racecheck synccheck initcheck; do
              echo "== $tool smoke" >> ${O}_sanitize.log
              timeout 900 $CS --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" >> ${O}_sanitize.log 2>&1
              echo "rc=$?" >> ${O}_sanitize.log
            done
            echo "== memcheck cora loopback M=2 (bench)" >> ${O}_sanitize.log
            timeout 1200 $CS --tool memcheck --print-limit 20 python bench.py --config cora --loopback 2 --steps 2 --warmup 1 --no-e2e --no-ncu >> ${O}_sanitize.log 2>&1
            echo "rc=$?" >> ${O}_sanitize.log
            echo "== racecheck cora loopback M=2 (bench)" >> ${O}_sanitize.log
            timeout 1800 $CS --tool racecheck --print-limit 20 python bench.py --config cora --loopback 2 --steps 1 --warmup 1 --no-e2e --no-ncu >> ${O}_sanitize.log 2>&1
            echo "rc=$?" >> ${O}_sanitize.log
            echo "== memcheck peer transport 2 processes" >> ${O}_sanitize.log
            timeout 1800 $CS --tool memcheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_peer.py -q -x -k "M2_N1_sgd" -p no:cacheprovider >> ${O}_sanitize.log 2>&1
            echo "rc=$?" >> ${O}_sanitize.log
            echo "== memcheck SpMM kernels (lean, tiled, slabs)" >> ${O}_sanitize.log
            timeout 1800 $CS --tool memcheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_spmm_variants.py -q -x -k "w48-MM_N1-MODE or w100-MM_N1-MODE or w64-MM_N2 or w256-SMAX64-MODE0" -p no:cacheprovider >> ${O}_sanitize.log 2>&1
            echo "rc=$?" >> ${O}_sanitize.log ;;
    sanitize2) CS=/usr/local/cuda/bin/compute-sanitizer   # the round-2 grouped SpMM kernel
            for tool in memcheck racecheck synccheck; do
              echo "== $tool grouped SpMM (w100 default, w48 N6, multi-window)" >> ${O}_sanitize2.log
              timeout 1500 $CS --tool $tool --target-processes all --print-limit 20 python -m pytest tests/test_gpu_spmm_variants.py -q -x \
                -k "w100-MM_N1-MODE0-ODES40000 or w48-MM_N6-MODE0 or w100-MM_N1-MODE2-ODES40000" -p no:cacheprovider >> ${O}_sanitize2.log 2>&1
              echo "rc=$?" >> ${O}_sanitize2.log
            done ;;
    hotncu) # L2 hit rate / DRAM bytes of the w=256 product with and without evict_last hot rows
            for spec in "base::" "pfh0:DIGEST_SPMM_PFH=1,DIGEST_HOT_ROWS=0" "pfh98k:DIGEST_SPMM_PFH=1,DIGEST_HOT_ROWS=98304" \
                        "pfh400k:DIGEST_SPMM_PFH=1,DIGEST_HOT_ROWS=400000" "pfh1m:DIGEST_SPMM_PFH=1,DIGEST_HOT_ROWS=1000000" \
                        "rowwarp:DIGEST_SPMM_V=7" \
                        "h4_490k:DIGEST_SPMM_PFH=1,DIGEST_SPMM_HINTS=4,DIGEST_HOT_ROWS=490000" \
                        "h4_980k:DIGEST_SPMM_PFH=1,DIGEST_SPMM_HINTS=4,DIGEST_HOT_ROWS=980000" \
                        "h4_1470k:DIGEST_SPMM_PFH=1,DIGEST_SPMM_HINTS=4,DIGEST_HOT_ROWS=1470000" \
                        "h1_490k:DIGEST_SPMM_PFH=1,DIGEST_SPMM_HINTS=1,DIGEST_HOT_ROWS=490000" ${HOTNCU_EXTRA}; do
              IFS=: read name kn <<< "$spec"
              echo "== $name $kn" >> ${O}_hotncu.log
              env DIGEST_KNOBS=1 $(echo $kn | tr ',' ' ') timeout 600 $NCU --metrics \
                gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex.sum \
                --clock-control none -k regex:k_spmm -s 1 -c 1 --csv --print-units base \
                python tools/spmm_bench.py --widths 256 --iters 1 >> ${O}_hotncu.log 2>&1
              env DIGEST_KNOBS=1 $(echo $kn | tr ',' ' ') timeout 300 python tools/spmm_bench.py --widths 256 --iters 5 >> ${O}_hotncu.log 2>&1
            done ;;
    wsweep) # w=256 SpMM variants on products M=1, one 8-part partition and Reddit M=1
            for v in ${WSWEEP:-0 7 17 18}; do
              for cp in "products:1" "products:8" "reddit:1"; do
                IFS=: read cfg parts <<< "$cp"
                echo "== V=$v $cfg/$parts" >> ${O}_wsweep.log
                env DIGEST_KNOBS=1 DIGEST_SPMM_V=$v ${WSWEEP_ENV} timeout 300 python tools/spmm_bench.py --config $cfg --parts $parts \
                  --widths ${NW:-256} --iters 5 >> ${O}_wsweep.log 2>&1
              done
            done ;;
    polncu) # the default (grouped) w=256 product vs the grouped kernel with the hot-bit L2 policy
            for spec in "grouped::" "g17_300k:DIGEST_SPMM_V=17,DIGEST_HOT_ROWS=300000" \
                        "g17_490k:DIGEST_SPMM_V=17,DIGEST_HOT_ROWS=490000" "g17_735k:DIGEST_SPMM_V=17,DIGEST_HOT_ROWS=735000" \
                        "rowwarp:DIGEST_SPMM_V=7"; do
              IFS=: read name kn <<< "$spec"
              echo "== $name $kn" >> ${O}_polncu.log
              env DIGEST_KNOBS=1 $(echo $kn | tr ',' ' ') timeout 600 $NCU --metrics \
                gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex.sum \
                --clock-control none -k regex:k_spmm -s 1 -c 1 --csv --print-units base \
                python tools/spmm_bench.py --widths 256 --iters 1 >> ${O}_polncu.log 2>&1
              env DIGEST_KNOBS=1 $(echo $kn | tr ',' ' ') timeout 300 python tools/spmm_bench.py --widths 256 --iters 5 >> ${O}_polncu.log 2>&1
            done ;;
    gemmraw) # A_hi = the raw fp32 tile (kind::tf32 reading the upper 19 bits) vs the split A_hi
            timeout 900 python tools/gemm_bench.py --iters 10 --shapes 100x256,256x256,256x48,48x256 > ${O}_gemmraw.log 2>&1
            env DIGEST_KNOBS=1 DIGEST_GEMM_RAWHI=1 timeout 900 python tools/gemm_bench.py --iters 10 --shapes 100x256,256x256,256x48,48x256 >> ${O}_gemmraw.log 2>&1
            timeout 900 python -m pytest tests/test_gpu_gemm_variants.py -q -p no:cacheprovider >> ${O}_gemmraw.log 2>&1 ;;
    timeline) timeout 900 python tools/timeline.py --config products --parts 8 --epochs 3 --sync-interval 1 \
                --out ${O}_timeline_products8.json > ${O}_timeline.log 2>&1
              timeout 900 python tools/timeline.py --config reddit --parts 4 --epochs 3 --sync-interval 1 \
                --out ${O}_timeline_reddit4.json >> ${O}_timeline.log 2>&1 ;;
    l2spmm) for sc in 0.03125 0.0625 0.125 0.25; do
              timeout 300 python tools/spmm_bench.py --scale $sc --widths 256,100,48 --iters 10 >> ${O}_l2spmm.log 2>&1
            done ;;
    matrix) # every config at its M (loopback = all M parts on this GPU)
            for spec in "products:2:async" "products:4:async" "products:8:async" \
                        "reddit:1:sync" "reddit:1:async" "reddit:2:sync" "reddit:2:async" \
                        "reddit:4:sync" "reddit:4:async" "reddit:8:sync" "reddit:8:async" \
                        "arxiv:4:sync" "arxiv:8:sync" "flickr:2:sync" "flickr:4:sync" "cora:2:sync"; do
              IFS=: read cfg m mode <<< "$spec"
              if [ "$m" = "1" ]; then lb=""; else lb="--loopback $m"; fi
              echo "== $cfg M=$m $mode" >> ${O}_matrix.log
              timeout 900 python bench.py --config $cfg $lb --mode $mode >> ${O}_matrix.jsonl 2>> ${O}_matrix.log
            done
            for spec in "products:8:0" "reddit:8:0" "reddit:1:0"; do
              IFS=: read cfg m rk <<< "$spec"
              timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
                --kernel-name regex:k_spmm --clock-control none --csv --log-file ${O}_matrix_ncu_${cfg}${m}.csv \
                python tools/spmm_bench.py --config $cfg --parts $m --rank $rk --iters 1 \
                --widths $([ $cfg = reddit ] && echo 256,48 || echo 256,100,48) >> ${O}_matrix.log 2>&1
            done ;;
    oracles) for spec in "cora:2:200:1" "cora:2:200:0" "flickr:2:1:0" "flickr:4:1:0" "arxiv:4:1:0" "arxiv:8:1:0" "reddit:1:1:0"; do
              IFS=: read cfg m ep th <<< "$spec"
              timeout 1500 python tools/oracle_full_epoch.py --config $cfg --parts $m --epochs $ep --threads $th >> ${O}_oracles.jsonl 2>> ${O}_oracles.log
            done
            grep -m1 "model name" /proc/cpuinfo >> ${O}_oracles.log ;;
    gemm)   timeout 900 python tools/gemm_bench.py --iters 10 > ${O}_gemm.log 2>&1 ;;
    ncuk)   # one SpMM kernel, full set + source: NCUK_KNOBS (comma list), NCUK_W width, NCUK_NAME tag
            env DIGEST_KNOBS=1 $(echo ${NCUK_KNOBS} | tr ',' ' ') timeout 900 $NCU --set full --import-source on \
              --clock-control none -k regex:k_spmm -c 1 -o ${O}_ncu_${NCUK_NAME} \
              python tools/spmm_bench.py --widths ${NCUK_W:-48} --iters 1 > ${O}_ncuk_${NCUK_NAME}.log 2>&1
            $NCU -i ${O}_ncu_${NCUK_NAME}.ncu-rep --page details --csv > ${O}_ncu_${NCUK_NAME}_details.csv 2>> ${O}_ncuk_${NCUK_NAME}.log
            $NCU -i ${O}_ncu_${NCUK_NAME}.ncu-rep --page source --csv > ${O}_ncu_${NCUK_NAME}_source.csv 2>> ${O}_ncuk_${NCUK_NAME}.log
            gzip -f ${O}_ncu_${NCUK_NAME}_source.csv; rm -f ${O}_ncu_${NCUK_NAME}.ncu-rep ;;
    ncudense) timeout 1200 $NCU --set full --import-source on --clock-control none \
                -k regex:"k_gemm|k_wgrad_bf16" -c ${NCUC:-14} -o ${O}_ncu_dense \
                python tools/gemm_bench.py --iters 1 --shapes ${NCUSHAPES:-256x48,100x256} > ${O}_ncudense.log 2>&1
              $NCU -i ${O}_ncu_dense.ncu-rep --page raw --csv > ${O}_ncu_dense_raw.csv 2>> ${O}_ncudense.log
              $NCU -i ${O}_ncu_dense.ncu-rep --page details --csv > ${O}_ncu_dense_details.csv 2>> ${O}_ncudense.log
              rm -f ${O}_ncu_dense.ncu-rep ;;
    *)      echo "unknown step $step" >> ${O}_errors.log ;;
  esac
done
ls -la gpurun_out > ${O}_ls.txt
