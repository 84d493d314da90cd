set -x
python bench.py > gpurun_out/final_bench.log 2>&1
tail -1 gpurun_out/final_bench.log > gpurun_out/final_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python tools/prof_eval.py > gpurun_out/final_launches_run.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tree_eval -s 1 -c 1 -o gpurun_out/final_eval python tools/prof_eval.py > gpurun_out/final_eval_run.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:build_kernel|upward|moments_prep|tile_|sign_" -s 7 -c 7 -o gpurun_out/final_aux python tools/prof_eval.py > gpurun_out/final_aux_run.log 2>&1
python tools/predict_scaling.py > gpurun_out/final_predict.json 2> gpurun_out/final_predict.err
python tools/shard_balance.py > gpurun_out/final_balance.log 2>&1
ls -la gpurun_out/
