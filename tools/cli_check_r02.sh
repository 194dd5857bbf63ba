python -m paper_2402_06787_b200 topology --nvswitch 2 -o /tmp/nvs2.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29671 -m paper_2402_06787_b200 run -t /tmp/nvs2.json --collective allreduce --mib 256 2>&1 | grep "^{"
timeout 300 python -m pytest tests/test_gpu_api.py -k cli -q -p no:cacheprovider 2>&1 | tail -2
