# session-4: two-stream software pipelining of consecutive steps (A/B probe)
python scripts/pipeline_probe.py 16777216 16384 64 int8 60
python scripts/pipeline_probe.py 16777216 32768 64 int8 60
python scripts/pipeline_probe.py 16777216 8192 64 int8 60
python scripts/pipeline_probe.py 16777216 4096 64 int8 60
python scripts/pipeline_probe.py 2147483648 65536 1 int8 40
python scripts/pipeline_probe.py 4194304 8192 256 float32 40
