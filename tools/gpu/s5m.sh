# session 5: cfg4 strip width forced to 352 / 288 / 256 against the model's choice (320)
mkdir -p gpurun_out
timeout 900 python tools/time_libs.py cfg4 paper_1803_00004_b200/libbf.so tools/var/libbf_tw352.so tools/var/libbf_tw288.so tools/var/libbf_tw256.so > gpurun_out/s5m_time.txt 2>&1
cat gpurun_out/s5m_time.txt
python - <<'PY'
import paper_1803_00004_b200._bf as b, os
from synth import CONFIGS, config_params
spec=CONFIGS["cfg4"]; p=config_params(spec)
for lib in ["paper_1803_00004_b200/libbf.so","tools/var/libbf_tw352.so","tools/var/libbf_tw288.so","tools/var/libbf_tw256.so"]:
    pass
PY
