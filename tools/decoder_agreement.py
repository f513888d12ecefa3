"""Decoder-path end-to-end agreement (bench.decoder_agreement) as a standalone
run: python tools/decoder_agreement.py [N] -> gpurun_out/decoder_agreement.json"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import bench

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    Path("gpurun_out").mkdir(exist_ok=True)
    out = {}
    for prec in ("fp32", "bf16"):
        out[prec] = bench.decoder_agreement(bench.WORKLOADS["wmt19_k50"], n, precision=prec)
        print(json.dumps({k: v for k, v in out[prec].items() if k != "divergences"}), flush=True)
    Path("gpurun_out/decoder_agreement.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
