"""LOBSTER ingestion throughput: mlob_store_load_lobster
(file read + GPU parse into the device store) against the reference's
data::load_lobster (oracle/_ref, one thread) on the same message / orderbook
pair.  The pair is synthetic: the synthetic generator's messages in LOBSTER
format and a fixed 10-level orderbook row per message (the loader parses every
message row and only the sampled orderbook rows; the row contents do not
change the work).  Prints one JSON line (messages/s, bytes/s)."""
import argparse
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02136_b200 import abi  # noqa: E402
from paper_2511_02136_b200.env import DeviceStore, HostStore  # noqa: E402


def write_pair(msgs, mpath, bpath, upt=100, depth=10):
    row = ",".join(f"{(10010 + i) * upt},{5 + i},{(10000 - i) * upt},{7 + i}" for i in range(depth)) + "\n"
    with open(mpath, "w") as mf, open(bpath, "w") as bf:
        lines = []
        for t, k, oid, q, p, sd in zip(msgs["time"].tolist(), msgs["kind"].tolist(), msgs["order_id"].tolist(),
                                       msgs["quantity"].tolist(), msgs["price"].tolist(), msgs["side"].tolist()):
            lines.append(f"{t // 1000000000}.{t % 1000000000:09d},{k + 1},{oid},{q},{p * upt},{1 if sd == 0 else -1}\n")
            if len(lines) == 100000:
                mf.write("".join(lines))
                bf.write(row * len(lines))
                lines = []
        mf.write("".join(lines))
        bf.write(row * len(lines))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--messages", type=int, default=4_000_000)
    p.add_argument("--sample-every", type=int, default=100)
    args = p.parse_args()
    d = tempfile.mkdtemp(prefix="lobster_", dir=os.environ.get("TMPDIR", "/tmp"))
    m, b = os.path.join(d, "msg.csv"), os.path.join(d, "book.csv")
    hs = HostStore.synth(abi.synth_config(n_messages=args.messages, state_sample_every=args.messages), 0)
    write_pair(hs.messages(), m, b)
    size = os.path.getsize(m) + os.path.getsize(b)
    DeviceStore.load_lobster(m, b, 100, args.sample_every)  # warm-up (CUDA context, module load)
    best = None
    for _ in range(3):
        w0 = time.perf_counter()
        st = DeviceStore.load_lobster(m, b, 100, args.sample_every)
        dt = time.perf_counter() - w0
        best = dt if best is None else min(best, dt)
    out = {"metric": "lobster ingestion messages/s", "unit": "messages/s", "value": args.messages / best,
           "bytes_per_s": size / best, "seconds": best,
           "config": {"messages": args.messages, "orderbook_levels": 10, "sample_every": args.sample_every,
                      "file_bytes": size, "states": len(st.states(cap=16))}}
    from oracle.oracle import Oracle, available
    if available("ref"):
        ref = Oracle("ref")
        w0 = time.perf_counter()
        ref.lobster(m, b, 100, args.sample_every)
        rdt = time.perf_counter() - w0
        out["cpu_baseline"] = {"value": args.messages / rdt, "unit": "messages/s", "cores": 1, "kind": "reference",
                               "sample": f"data::load_lobster on the same {size / 1e6:.0f} MB pair, wall {rdt:.2f}s"}
    print(json.dumps(out), flush=True)
    for f in (m, b):
        os.remove(f)
    os.rmdir(d)


if __name__ == "__main__":
    main()
