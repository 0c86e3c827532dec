"""Site-compiler worker process (engine.CompilePool): reads length-prefixed
pickled lists of (assertions, origin lookup) from stdin, compiles each with
engine._compile_one, writes the pickled result list to stdout.  An
exception (a CapacityError, say) is sent back as the result and re-raised by
the pool in the caller."""
import pickle
import struct
import sys


def main() -> None:
    from .engine import _compile_one

    rd, wr = sys.stdin.buffer, sys.stdout.buffer
    while True:
        head = rd.read(8)
        if len(head) != 8:
            return
        (n,) = struct.unpack("<Q", head)
        items = pickle.loads(rd.read(n))
        try:
            res = [_compile_one(it) for it in items]
        except BaseException as exc:  # noqa: BLE001 - forwarded to the caller
            res = exc
        data = pickle.dumps(res, protocol=pickle.HIGHEST_PROTOCOL)
        wr.write(struct.pack("<Q", len(data)) + data)
        wr.flush()


if __name__ == "__main__":
    main()
