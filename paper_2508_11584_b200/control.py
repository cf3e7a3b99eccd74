"""Control endpoint — SPEC's ``control`` transport: a local stream socket
carrying length-prefixed messages (4-byte little-endian length + UTF-8 payload). Requests are
the textual commands ``SETRATE <head> <hz>``, ``PAUSE <head>``, ``RESUME <head>``, ``STOP``,
``STATS``, ``FAULT <head>``; every request receives exactly one reply, ``OK [body]`` or
``ERR <code> <detail>``, in request order per connection (the implicit request id).

``ControlServer(dispatch, path)`` serves any ``dispatch(str) -> str`` callable (normally
``VPEngine.dispatch``) on a Unix-domain socket; ``send(path, *commands)`` is the client, also
usable from another process: ``python -m paper_2508_11584_b200.control <path> STATS``.
"""

from __future__ import annotations

import os
import socket
import struct
import sys
import threading

from .errors import ProtocolError

MAX_MESSAGE = 1 << 20


def _recv_exact(sock: socket.socket, n: int) -> bytes | None:
    buf = bytearray()
    while len(buf) < n:
        chunk = sock.recv(n - len(buf))
        if not chunk:
            return None if not buf else bytes(buf)
        buf += chunk
    return bytes(buf)


def read_message(sock: socket.socket) -> str | None:
    """One framed message, or None at a clean end of stream. ProtocolError on a torn frame."""
    head = _recv_exact(sock, 4)
    if head is None:
        return None
    if len(head) < 4:
        raise ProtocolError("truncated length prefix")
    (n,) = struct.unpack("<I", head)
    if n > MAX_MESSAGE:
        raise ProtocolError(f"message of {n} bytes exceeds {MAX_MESSAGE}")
    body = _recv_exact(sock, n) if n else b""
    if body is None or len(body) < n:
        raise ProtocolError("truncated message body")
    try:
        return body.decode("utf-8")
    except UnicodeDecodeError as exc:
        raise ProtocolError("message is not UTF-8") from exc


def write_message(sock: socket.socket, text: str) -> None:
    data = text.encode("utf-8")
    sock.sendall(struct.pack("<I", len(data)) + data)


class ControlServer:
    """Serves ``dispatch`` on a Unix stream socket at ``path`` until ``close()``. Each connection
    gets its own thread; replies are serialised per connection. A STOP reply is sent before the
    server stops accepting (replies even during shutdown)."""

    def __init__(self, dispatch, path: str):
        self.dispatch, self.path = dispatch, path
        if os.path.exists(path):
            os.unlink(path)
        self._sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        self._sock.bind(path)
        self._sock.listen(8)
        self._sock.settimeout(0.1)
        self._closing = threading.Event()
        self._lock = threading.Lock()  # one command at a time into the engine
        self._conns: list[threading.Thread] = []
        self._t = threading.Thread(target=self._accept, name="vpe-control", daemon=True)
        self._t.start()

    def _accept(self):
        while not self._closing.is_set():
            try:
                conn, _ = self._sock.accept()
            except socket.timeout:
                continue
            except OSError:
                break
            t = threading.Thread(target=self._serve, args=(conn,), daemon=True)
            t.start()
            self._conns.append(t)

    def _serve(self, conn: socket.socket):
        conn.settimeout(None)
        with conn:
            while True:
                try:
                    msg = read_message(conn)
                except ProtocolError as exc:
                    write_message(conn, f"ERR ProtocolError {exc}")
                    return
                except OSError:
                    return
                if msg is None:
                    return
                if self._closing.is_set():
                    reply = "ERR ShuttingDown engine is shutting down"
                else:
                    with self._lock:
                        try:
                            reply = self.dispatch(msg)
                        except Exception as exc:  # the dispatcher must not kill the endpoint
                            reply = f"ERR {type(exc).__name__} {exc}"
                try:
                    write_message(conn, reply)
                except OSError:
                    return

    def close(self):
        self._closing.set()
        try:
            self._sock.close()
        finally:
            self._t.join(timeout=2)
            if os.path.exists(self.path):
                os.unlink(self.path)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def send(path: str, *commands: str, timeout: float = 10.0) -> list[str]:
    """Send commands over one connection; returns one reply per command, in order."""
    with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as s:
        s.settimeout(timeout)
        s.connect(path)
        out = []
        for c in commands:
            write_message(s, c)
            r = read_message(s)
            if r is None:
                raise ProtocolError("server closed the connection before replying")
            out.append(r)
        return out


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if len(argv) < 2:
        print("usage: python -m paper_2508_11584_b200.control <socket> <COMMAND ...>", file=sys.stderr)
        return 2
    for r in send(argv[0], " ".join(argv[1:])):
        print(r)
        if r.startswith("ERR"):
            return 1
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
