"""Thread-backed stand-in for the ``greenlet`` package (TEST INFRASTRUCTURE).

The reference package imports ``greenlet`` in
``/root/reference/pkg/src/collectium/transport/sim.py:17`` for its virtual-time
simulator; greenlet is not installed in this image and there is no network.
This module provides the subset that ``sim.py`` uses (``greenlet(run,
parent)``, ``switch``, ``throw``, ``dead``, ``getcurrent``, ``GreenletExit``)
with one OS thread per greenlet and strict hand-off through semaphores, so at
most one of them runs at a time — the same cooperative semantics, only slower.

Only ``oracle/reference.py`` puts this directory on ``sys.path``; nothing in
the product package imports it.
"""

import threading

__version__ = "0-thread-shim"


class GreenletExit(BaseException):
    pass


_tls = threading.local()


class greenlet:  # noqa: N801 - mirrors the real package's class name
    def __init__(self, run=None, parent=None):
        self._run = run
        self.parent = parent if parent is not None else getcurrent()
        self._gate = threading.Semaphore(0)
        self._inbox = ()
        self._pending_exc = None
        self._started = False
        self.dead = False

    # -- scheduling -------------------------------------------------------
    def _main(self):
        _tls.current = self
        try:
            self._gate.acquire()
            self._raise_pending()
            self._run(*self._inbox)
        except GreenletExit:
            pass
        finally:
            self.dead = True
            target = self.parent
            target._inbox = ()
            target._gate.release()

    def _raise_pending(self):
        if self._pending_exc is not None:
            exc, self._pending_exc = self._pending_exc, None
            raise exc

    def _block(self):
        self._gate.acquire()
        self._raise_pending()

    def switch(self, *args):
        me = getcurrent()
        self._inbox = args
        if not self._started and self._run is not None:
            self._started = True
            threading.Thread(target=self._main, daemon=True).start()
        self._gate.release()
        me._block()
        return me._inbox[0] if me._inbox else None

    def throw(self, typ=GreenletExit):
        if not self._started:
            self.dead = True
            return
        if self.dead:
            return
        self._pending_exc = typ() if isinstance(typ, type) else typ
        me = getcurrent()
        self._gate.release()
        me._block()


def getcurrent():
    g = getattr(_tls, "current", None)
    if g is None:
        g = greenlet.__new__(greenlet)
        g._run = None
        g.parent = None
        g._gate = threading.Semaphore(0)
        g._inbox = ()
        g._pending_exc = None
        g._started = True
        g.dead = False
        _tls.current = g
    return g
